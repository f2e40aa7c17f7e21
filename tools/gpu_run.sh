for v in pix smp pix smp; do MF_PATH_ORDER=$v python tools/c5_quick.py 2>&1 | cut -c1-60 | sed "s/^/$v /"; done > gpurun_out/c5.log
for v in pix smp; do MF_PATH_ORDER=$v python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v c3', d['value'], d['roofline']['frac'])"; done >> gpurun_out/c5.log
