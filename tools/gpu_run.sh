timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -2 gpurun_out/bench_c4.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], [round(x,1) for x in r['kernel_ms_per_scene']])"
