set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -k "megakernel or config3 or grid or dropin" > gpurun_out/gpu_tests_sel.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_sel.log
for wl in config3 config5; do
  st=3; [ "$wl" = config5 ] && st=1
  timeout 900 python bench.py --workload $wl --steps $st --warmup 3 --no-cpu > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
done
