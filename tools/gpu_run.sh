mkdir -p gpurun_out
for r in 1 2; do
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=line > gpurun_out/gpu_tests_rep$r.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_rep$r.log
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
