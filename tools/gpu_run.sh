mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -k "query or helpers" > gpurun_out/gpu_tests_sel.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_sel.log
timeout 900 python bench.py --workload config1 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_config1.json 2> gpurun_out/bench_config1.err
