mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gp.py -q -p no:cacheprovider --tb=short > gpurun_out/gpu_tests_sel.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_sel.log
timeout 900 python bench.py --workload gp --steps 3 --warmup 1 > gpurun_out/bench_gp.json 2> gpurun_out/bench_gp.err
timeout 600 python tools/gp_profile.py > gpurun_out/gp_profile.txt 2>&1
