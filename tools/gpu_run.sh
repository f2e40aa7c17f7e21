mkdir -p gpurun_out
for v in u1 u4 u8; do
MF_LIB_PATH=variants/$v.so timeout 900 python bench.py --workload gp --steps 3 --warmup 1 > gpurun_out/bench_gp_$v.json 2>&1
done
timeout 900 python -m pytest tests/test_gpu_gp.py -q -p no:cacheprovider --tb=short > gpurun_out/gp_tests.log 2>&1
echo "rc=$?" >> gpurun_out/gp_tests.log
