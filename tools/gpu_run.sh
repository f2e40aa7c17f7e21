timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | grep -vE "^  |Warning|warnings.warn" | tail -6 > gpurun_out/gpu_tests.log
python tools/c5_quick.py 2>&1 | cut -c1-70 >> gpurun_out/gpu_tests.log
