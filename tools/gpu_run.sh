timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | grep -vE "^  |Warning|warnings.warn" | tail -15 > gpurun_out/gpu_tests.log
