mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -k "helpers or curves" > gpurun_out/gpu_tests_sel.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_sel.log
