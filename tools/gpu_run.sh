mkdir -p gpurun_out
( python tools/ab_env.py MF_GRID_TEXTURE config5 256 16; python tools/ab_env.py MF_GRID_TEXTURE config5 512 16 ) > gpurun_out/ab.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -k "grid" > gpurun_out/gpu_tests_sel.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_sel.log
