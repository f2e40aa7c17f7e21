mkdir -p gpurun_out
timeout 1200 python tools/time_variants.py variants/*.so > gpurun_out/variants.txt 2>&1
