mkdir -p gpurun_out
timeout 1500 python tools/time_variants.py variants/noguard.so variants/guard.so variants/noguard.so variants/guard.so > gpurun_out/variants.txt 2>&1
