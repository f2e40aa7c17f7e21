mkdir -p gpurun_out
timeout 1500 python tools/time_variants.py variants/old.so variants/new.so variants/old.so variants/new.so > gpurun_out/variants.txt 2>&1
