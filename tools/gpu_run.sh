mkdir -p gpurun_out
timeout 1500 python tools/time_variants.py variants/nopf.so variants/pf.so variants/nopf.so variants/pf.so > gpurun_out/variants.txt 2>&1
