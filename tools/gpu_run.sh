mkdir -p gpurun_out
timeout 1500 python tools/time_variants.py variants/base.so variants/constm.so variants/base.so variants/constm.so > gpurun_out/variants.txt 2>&1
