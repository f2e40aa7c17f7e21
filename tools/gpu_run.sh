mkdir -p gpurun_out
timeout 1200 python tools/time_variants.py variants/out.so variants/spec1.so variants/ndfg.so variants/spec1mb7.so variants/out.so variants/spec1.so variants/ndfg.so variants/spec1mb7.so > gpurun_out/variants.txt 2>&1
