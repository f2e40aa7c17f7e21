mkdir -p gpurun_out
timeout 300 python tools/timeline.py > gpurun_out/timeline.txt 2>&1
