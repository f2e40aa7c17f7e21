python tools/dbg_w.py > gpurun_out/dbg_w.log 2>&1
