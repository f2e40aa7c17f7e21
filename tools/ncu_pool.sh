#!/bin/bash
# ncu --set full capture of the single-plane pool kernel (config-2 bench)
set -u
mkdir -p gpurun_out
python bench.py --no-cpu --steps 3 --warmup 3 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"pool_kernel" -s 3 -c 1 \
    -o gpurun_out/pool_full -f python bench.py --no-cpu --steps 3 --warmup 3 \
    > gpurun_out/ncu_pool.log 2>&1
echo "ncu rc=$?"
