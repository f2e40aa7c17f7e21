#!/bin/bash
# One gpurun call: bench (no profiler) -> ncu launch list -> ncu --set full
# of the path kernel.  Outputs under gpurun_out/; summarise afterwards with
#   python tools/summarize_ncu.py <tag> gpurun_out/path_full.ncu-rep gpurun_out/launches.csv
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
rc=$?
echo "bench rc=$rc"; cat gpurun_out/bench.json
[ $rc -eq 0 ] || exit $rc
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "reference rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 \
    > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"pool_kernel|path_kernel" -s 3 -c 1 \
    -o gpurun_out/path_full -f python bench.py --steps 3 --warmup 3 \
    > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
