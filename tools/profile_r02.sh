#!/bin/bash
# Round-2 measurement pass (one gpurun call): bench lines of every workload
# (no profiler), the ncu launch list of the headline bench command, and
# ncu --set full captures of the dominant kernel of configs 4, 3 and 5.
# Summarise afterwards with tools/summarize_ncu.py.
set -u
mkdir -p gpurun_out
for wl in ${WORKLOADS:-config1 config2 config3 config5}; do
  st=3; [ "$wl" = config5 ] && st=1
  timeout 900 python bench.py --workload $wl --steps $st --warmup 3 --no-cpu \
      > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
  echo "bench $wl rc=$?"; cut -c1-300 gpurun_out/bench_$wl.json
done
if [ "${NCU:-1}" = 1 ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch_c4.log 2>&1
echo "ncu launches rc=$?"
# config 4: the centre panel (sigma 0.05, l_z 0.1) = 5th pool launch
ncu --set full --clock-control none --import-source on -k regex:"pool_kernel" -s 4 -c 1 \
    -o gpurun_out/c4_full -f python bench.py --steps 1 --warmup 3 --no-cpu \
    > gpurun_out/ncu_c4_full.log 2>&1
echo "ncu c4 full rc=$?"
bash tools/ncu_c3.sh
MF_NCU_C5=1 bash -c 'sed -e s/c3_full/c5_full/ tools/ncu_c3.sh | bash'
fi
