#!/bin/bash
# Round-2 measurement pass (one gpurun call): GPU tests, bench lines of
# every workload (no profiler), the ncu launch list of the headline bench
# command, and ncu --set full captures of the dominant kernel of each
# workload.  Summarise afterwards with tools/profile_summary.py.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/gpu_tests_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err
echo "bench config4 rc=$?"
for wl in ${WORKLOADS:-config1 config2 config3 config5 gp}; do
  st=3; [ "$wl" = config5 ] && st=1
  timeout 900 python bench.py --workload $wl --steps $st --warmup 3 --no-cpu \
      > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
  echo "bench $wl rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
if [ "${NCU:-1}" = 1 ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch_c4.log 2>&1
echo "ncu launches rc=$?"
# config 4 at bench size: the centre panel (sigma 0.05, l_z 0.1) = 5th pool launch
ncu --set full --clock-control none --import-source on -k regex:"pool_kernel" -s 4 -c 1 \
    -o gpurun_out/c4_full -f python bench.py --steps 1 --warmup 3 --no-cpu \
    > gpurun_out/ncu_c4_full.log 2>&1
echo "ncu c4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"query_kernel" -s 1 -c 1 \
    -o gpurun_out/c1_full -f python tools/ncu_query.py 1 > gpurun_out/ncu_c1.log 2>&1
echo "ncu c1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"curved_pool_kernel" -s 1 -c 1 \
    -o gpurun_out/c3_full -f python tools/ncu_render.py config3 512 256 > gpurun_out/ncu_c3.log 2>&1
echo "ncu c3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"grid_pool_kernel" -s 1 -c 1 \
    -o gpurun_out/c5_full -f python tools/ncu_render.py config5 512 64 > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?"
fi
