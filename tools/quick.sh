#!/bin/bash
# One gpurun call for an optimisation step: GPU parity suite, a bench line
# (no CPU baseline) and the per-config throughput table.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/q_tests.log
python bench.py --no-cpu > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
echo "bench rc=$?"; cat gpurun_out/q_bench.json
timeout 600 python tools/perf_configs.py > gpurun_out/q_perf.json 2> gpurun_out/q_perf.err
echo "perf rc=$?"; cat gpurun_out/q_perf.json
