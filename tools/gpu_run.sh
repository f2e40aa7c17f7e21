timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short -s -k "not nothing" 2>&1 | grep -vE "^  |Warning|warnings.warn" | grep -E "config3 128|passed|failed|Error|^E |FAIL" | tail -30 > gpurun_out/gpu_tests.log
timeout 600 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_config3.json 2> gpurun_out/bench_config3.err
python -c "
import json; d=json.load(open('gpurun_out/bench_config3.json')); r=d['roofline']
print('c3', d['value'], d['ms_per_step'], r['frac'], d['stats_per_path']['track_steps'])" >> gpurun_out/gpu_tests.log
