export POSDUMP_WATCHDOG_MS=2000
for spec in ":: --workload c1"; do
  env_s="${spec%%::*}"; args="${spec#*::}"
  echo "== $spec"
  env $env_s timeout 60 python bench.py --steps 3 --warmup 3 --trace --no-cpu-baseline $args > gpurun_out/q.out 2> gpurun_out/q.err; echo rc=$?
  grep -o '"value": [0-9.]*' gpurun_out/q.out; grep "ship_queue\|Error" gpurun_out/q.err | head -4
done
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "direct" 2>&1 | tail -3
