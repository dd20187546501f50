export POSDUMP_WATCHDOG_MS=2000
timeout 60 python bench.py --steps 3 --warmup 3 --trace --no-cpu-baseline --workload c1 > gpurun_out/q.out 2> gpurun_out/q.err; echo rc=$?
grep "ship_queue" gpurun_out/q.err | head -4
