export POSDUMP_WATCHDOG_MS=3000
timeout 60 python bench.py --steps 3 --warmup 3 --trace --no-cpu-baseline --workload c1 > gpurun_out/q.out 2> gpurun_out/q.err; echo rc=$?
grep "ship_queue" gpurun_out/q.err | head -2; grep -o '"value": [0-9.]*' gpurun_out/q.out
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
S="--steps 20 --warmup 3"
for a in "" "--workload c1" "--waves 2"; do timeout 120 python tools/sweep.py ":: $S $a"; done 2>&1 | tee gpurun_out/queue2.txt
