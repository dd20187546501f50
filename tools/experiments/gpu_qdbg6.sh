timeout 300 python tools/probe_queue.py 2>&1 | tail -12
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
S="--steps 20 --warmup 3"
for a in "" "--mode pack" "--workload c1" "--waves 2" "--workload c1 --waves 4"; do timeout 120 python tools/sweep.py ":: $S $a"; done 2>&1 | tee gpurun_out/queue2.txt
timeout 120 python tools/sweep.py ":: --steps 5 --warmup 3 --trace" 2>&1 | tail -4
timeout 300 python tools/sweep.py ":: --steps 5 --warmup 3 --workload c4 --waves 8" ":: --steps 5 --warmup 3 --workload c4 --waves 1" 2>&1 | tee -a gpurun_out/queue2.txt
