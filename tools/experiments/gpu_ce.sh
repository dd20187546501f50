timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 200 python tools/probe_interference.py 2>&1 | tail -2
S="--steps 20 --warmup 3"
for a in "" "--workload c1" "--workload c1 --waves 4" "--waves 2"; do timeout 120 python tools/sweep.py ":: $S $a"; done 2>&1 | tee gpurun_out/ce1.txt
timeout 120 python tools/sweep.py "POSDUMP_DIRECT_DRAIN=sm :: $S" "POSDUMP_DIRECT_DRAIN=queue :: $S" 2>&1 | tee -a gpurun_out/ce1.txt
timeout 120 python tools/sweep.py ":: --steps 5 --warmup 3 --trace" 2>&1 | tail -3
timeout 300 python tools/sweep.py ":: --steps 5 --warmup 3 --workload c4 --waves 8" ":: --steps 5 --warmup 3 --workload c4 --waves 1" 2>&1 | tee -a gpurun_out/ce1.txt
