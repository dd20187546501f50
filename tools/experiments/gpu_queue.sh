timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
S="--steps 20 --warmup 3"
python tools/sweep.py ":: $S" "POSDUMP_DIRECT_QUEUE=0 :: $S" ":: --steps 5 --warmup 3 --trace" ":: $S --waves 2" ":: $S --workload c1" "POSDUMP_DIRECT_QUEUE=0 :: $S --workload c1" ":: $S --workload c1 --waves 4" ":: --steps 5 --warmup 3 --workload c4 --waves 8" ":: --steps 5 --warmup 3 --workload c4 --waves 1" 2>&1 | tee gpurun_out/queue1.txt
