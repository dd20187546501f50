timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" "POSDUMP_SCAN=single :: $S" ":: $S --workload c1" ":: $S --workload c1 --waves 1" ":: --steps 5 --warmup 3 --workload c4 --waves 1" ":: --steps 5 --warmup 3 --workload c4" ":: --steps 5 --warmup 3 --trace" 2>&1 | tee gpurun_out/tiles.txt
