timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" "POSDUMP_SCAN=single :: $S" ":: --steps 5 --warmup 3 --trace" ":: $S" 2>&1 | tee gpurun_out/o1t.txt
