timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
S="--steps 5 --warmup 3 --workload c4"
python tools/sweep.py ":: $S --waves 4" ":: $S --waves 8" ":: $S --waves 16" ":: --steps 20 --warmup 3" ":: --steps 20 --warmup 3 --workload c1 --waves 4" 2>&1 | tee gpurun_out/c4b_sweep.txt
