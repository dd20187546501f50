timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
S="--steps 20 --warmup 3"
python tools/sweep.py ":: $S --mode pack" ":: $S" ":: --steps 5 --warmup 3 --trace" ":: $S --waves 2" ":: $S --workload c1" ":: $S --workload c1 --waves 4" ":: $S --workload c1 --mode pack" 2>&1 | tee gpurun_out/scan1.txt
