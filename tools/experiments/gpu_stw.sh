S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" ":: $S --mode pack" ":: --steps 5 --warmup 3 --trace" ":: $S --workload c1" 2>&1 | tee gpurun_out/stw.txt
