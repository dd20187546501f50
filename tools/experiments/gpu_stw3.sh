S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" ":: $S --mode pack" "POSDUMP_DIRECT_DRAIN=queue :: $S" 2>&1 | tee gpurun_out/stw3.txt
