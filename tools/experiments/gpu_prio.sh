S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" ":: $S --drain-priority 0" ":: $S --ckpt-priority 0 --drain-priority 0" ":: $S --drain-priority 0" ":: $S" 2>&1 | tee gpurun_out/prio.txt
