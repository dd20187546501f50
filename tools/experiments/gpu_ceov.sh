S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" "POSDUMP_CE_OVERLAP=1 :: $S" ":: $S" "POSDUMP_CE_OVERLAP=1 :: $S" "POSDUMP_CE_OVERLAP=1 :: --steps 5 --warmup 3 --workload c4" 2>&1 | tee gpurun_out/ceov.txt
