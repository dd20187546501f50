S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" "POSDUMP_NSEG=2 :: $S" "POSDUMP_NSEG=4 :: $S" "POSDUMP_NSEG=8 :: $S" "POSDUMP_NSEG=16 :: $S" "POSDUMP_HASH_CFG=384x12 :: $S" "POSDUMP_HASH_CFG=512r12 :: $S" 2>&1 | tee gpurun_out/nseg.txt
