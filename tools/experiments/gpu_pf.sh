S="--steps 20 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" "POSDUMP_PF=slide :: $S" "POSDUMP_PF=slide;POSDUMP_PF_STEPS=16 :: $S" "POSDUMP_PF=slide;POSDUMP_PF_STEPS=64 :: $S" "POSDUMP_PF=slide;POSDUMP_PF_STEPS=128 :: $S" \
   ":: $S --workload c1 --waves 1" "POSDUMP_PF=slide :: $S --workload c1 --waves 1" "POSDUMP_PF=slide;POSDUMP_PF_STEPS=64 :: $S --workload c1 --waves 1" 2>&1 | tee gpurun_out/pf.txt
