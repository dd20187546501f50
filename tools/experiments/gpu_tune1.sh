S="--steps 20 --warmup 3"
python tools/sweep.py ":: $S" "POSDUMP_PF=65536 :: $S" "POSDUMP_PF=32768 :: $S" \
  "POSDUMP_HASH_CFG=512r16 :: $S" "POSDUMP_HASH_CFG=256x16 :: $S" "POSDUMP_NSEG=2 :: $S" "POSDUMP_NSEG=2;POSDUMP_PF=65536 :: $S" \
  ":: $S --waves 2" ":: $S --waves 3" ":: $S --waves 4" ":: $S --no-host-apply" ":: --steps 5 --warmup 3 --trace" \
  ":: $S --workload c1" ":: $S --workload c1 --waves 4" "POSDUMP_PF=65536 :: $S --workload c1" "POSDUMP_HASH_CFG=512r16 :: $S --workload c1" 2>&1 | tee gpurun_out/tune1.txt
