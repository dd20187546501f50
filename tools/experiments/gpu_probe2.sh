./tools/batch_micro 2>&1 | tee gpurun_out/batch_micro.txt
S="--steps 20 --warmup 3"
python tools/sweep.py ":: $S --workload c1 --mode direct" ":: $S --workload c1 --mode direct --waves 4" "POSDUMP_HASH_CFG=512r12 :: $S" "POSDUMP_HASH_CFG=384x12 :: $S" "POSDUMP_HASH_CFG=512r12 :: $S --workload c1" 2>&1 | tee gpurun_out/probe2.txt
