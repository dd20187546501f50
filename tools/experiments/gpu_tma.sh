POSDUMP_HASH_CFG=512t6 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "digest or crc32 or direct or tiled or c1_full or delta or unaligned or o1" 2>&1 | tail -2
POSDUMP_HASH_CFG=512t8 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "digest or crc32 or tiled" 2>&1 | tail -2
S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" "POSDUMP_HASH_CFG=512t6 :: $S" "POSDUMP_HASH_CFG=512t8 :: $S" ":: $S --workload c1 --waves 1" "POSDUMP_HASH_CFG=512t6 :: $S --workload c1 --waves 1" "POSDUMP_HASH_CFG=512t6 :: --steps 5 --warmup 3 --workload c4 --waves 1" ":: --steps 5 --warmup 3 --workload c4 --waves 1" 2>&1 | tee gpurun_out/tma.txt
