timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "direct or host_image or pipelined" 2>&1 | tail -15
S="--steps 20 --warmup 3"
python tools/sweep.py ":: $S" ":: $S --mode direct" ":: $S --mode direct --waves 2" ":: $S --mode direct --waves 4" \
  "POSDUMP_HOST_CTAS=8 :: $S --mode direct" "POSDUMP_HOST_CTAS=32 :: $S --mode direct" ":: --steps 5 --warmup 3 --trace --mode direct" \
  ":: $S --workload c1 --mode direct" ":: $S --workload c1 --mode direct --waves 4" 2>&1 | tee gpurun_out/direct1.txt
