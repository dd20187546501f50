# final check of the adaptive copy-engine head (default) vs one batch per wave
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/sweep.py ":: --steps 40 --warmup 3" "POSDUMP_CE_HEAD=0 :: --steps 40 --warmup 3" ":: --steps 40 --warmup 3 --workload c1" "POSDUMP_CE_HEAD=0 :: --steps 40 --warmup 3 --workload c1" \
  ":: --steps 8 --warmup 3 --workload c4" "POSDUMP_CE_HEAD=0 :: --steps 8 --warmup 3 --workload c4" 2>&1 | cut -c1-140 | tee gpurun_out/cehead5.txt
