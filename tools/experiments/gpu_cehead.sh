# first batch of k runs submitted alone (copy engine starts earlier?)
python tools/sweep.py ":: --steps 40 --warmup 3" "POSDUMP_CE_HEAD=4 :: --steps 40 --warmup 3" "POSDUMP_CE_HEAD=16 :: --steps 40 --warmup 3" \
  ":: --steps 40 --warmup 3" "POSDUMP_CE_HEAD=4 :: --steps 40 --warmup 3" "POSDUMP_CE_HEAD=64 :: --steps 30 --warmup 3 --workload c1" ":: --steps 30 --warmup 3 --workload c1" 2>&1 | cut -c1-200
