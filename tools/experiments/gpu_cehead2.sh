# geometric copy-engine sub-batches (default) vs one batch per wave vs a 4-run head only
timeout 600 python -m pytest tests -m gpu -x -q -k "direct or delta or never_span" 2>&1 | tail -1
python tools/sweep.py ":: --steps 40 --warmup 3" "POSDUMP_CE_HEAD=0 :: --steps 40 --warmup 3" ":: --steps 40 --warmup 3" \
  ":: --steps 30 --warmup 3 --workload c1" "POSDUMP_CE_HEAD=0 :: --steps 30 --warmup 3 --workload c1" ":: --steps 30 --warmup 3 --workload c1" \
  ":: --steps 8 --warmup 3 --workload c4" "POSDUMP_CE_HEAD=0 :: --steps 8 --warmup 3 --workload c4" 2>&1 | cut -c1-200
