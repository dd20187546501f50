# adaptive copy-engine head batch (default) vs one batch vs fixed heads
timeout 600 python -m pytest tests -m gpu -x -q -k "direct or delta or never_span or buffer_set" 2>&1 | tail -1
for wl in "" "--workload c1"; do
python tools/sweep.py ":: --steps 40 --warmup 3 $wl" "POSDUMP_CE_HEAD=0 :: --steps 40 --warmup 3 $wl" "POSDUMP_CE_HEAD=4 :: --steps 40 --warmup 3 $wl" \
  "POSDUMP_CE_HEAD=64 :: --steps 40 --warmup 3 $wl" ":: --steps 40 --warmup 3 $wl" 2>&1 | cut -c1-130
done
python tools/sweep.py ":: --steps 8 --warmup 3 --workload c4" "POSDUMP_CE_HEAD=0 :: --steps 8 --warmup 3 --workload c4" 2>&1 | cut -c1-130
