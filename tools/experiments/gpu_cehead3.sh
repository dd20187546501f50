# copy-engine head batch size
for wl in "" "--workload c1"; do
python tools/sweep.py "POSDUMP_CE_HEAD=0 :: --steps 40 --warmup 3 $wl" "POSDUMP_CE_HEAD=4 :: --steps 40 --warmup 3 $wl" "POSDUMP_CE_HEAD=16 :: --steps 40 --warmup 3 $wl" \
  "POSDUMP_CE_HEAD=64 :: --steps 40 --warmup 3 $wl" "POSDUMP_CE_HEAD=0 :: --steps 40 --warmup 3 $wl" "POSDUMP_CE_HEAD=16 :: --steps 40 --warmup 3 $wl" 2>&1 | cut -c1-130
done
