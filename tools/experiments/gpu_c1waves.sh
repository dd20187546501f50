# C1 wave plans: equal waves vs a one-hash-round first wave
python tools/sweep.py ":: --steps 30 --warmup 3 --workload c1" "POSDUMP_FIRST_WAVE=0.14 :: --steps 30 --warmup 3 --workload c1" \
  "POSDUMP_FIRST_WAVE=0.14 :: --steps 30 --warmup 3 --workload c1 --waves 2" "POSDUMP_FIRST_WAVE=0.14 :: --steps 30 --warmup 3 --workload c1 --waves 3" \
  ":: --steps 30 --warmup 3 --workload c1 --waves 2" ":: --steps 30 --warmup 3 --workload c1" 2>&1 | cut -c1-260
