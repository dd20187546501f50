# C4 wave plans in copy-engine direct mode
python tools/sweep.py ":: --steps 8 --warmup 3 --workload c4" ":: --steps 8 --warmup 3 --workload c4 --waves 16" \
  "POSDUMP_FIRST_WAVE=0.04 :: --steps 8 --warmup 3 --workload c4 --waves 12" "POSDUMP_FIRST_WAVE=0.06 :: --steps 8 --warmup 3 --workload c4 --waves 8" 2>&1 | cut -c1-330
