S="--steps 20 --warmup 3"
for a in "" "POSDUMP_DIRECT_QUEUE=0" "--workload c1" "--workload c1 --waves 4"; do
  if [[ "$a" == POSDUMP* ]]; then timeout 120 python tools/sweep.py "$a :: $S"; else timeout 120 python tools/sweep.py ":: $S $a"; fi
done 2>&1 | tee gpurun_out/queue3.txt
timeout 120 python tools/sweep.py ":: --steps 5 --warmup 3 --trace" 2>&1 | tail -3
timeout 300 python tools/sweep.py ":: --steps 5 --warmup 3 --workload c4 --waves 8" ":: --steps 5 --warmup 3 --workload c4 --waves 1" 2>&1 | tee -a gpurun_out/queue3.txt
