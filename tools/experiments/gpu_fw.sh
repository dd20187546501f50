python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" ":: $S --waves 2" "POSDUMP_FIRST_WAVE=0.1 :: $S --waves 2" "POSDUMP_FIRST_WAVE=0.2 :: $S --waves 2" "POSDUMP_FIRST_WAVE=0.1 :: $S --waves 3" "POSDUMP_FIRST_WAVE=0.05 :: $S --waves 3" ":: $S" 2>&1 | tee gpurun_out/fw.txt
