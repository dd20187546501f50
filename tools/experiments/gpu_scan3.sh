timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
S="--steps 20 --warmup 3"
python tools/sweep.py ":: $S" ":: --steps 5 --warmup 3 --trace" ":: $S --waves 2" "POSDUMP_HOST_CTAS=32 :: $S" ":: $S --workload c1" 2>&1 | tee gpurun_out/scan3.txt
