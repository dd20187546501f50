timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
S="--steps 30 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" ":: $S --mode pack" ":: --steps 5 --warmup 3 --trace" 2>&1 | tee gpurun_out/stw2.txt
