# A/B on one box: engine-delimited STW window (default) vs the traced window (stamps + timer events)
python tools/sweep.py ":: --steps 40 --warmup 3" ":: --steps 40 --warmup 3 --trace" ":: --steps 40 --warmup 3" ":: --steps 40 --warmup 3 --trace" > gpurun_out/ab_stw.txt 2>&1
grep -v "^{" gpurun_out/ab_stw.txt | grep "::" | cut -c1-330
