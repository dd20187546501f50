timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
P=gpurun_out/prof2; mkdir -p $P
S="--steps 20 --warmup 3"
timeout 120 python tools/sweep.py ":: $S" ":: --steps 5 --warmup 3 --trace" 2>&1 | tee $P/sweep.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $P/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hash_chunks<0" -s 6 -c 1 -o $P/hash_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pack_scan -s 6 -c 1 -o $P/scan_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls $P
