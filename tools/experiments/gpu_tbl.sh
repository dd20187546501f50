timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
S="--steps 20 --warmup 3 --no-cpu-baseline"
timeout 900 python tools/sweep.py ":: $S" ":: $S --workload c1" ":: --steps 5 --warmup 3 --workload c4" 2>&1 | tee gpurun_out/tbl.txt
mkdir -p gpurun_out/prof5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_chunks -s 12 -c 3 -o gpurun_out/prof5/hash_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; ls gpurun_out/prof5
