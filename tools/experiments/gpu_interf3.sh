timeout 200 python tools/probe_interference2.py 2>&1 | tail -1
POSDUMP_COPY=vec timeout 200 python tools/probe_interference2.py 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "direct or delta or scatter or compact" 2>&1 | tail -2
POSDUMP_COPY=vec timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "delta or scatter or compact or restore or pipelined" 2>&1 | tail -2
S="--steps 20 --warmup 3"
timeout 120 python tools/sweep.py ":: $S" ":: --steps 5 --warmup 3 --trace" 2>&1 | tail -4
mkdir -p gpurun_out/prof3
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_hash_chunks<0' -s 6 -c 1 -o gpurun_out/prof3/hash_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; ls gpurun_out/prof3
