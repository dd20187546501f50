timeout 200 python tools/probe_interference2.py 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_hash_chunks<0' -s 6 -c 1 -o gpurun_out/prof3/hash_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; ls gpurun_out/prof3
