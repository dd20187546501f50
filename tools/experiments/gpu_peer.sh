timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py --workload c3 --steps 2 --warmup 3 --peer-cache-gb 40 > gpurun_out/bench_c3_peer.jsonl 2> gpurun_out/bench_c3_peer.err; tail -c 2000 gpurun_out/bench_c3_peer.jsonl; tail -3 gpurun_out/bench_c3_peer.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hash_chunks<0" -s 6 -c 1 -o gpurun_out/prof/hash_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; ls gpurun_out/prof
