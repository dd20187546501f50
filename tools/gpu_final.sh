# Final numbers of a round (under gpurun): ncu launch list + hash capture of
# the default bench, then every workload's bench line and the reference arm.
P=gpurun_out/final; mkdir -p $P
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $P/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_chunks -s 12 -c 4 -o $P/hash_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tiles -s 6 -c 1 -o $P/scan_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_bulk -s 3 -c 1 -o $P/gather_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 python bench.py > $P/bench_c2.jsonl 2> $P/bench_c2.err; cut -c1-400 $P/bench_c2.jsonl
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $P/bench_ref.jsonl 2>&1; cut -c1-300 $P/bench_ref.jsonl
timeout 900 python bench.py --workload c1 > $P/bench_c1.jsonl 2>/dev/null; cut -c1-300 $P/bench_c1.jsonl
timeout 900 python bench.py --workload c4 --steps 5 > $P/bench_c4.jsonl 2>/dev/null; cut -c1-300 $P/bench_c4.jsonl
timeout 900 python bench.py --workload c3 --steps 2 > $P/bench_c3.jsonl 2>/dev/null; cut -c1-300 $P/bench_c3.jsonl
timeout 900 python bench.py --workload c5 --steps 2 > $P/bench_c5.jsonl 2>/dev/null; cut -c1-300 $P/bench_c5.jsonl
ls -la $P
