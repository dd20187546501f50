set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
P=gpurun_out/prof
mkdir -p $P
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $P/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_chunks -s 6 -c 1 -o $P/hash_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pack_scan -s 6 -c 1 -o $P/scan_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_host -s 6 -c 1 -o $P/drain_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_chunks -s 20 -c 1 -o $P/hash_c4 python bench.py --workload c4 --steps 1 --warmup 3 --waves 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_copy_bulk -c 1 -o $P/scatter_c4 python bench.py --workload c4 --steps 1 --warmup 3 --waves 8 --no-cpu-baseline > /dev/null 2>&1
ls -la $P
timeout 600 python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.jsonl
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.jsonl 2>&1; cat gpurun_out/bench_ref.jsonl
