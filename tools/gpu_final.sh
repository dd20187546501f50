mkdir -p gpurun_out/prof4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_chunks -s 12 -c 3 -o gpurun_out/prof4/hash_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof4/ncu.log 2>&1; tail -3 gpurun_out/prof4/ncu.log
ls -la gpurun_out/prof4
timeout 900 python bench.py > gpurun_out/prof4/bench_c2.jsonl 2> gpurun_out/prof4/bench_c2.err; cat gpurun_out/prof4/bench_c2.jsonl | cut -c1-400
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/prof4/bench_ref.jsonl 2>&1; cut -c1-300 gpurun_out/prof4/bench_ref.jsonl
timeout 900 python bench.py --workload c1 > gpurun_out/prof4/bench_c1.jsonl 2>/dev/null; cut -c1-300 gpurun_out/prof4/bench_c1.jsonl
timeout 900 python bench.py --workload c4 --steps 5 > gpurun_out/prof4/bench_c4.jsonl 2>/dev/null; cut -c1-300 gpurun_out/prof4/bench_c4.jsonl
timeout 900 python bench.py --workload c3 --steps 2 > gpurun_out/prof4/bench_c3.jsonl 2>/dev/null; cut -c1-300 gpurun_out/prof4/bench_c3.jsonl
timeout 900 python bench.py --workload c5 --steps 2 > gpurun_out/prof4/bench_c5.jsonl 2>gpurun_out/prof4/bench_c5.err; cut -c1-300 gpurun_out/prof4/bench_c5.jsonl; tail -2 gpurun_out/prof4/bench_c5.err
