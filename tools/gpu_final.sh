# Final numbers of a round (under gpurun): tests, smoke, the default bench
# (BASELINE config 5) and its reference arm, the other workloads' lines, and
# the ncu launch list of the default bench command.
P=gpurun_out/final; mkdir -p $P
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | tee $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee $P/smoke.log
timeout 900 python bench.py > $P/bench_c5.jsonl 2> $P/bench_c5.err; cut -c1-300 $P/bench_c5.jsonl
timeout 900 python bench.py --impl reference > $P/bench_ref.jsonl 2> $P/bench_ref.err; cut -c1-300 $P/bench_ref.jsonl
timeout 600 python bench.py --workload c2 --steps 20 > $P/bench_c2.jsonl 2>/dev/null; cut -c1-300 $P/bench_c2.jsonl
timeout 600 python bench.py --workload c1 --steps 20 > $P/bench_c1.jsonl 2>/dev/null; cut -c1-300 $P/bench_c1.jsonl
timeout 900 python bench.py --workload c4 --steps 5 > $P/bench_c4.jsonl 2>/dev/null; cut -c1-300 $P/bench_c4.jsonl
timeout 900 python bench.py --workload c3 --steps 3 > $P/bench_c3.jsonl 2>/dev/null; cut -c1-300 $P/bench_c3.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $P/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-app-load > /dev/null 2>&1
ls -la $P
