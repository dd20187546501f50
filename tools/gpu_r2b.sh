# Round-2 check after the host-leg change (short runs by k_ship_runs): tests, smoke, c5/c2/c1 lines.
set -x
P=gpurun_out/r2b; mkdir -p $P
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > $P/pytest_gpu.log; tail -3 $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; tail -2 $P/smoke.log
timeout 600 python bench.py --no-cpu-baseline > $P/bench_c5.jsonl 2> $P/bench_c5.err; cut -c1-400 $P/bench_c5.jsonl; grep step $P/bench_c5.err
timeout 600 python bench.py --workload c2 --steps 20 --no-cpu-baseline > $P/bench_c2.jsonl 2>$P/bench_c2.err; cut -c1-400 $P/bench_c2.jsonl
timeout 600 python bench.py --workload c1 --steps 20 --no-cpu-baseline > $P/bench_c1.jsonl 2>$P/bench_c1.err; cut -c1-400 $P/bench_c1.jsonl
