P=gpurun_out/r2g; mkdir -p $P
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | tee $P/pytest_gpu.log
timeout 900 compute-sanitizer --tool memcheck --log-file $P/memcheck.txt python -m pytest tests/test_gpu_parity.py -q -x -k "direct or restore or delta or scatter" > $P/memcheck_pytest.log 2>&1; tail -2 $P/memcheck_pytest.log; tail -3 $P/memcheck.txt
timeout 600 python bench.py --no-cpu-baseline > $P/bench_c5.jsonl 2> $P/bench_c5.err; cut -c1-300 $P/bench_c5.jsonl
