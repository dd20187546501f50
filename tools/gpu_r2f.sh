P=gpurun_out/r2f; mkdir -p $P
timeout 300 ./tools/gather_micro > $P/gather_micro.txt 2>&1; grep -E "17166|2048" $P/gather_micro.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ship -s 3 -c 1 -o $P/ncu_ship_c1 python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_ship.log 2>&1; tail -2 $P/ncu_ship.log
timeout 900 compute-sanitizer --tool memcheck --log-file $P/memcheck.txt python -m pytest tests/test_gpu_parity.py -q -x -k "direct or restore or delta or scatter" > $P/memcheck_pytest.log 2>&1; tail -2 $P/memcheck_pytest.log; tail -3 $P/memcheck.txt
