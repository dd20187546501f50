# gather micro, new host-leg test, c2 trace, ncu of k_ship_runs in the c2 bench
P=gpurun_out/r2c; mkdir -p $P
timeout 120 ./tools/gather_micro > $P/gather_micro.txt 2>&1; cat $P/gather_micro.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "short_and_long_runs or direct_precopy_into_image" 2>&1 | tail -3
timeout 300 python bench.py --workload c2 --steps 10 --no-cpu-baseline --trace > $P/c2_trace.jsonl 2> $P/c2_trace.err; grep '^{' $P/c2_trace.err | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ship_runs -s 40 -c 2 -o $P/ncu_ship_c2 python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_ship.log 2>&1; tail -3 $P/ncu_ship.log
