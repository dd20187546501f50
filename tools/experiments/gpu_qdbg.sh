export POSDUMP_WATCHDOG_MS=3000
timeout 120 python bench.py --steps 3 --warmup 3 --trace --no-cpu-baseline > gpurun_out/qdbg.out 2> gpurun_out/qdbg.err; echo rc=$?
tail -5 gpurun_out/qdbg.out; grep -v "^{\"precopy" gpurun_out/qdbg.err | tail -30
timeout 120 python bench.py --steps 3 --warmup 3 --trace --no-cpu-baseline --ckpt-priority 0 > gpurun_out/qdbg2.out 2> gpurun_out/qdbg2.err; echo rc=$?
tail -3 gpurun_out/qdbg2.out | cut -c1-300; tail -8 gpurun_out/qdbg2.err
