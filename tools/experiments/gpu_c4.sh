free -g | head -2; nproc
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --waves 8 --no-cpu-baseline > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err; tail -c 2500 gpurun_out/bench_c4.jsonl; tail -5 gpurun_out/bench_c4.err
python tools/sweep.py ":: --steps 5 --warmup 3 --workload c4 --waves 1" ":: --steps 5 --warmup 3 --workload c4 --waves 16" 2>&1 | tee gpurun_out/c4_sweep.txt
