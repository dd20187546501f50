# Round-end style check on one B200 (under gpurun): tests, smoke, bench lines.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c5.jsonl 2> gpurun_out/bench_c5.err; tail -c 3000 gpurun_out/bench_c5.jsonl
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.jsonl 2>gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.jsonl
