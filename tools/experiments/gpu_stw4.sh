# STW window holding only the gather (pos_final_stop) vs the traced window
timeout 600 python -m pytest tests -m gpu -x -q -k "delta or direct or smoke" 2>&1 | tail -2
python tools/sweep.py ":: --steps 30 --warmup 3" ":: --steps 30 --warmup 3 --workload c1" ":: --steps 10 --warmup 3 --workload c4" > gpurun_out/stw4.txt 2>&1
cat gpurun_out/stw4.txt
python bench.py --steps 4 --warmup 3 --no-cpu-baseline --trace 2>&1 >/dev/null | grep -v ship_queue | tail -2
