# first-chunk warm-up overlapped with the table prologue
timeout 600 python -m pytest tests -m gpu -x -q -k "digest or direct or pipelined or delta" 2>&1 | tail -2
./tools/hash_micro 2>&1 | grep -E "^pf=0 |back-to-back" | head -9
timeout 300 python tools/probe_hash.py
python tools/sweep.py ":: --steps 30 --warmup 3" ":: --steps 20 --warmup 3 --workload c1" 2>&1 | cut -c1-300
