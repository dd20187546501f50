timeout 300 python tools/probe_queue.py 2>&1 | tail -12
