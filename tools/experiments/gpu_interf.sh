timeout 300 python tools/probe_interference.py 2>&1 | tail -3
