set -x
free -g; nproc; lscpu | head -30; numactl -H 2>/dev/null | head; nvidia-smi; nvidia-smi topo -m
python - <<'PY'
import time, torch
t=time.time(); x=torch.empty(int(32e9), dtype=torch.uint8, pin_memory=True); print("pin 32GB", time.time()-t)
del x
PY
ulimit -l
cat /proc/meminfo | head -5
