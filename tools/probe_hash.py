"""Hash-kernel size scaling: k_hash_chunks (kModeHash) alone, CUDA-event timed,
over chunk counts from 1 to 16 Ki (64 KiB chunks, 4 MiB buffers), L2 flushed
before every launch (and once with a warm L2).  The intercept of time vs
bytes is the kernel's fixed cost (launch + table prologue + ramp); the slope
its streaming rate."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_12079_b200 as pd

CH = 65536
flush = pd.DeviceMemory(256 << 20)
mem = pd.DeviceMemory((16384 + 64) * CH)
pd.fill_batch([(mem.ptr, mem.nbytes, 7)])
pd.device_synchronize()
out = {}
for nch in [int(x) for x in os.environ.get("PROBE_CHUNKS", "1,148,592,1526,3052,6104,16384").split(",")]:
    per = 64  # chunks per buffer
    bufs, h, left, off = [], 1, nch, 0
    while left:
        k = min(per, left)
        bufs.append(pd.GpuBuffer(handle=h, dev_ptr=mem.ptr + off, size=k * CH))
        off += k * CH
        left -= k
        h += 1
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=CH, cache_capacity=0))
    eng.register_buffers(bufs)
    for warm in (False, True):
        ts = []
        for i in range(12):
            if not warm:
                pd.check(pd.lib().pos_memset(flush.ptr, i & 0xFF, flush.nbytes, None))
            eng.hash_chunks()
            pd.device_synchronize()
            if i >= 2:
                ts.append(eng.kernel_ms("hash") * 1e3)
        med = statistics.median(ts)
        out[f"{nch}{'w' if warm else ''}"] = {"us": round(med, 2), "min": round(min(ts), 2),
                                              "GBps": round(nch * CH / med / 1e3, 1)}
    eng.close() if hasattr(eng, "close") else None
    del eng
print(json.dumps(out))
