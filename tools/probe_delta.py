"""STW delta probe: the bulk gather (k_copy_bulk) + post-stop hash of the C2
window write set, alone and with a concurrent 256 MiB pinned D2H."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2405_12079_b200 as pd
from paper_2405_12079_b200.posdump import D2H
import bench

wl = bench.Workload("c2")
mem = pd.DeviceMemory(wl.total + 256 * len(wl.sizes))
bufs, off = [], 0
for i, n in enumerate(wl.sizes):
    bufs.append(pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + off, size=n))
    off += (n + 255) // 256 * 256
pd.fill_batch([(b.dev_ptr, b.size, 5000 + b.handle) for b in bufs])
eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=512 << 20))
eng.register_buffers(bufs)
eng.plan_precopy()
win = sorted({h for k in wl.window(1) for h, _ in k})
big = pd.DeviceMemory(256 << 20)
pin = pd.PinnedHost(256 << 20)
s, cp = pd.Stream(1), pd.Stream()
for concurrent in (False, True):
    res = []
    for rep in range(6):
        eng.record_dirty(win)
        eng.prepare_final_stop(stream=s)
        s.synchronize()
        if concurrent:
            pd.check(pd.lib().pos_memcpy(pin.ptr, big.ptr, big.nbytes, D2H, int(cp)))
        eng.event_record(3, s)
        off, n = eng.at_final_stop(stream=s, stw_end_slot=4)
        pd.device_synchronize()
        res.append((round(eng.event_elapsed(3, 4), 4), round(eng.kernel_ms("delta"), 4), round(eng.kernel_ms("delta_hash"), 4)))
        eng.clear_dirty()
    print(json.dumps({"concurrent_d2h": concurrent, "buffers": len(win), "bytes": n, "stw_ms,gather_ms,hash_ms": res}))
