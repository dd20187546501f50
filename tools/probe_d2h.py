"""Host-link probe: pinned D2H bandwidth for slice sizes / buffer offsets,
and with/without concurrent host-memory traffic (evidence for the host_link
roofline denominator)."""
import os, sys, time, json, threading
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_12079_b200 as pd
from paper_2405_12079_b200.posdump import D2H
import bench

print("numa", bench.bind_numa_local(0))
eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=512 << 20))
cache, cap = eng.cache()
s = pd.Stream()
res = {}
for pin_mb in (300, 600):
    pin = pd.PinnedHost(pin_mb << 20)
    for n_mb in (64, 256):
        n = n_mb << 20
        for slice_mb in (0, 2, 8, 64):
            best = 0
            for _ in range(4):
                eng.event_record(0, s)
                if slice_mb == 0:
                    pd.check(pd.lib().pos_memcpy(pin.ptr, cache, n, D2H, int(s)))
                else:
                    eng.d2h_async(pin.ptr, 0, n, stream=s, slice_bytes=slice_mb << 20)
                eng.event_record(1, s)
                best = max(best, n / (eng.event_elapsed(0, 1) * 1e-3) / 1e9)
            res[f"pin{pin_mb}_n{n_mb}_slice{slice_mb}"] = round(best, 2)
    # with host traffic
    img = np.zeros(256 << 20, np.uint8)
    stop = threading.Event()
    def hog():
        while not stop.is_set():
            img[:] = 1
    t = threading.Thread(target=hog); t.start()
    best = 0
    for _ in range(4):
        eng.event_record(0, s)
        eng.d2h_async(pin.ptr, 0, 64 << 20, stream=s)
        eng.event_record(1, s)
        best = max(best, (64 << 20) / (eng.event_elapsed(0, 1) * 1e-3) / 1e9)
    stop.set(); t.join()
    res[f"pin{pin_mb}_with_host_memset"] = round(best, 2)
    pin.close()
print(json.dumps(res))
