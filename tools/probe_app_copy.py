"""App copies during a checkpoint's host leg (engines.hpp:153-159: app >
ckpt at chunk granularity).  While a direct pre-copy moves 7.5 GB of runs
(60 x 125 MB buffers) to the host image, the application issues a 16 MiB
H2D and a 16 MiB D2H on its own stream: latency of each vs alone."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2405_12079_b200 as pd
from paper_2405_12079_b200.posdump import D2H, H2D

N, SZ = 60, 125_000_000
stride = (SZ + 255) // 256 * 256
mem = pd.DeviceMemory(N * stride)
bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * stride, size=SZ) for i in range(N)]
pd.fill_batch([(b.dev_ptr, b.size, 5000 + b.handle) for b in bufs])
pd.device_synchronize()
eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=1 << 30))
eng.register_buffers(bufs)
img = pd.PinnedHost(N * stride, image=True)
eng.register_image([img.array[i * stride:i * stride + SZ] for i in range(N)])
app_dev = pd.DeviceMemory(16 << 20)
app_host = pd.PinnedHost(16 << 20)
ckpt, drain, app = pd.Stream(priority=1), pd.Stream(priority=1), pd.Stream()


def app_copy(kind):
    eng.event_record(20, app)
    if kind == "h2d":
        pd.check(pd.lib().pos_memcpy(app_dev.ptr, app_host.ptr, 16 << 20, H2D, int(app)))
    else:
        pd.check(pd.lib().pos_memcpy(app_host.ptr, app_dev.ptr, 16 << 20, D2H, int(app)))
    eng.event_record(21, app)
    app.synchronize()
    return eng.event_elapsed(20, 21)


out = {}
for kind in ("h2d", "d2h"):
    out[f"{kind}_alone_ms"] = round(min(app_copy(kind) for _ in range(5)), 3)
for kind in ("h2d", "d2h"):
    eng.event_record(0, ckpt)
    eng.precopy_direct(waves=4, stream=ckpt, drain_stream=drain)
    time.sleep(0.02)  # the copy engine is busy with the runs now
    lat = app_copy(kind)
    eng.event_record(1, drain)
    drain.synchronize()
    eng.precopy_direct_result()
    out[f"{kind}_during_precopy_ms"] = round(lat, 3)
    out[f"precopy_ms_{kind}"] = round(eng.event_elapsed(0, 1), 1)
    eng.commit_epoch()
    eng.set_target_fresh(True)
print(out)
