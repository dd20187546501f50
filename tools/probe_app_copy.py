"""App copies during a checkpoint's host leg (engines.hpp:153-159: app >
ckpt at chunk granularity).  While a direct pre-copy moves 7.5 GB of runs
(60 x 125 MB buffers) to the host image, the application issues a 16 MiB
H2D / D2H on its own stream, either as a plain cudaMemcpyAsync ("raw") or
through pos_app_copy ("managed": the host leg yields to it): latency vs
alone, and the pre-copy's duration."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
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


def app_copy(kind, managed):
    eng.event_record(20, app)
    dst, src = (app_dev.ptr, app_host.ptr) if kind == "h2d" else (app_host.ptr, app_dev.ptr)
    k = H2D if kind == "h2d" else D2H
    if managed:
        eng.app_copy(dst, src, 16 << 20, k, stream=app)
    else:
        pd.check(pd.lib().pos_memcpy(dst, src, 16 << 20, k, int(app)))
    eng.event_record(21, app)
    app.synchronize()
    return eng.event_elapsed(20, 21)


out = {}
for kind in ("h2d", "d2h"):
    out[f"{kind}_alone_ms"] = round(min(app_copy(kind, False) for _ in range(5)), 3)
for slice_mb, window in ((16, 3), (8, 2), (64, 4)):
    eng.set_host_leg(slice_mb << 20, window)
    for managed in (False, True):
        for kind in ("h2d", "d2h"):
            eng.set_target_fresh(True)
            eng.event_record(0, ckpt)
            eng.precopy_direct(waves=4, stream=ckpt, drain_stream=drain)
            time.sleep(0.03)  # the copy engine is busy with the runs now
            lat = app_copy(kind, managed)
            eng.precopy_direct_result()
            eng.event_record(1, drain)
            drain.synchronize()
            tag = f"slice{slice_mb}M_w{window}_{'managed' if managed else 'raw'}_{kind}"
            out[tag] = {"app_ms": round(lat, 3), "precopy_ms": round(eng.event_elapsed(0, 1), 1),
                        "precopy_GBps": round(N * SZ / eng.event_elapsed(0, 1) / 1e6, 2)}
            eng.commit_epoch()
out["slices, app_yields"] = eng.host_leg_stats()
print(json.dumps(out, indent=1))
