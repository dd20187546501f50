"""Does a live zero-copy drain slow the hash kernel?  Engine A hashes 1 GiB
(pos_hash_chunks) alone, then while engine B's direct pre-copy drains 1 GiB
into a pinned image (SM stores over PCIe), then while a copy-engine D2H of
1 GiB runs."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2405_12079_b200 as pd  # noqa: E402

N = 64
SZ = 16 << 20


def make(seed):
    mem = pd.DeviceMemory(N * SZ)
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * SZ, size=SZ) for i in range(N)]
    pd.fill_batch([(b.dev_ptr, SZ, seed + i) for i, b in enumerate(bufs)])
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=64 << 20))
    eng.register_buffers(bufs)
    return mem, bufs, eng


ma, ba, A = make(100)
mb, bb, B = make(200)
pin = pd.PinnedHost(N * SZ)
B.register_image([pin.array[i * SZ:(i + 1) * SZ] for i in range(N)])
hostbuf = pd.PinnedHost(N * SZ)
sa, sb, db = pd.Stream(priority=1), pd.Stream(priority=1), pd.Stream(priority=1)
pd.device_synchronize()


def hash_a():
    A.hash_chunks(stream=sa)
    sa.synchronize()
    return A.kernel_ms("hash")


for _ in range(3):
    hash_a()
alone = min(hash_a() for _ in range(5))
res = {"alone_ms": alone}
for mode in ("queue_drain", "ce_d2h", "queue_drain_no_copy"):
    ts = []
    for r in range(4):
        if mode.startswith("queue_drain"):
            B.commit_epoch() if mode == "queue_drain_no_copy" and r > 0 else None
            B.precopy_direct(waves=1, stream=sb, drain_stream=db)
        else:
            pd.check(pd.lib().pos_memcpy(hostbuf.ptr, mb.ptr, N * SZ, 2, int(sb)))
        time.sleep(0.0005)  # let the concurrent work get going
        ts.append(hash_a())
        sb.synchronize()
        db.synchronize()
        if mode.startswith("queue_drain"):
            B.precopy_direct_result()
            if mode == "queue_drain":
                B.register_buffers(bb)  # fresh epoch: everything dirty again
                B.register_image([pin.array[i * SZ:(i + 1) * SZ] for i in range(N)])
    res[mode + "_ms"] = min(ts)
print(res)
