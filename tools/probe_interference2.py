"""STW gather (TMA bulk copy into the cache) alone vs beside a copy-engine
direct drain (copy-engine runs, ~16K of 64 KiB) and beside a plain
CE D2H of 1 GiB."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_12079_b200 as pd  # noqa: E402

N, SZ = 64, 16 << 20


def make(seed, cache):
    mem = pd.DeviceMemory(N * SZ)
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * SZ, size=SZ) for i in range(N)]
    pd.fill_batch([(b.dev_ptr, SZ, seed + i) for i, b in enumerate(bufs)])
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=cache))
    eng.register_buffers(bufs)
    return mem, bufs, eng


ma, ba, A = make(100, 256 << 20)
mb, bb, B = make(200, 64 << 20)
pin = pd.PinnedHost(N * SZ)
hostbuf = pd.PinnedHost(N * SZ)
sa, sb, db = pd.Stream(priority=1), pd.Stream(priority=1), pd.Stream(priority=1)
pd.device_synchronize()


def gather_a():
    A.record_dirty([1, 2, 3, 4])  # 64 MiB STW delta
    A.at_final_stop(stream=sa)
    sa.synchronize()
    t = A.kernel_ms("delta")
    A.commit_epoch()
    return t


for _ in range(3):
    gather_a()
res = {"alone_ms": min(gather_a() for _ in range(5))}
for mode in ("ce_runs", "ce_d2h"):
    ts = []
    for r in range(4):
        if mode == "ce_runs":
            B.register_buffers(bb)
            B.register_image([pin.array[i * SZ:(i + 1) * SZ] for i in range(N)])
            B.precopy_direct(waves=1, stream=sb, drain_stream=db)  # returns after submitting the runs
        else:
            pd.check(pd.lib().pos_memcpy(hostbuf.ptr, mb.ptr, N * SZ, 2, int(db)))
        time.sleep(0.001)
        ts.append(gather_a())
        db.synchronize()
        sb.synchronize()
        if mode == "ce_runs":
            B.precopy_direct_result()
    res[mode + "_ms"] = min(ts)
print(res)
