"""Which engine moves a c2-sized direct pre-copy: launch count and host-leg
stats around one pre-copy (k_ship_runs batches vs copy-engine slices)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_12079_b200 as pd
import bench

wl = bench.Workload("c2")
mem = pd.DeviceMemory(wl.total + 256 * len(wl.sizes))
bufs, off, offs = [], 0, []
for i, n in enumerate(wl.sizes):
    bufs.append(pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + off, size=n))
    offs.append(off)
    off += (n + 255) // 256 * 256
pd.fill_batch([(b.dev_ptr, b.size, 5000 + b.handle) for b in bufs])
eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=0))
eng.register_buffers(bufs)
pin = pd.PinnedHost(off, image=True)
eng.register_image([pin.array[o:o + b.size] for o, b in zip(offs, bufs)])
ckpt, drain = pd.Stream(), pd.Stream()
for e in range(3):
    l0 = eng.launches
    eng.precopy_direct(waves=16, stream=ckpt, drain_stream=drain)
    drain.synchronize(); ckpt.synchronize()
    n, pay = eng.precopy_direct_result()
    print(json.dumps({"epoch": e, "launches": eng.launches - l0, "chunks": n, "payload": pay,
                      "host_leg(slices, app_yields, cancelled)": eng.host_leg_stats(),
                      "max_size": max(wl.sizes), "n_bufs": len(wl.sizes)}))
    eng.set_target_fresh(True) if hasattr(eng, "set_target_fresh") else None
    eng.commit_epoch()
