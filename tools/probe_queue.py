"""Bisect the direct-queue stall: variants of one direct pre-copy, each
reporting whether the ship-queue watchdog fired and when the scan started."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_12079_b200 as pd  # noqa: E402


def run(name, nbuf, size, prio, one_alloc, prepare, app, big_scan=False):
    if one_alloc:
        mem = pd.DeviceMemory(nbuf * size)
        ptrs = [mem.ptr + i * size for i in range(nbuf)]
    else:
        mems = [pd.DeviceMemory(size) for _ in range(nbuf)]
        ptrs = [m.ptr for m in mems]
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=p, size=size) for i, p in enumerate(ptrs)]
    pd.fill_batch([(p, size, 10 + i) for i, p in enumerate(ptrs)])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=0))
    eng.register_buffers(bufs)
    pin = pd.PinnedHost(nbuf * size)
    eng.register_image([pin.array[i * size:(i + 1) * size] for i in range(nbuf)])
    s, d = pd.Stream(priority=prio), pd.Stream(priority=prio)
    a = pd.Stream() if app else None
    t0 = time.perf_counter()
    eng.precopy_direct(waves=1, stream=s, drain_stream=d)
    if prepare:
        eng.prepare_final_stop(stream=s)
    if a is not None:
        eng.event_record(2, a)
        eng.stream_wait_event(2, s)
    d.synchronize()
    s.synchronize()
    dt = time.perf_counter() - t0
    qs = (C.c_uint64 * 14)()
    pd.lib().pos_debug_ship_queue(eng.ctx, qs)
    err = qs[4]
    scan_late = (qs[13] - qs[10]) / 1e6 if qs[13] and qs[10] else -1
    print(f"{name:28s} wall {dt*1e3:8.1f} ms  watchdog {'FIRED' if err else 'ok   '}  scan start +{scan_late:.3f} ms "
          f"tail {qs[0]}", flush=True)
    try:
        eng.precopy_direct_result()
    except pd.SimError:
        pass
    eng.close()


os.environ.setdefault("POSDUMP_WATCHDOG_MS", "1000")
run("small test-like", 4, 300000, 0, False, False, False)
run("c1 sizes, separate allocs", 64, 16 << 20, 0, False, False, False)
run("c1 sizes, one alloc", 64, 16 << 20, 0, True, False, False)
run("c1 + prepare_final_stop", 64, 16 << 20, 0, True, True, False)
run("c1 + app wait", 64, 16 << 20, 0, True, False, True)
run("c1 prio 1", 64, 16 << 20, 1, True, False, False)
run("small prio 1", 4, 300000, 1, False, False, False)
run("16 buffers x 16 MiB", 16, 16 << 20, 0, True, False, False)
run("4 buffers x 16 MiB", 4, 16 << 20, 0, True, False, False)
