"""Bisect: direct pre-copy of N x size buffers, W waves (one subprocess per case)."""
import os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def case(n, size, waves, variant=0):
    import numpy as np
    import paper_2405_12079_b200 as pd
    mem = pd.DeviceMemory(n * ((size + 255) // 256 * 256))
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * ((size + 255) // 256 * 256), size=size) for i in range(n)]
    pd.fill_batch([(b.dev_ptr, b.size, 5000 + b.handle) for b in bufs])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=0))
    eng.register_buffers(bufs)
    stride = (size + 255) // 256 * 256
    img = pd.PinnedHost(n * stride, image=True)
    eng.register_image([img.array[i * stride:i * stride + size] for i in range(n)])
    s, d = pd.Stream(priority=1), pd.Stream(priority=1)
    app = pd.Stream()
    if variant & 1:
        eng.record_dirty([n - k for k in range(8)])
    if variant & 2:
        import threading
        def run_app():
            for k in range(8):
                pd.fill_bytes(bufs[n - 1 - k].dev_ptr, size, 77 + k, stream=app)
            eng.event_record(2, app)
        th = threading.Thread(target=run_app)
        th.start()
    if variant & 4:
        eng.event_record(0, s)
    t = time.time()
    eng.precopy_direct(waves=waves, stream=s, drain_stream=d)
    nch, pay = eng.precopy_direct_result()
    d.synchronize()
    print(f"ok n={n} size={size} waves={waves} variant={variant} chunks={nch} {time.time()-t:.2f}s", flush=True)

if __name__ == "__main__":
    if len(sys.argv) > 1:
        case(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
        sys.exit(0)
    for n, size, w, v in [(60, 125_000_000, 1, 1), (60, 125_000_000, 1, 2), (60, 125_000_000, 1, 4),
                          (960, 125_000_000, 16, 1), (960, 125_000_000, 16, 3), (960, 125_000_000, 16, 7),
                          (64, 16 << 20, 4, 7)]:
        try:
            r = subprocess.run([sys.executable, __file__, str(n), str(size), str(w), str(v)], timeout=40,
                               capture_output=True, text=True, env=dict(os.environ, POSDUMP_TRACE="1"))
            print(r.stdout.strip() or f"FAIL n={n} size={size} w={w}: {r.stderr.strip()[-300:]}", flush=True)
        except subprocess.TimeoutExpired as ex:
            print(f"HANG n={n} size={size} waves={w} variant={v}: {(ex.stderr or b'')[-200:]}", flush=True)
