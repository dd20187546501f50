"""Host-link probe for the direct pre-copy's destination: pinned D2H into a
cudaHostAlloc buffer vs into the 120 GB huge-page image (pos_host_image_alloc),
single copies and a whole-image sweep in 16 MiB slices on 1 or 2 streams."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_12079_b200 as pd
from paper_2405_12079_b200.posdump import D2H
import bench

print("numa", bench.bind_numa_local(0), flush=True)
eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=64 << 20))
src = pd.DeviceMemory(1 << 30)
s1, s2 = pd.Stream(), pd.Stream()
res = {}
mc = pd.lib().pos_memcpy

def timed(fn, nbytes, streams=(s1,)):
    eng.event_record(0, s1)
    for s in streams[1:]:
        s.wait(s1)
    fn()
    for s in streams[1:]:
        s1.wait(s)
    eng.event_record(1, s1)
    return round(nbytes / (eng.event_elapsed(0, 1) * 1e-3) / 1e9, 2)

pin = pd.PinnedHost(256 << 20)
res["hostalloc_256M"] = max(timed(lambda: pd.check(mc(pin.ptr, src.ptr, 256 << 20, D2H, int(s1))), 256 << 20) for _ in range(5))
G = int(os.environ.get("IMG_GB", "120"))
img = pd.PinnedHost(G * 10**9, image=True)
for off_gb in (0, G // 2, G - 1):
    o = off_gb * 10**9
    res[f"image_256M_at_{off_gb}GB"] = max(timed(lambda: pd.check(mc(img.ptr + o, src.ptr, 256 << 20, D2H, int(s1))), 256 << 20) for _ in range(3))
S = 16 << 20
for gb in (4, G):
    n = gb * 10**9 // S * S
    def sweep(streams):
        k = 0
        for o in range(0, n, S):
            pd.check(mc(img.ptr + o, src.ptr + (o % (1 << 30)), S, D2H, int(streams[k % len(streams)])))
            k += 1
    res[f"image_sweep_{gb}GB_16M_1stream"] = timed(lambda: sweep((s1,)), n)
    res[f"image_sweep_{gb}GB_16M_2streams"] = timed(lambda: sweep((s1, s2)), n, (s1, s2))
    S2 = 64 << 20
    def sweep64():
        for o in range(0, n // S2 * S2, S2):
            pd.check(mc(img.ptr + o, src.ptr + (o % (1 << 30)), S2, D2H, int(s1)))
    res[f"image_sweep_{gb}GB_64M_1stream"] = timed(sweep64, n // S2 * S2)
    res[f"image_sweep_{gb}GB_16M_1stream_again"] = timed(lambda: sweep((s1,)), n)
    print(json.dumps(res), flush=True)
del img
# cudaHostAlloc'd destination at scale (the image is mmap + cudaHostRegister)
H = int(os.environ.get("HOSTALLOC_GB", "16"))
big = pd.PinnedHost(H * 10**9)
n = H * 10**9 // S * S
def sweep_h():
    for o in range(0, n, S):
        pd.check(mc(big.ptr + o, src.ptr + (o % (1 << 30)), S, D2H, int(s1)))
res[f"hostalloc_sweep_{H}GB_16M_1stream"] = timed(sweep_h, n)
res[f"hostalloc_sweep_{H}GB_16M_1stream_again"] = timed(sweep_h, n)
print(json.dumps(res), flush=True)
