"""Direct-wave probe: hash time of the direct waves (k_hash_chunks<kModeDirect>)
and when the host leg starts, on a c5-like (125 MB buffers) and a c2-like
(224 x ~450 KB) state.  LIBPOSDUMP=<path> picks a library build."""
import os, sys, json, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_12079_b200 import _lib
if os.environ.get("LIBPOSDUMP"):
    _lib.LIB_PATH = os.environ["LIBPOSDUMP"]
import paper_2405_12079_b200 as pd

def run(name, sizes, waves, steps=5, hash_sms=0):
    total = sum((n + 255) // 256 * 256 for n in sizes)
    mem = pd.DeviceMemory(total)
    bufs, off = [], 0
    for i, n in enumerate(sizes):
        bufs.append(pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + off, size=n))
        off += (n + 255) // 256 * 256
    pd.fill_batch([(b.dev_ptr, b.size, 77 + b.handle) for b in bufs])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=1 << 30))
    eng.register_buffers(bufs)
    if hash_sms:
        eng.set_hash_sms(hash_sms)
    img = pd.PinnedHost(total, image=True)
    eng.register_image([img.array[o:o + b.size] for o, b in zip(
        [sum((n + 255) // 256 * 256 for n in sizes[:i]) for i in range(len(sizes))], bufs)])
    ckpt, drain = pd.Stream(priority=1), pd.Stream(priority=1)
    flush = pd.DeviceMemory(256 << 20)
    out = []
    for e in range(steps + 1):
        pd.fill_batch([(b.dev_ptr, b.size, 1000 * e + b.handle) for b in bufs])  # everything dirty
        pd.check(pd.lib().pos_memset(flush.ptr, e & 0xFF, flush.nbytes, None))
        pd.device_synchronize()
        eng.event_record(0, ckpt)
        eng.precopy_direct(waves=waves, stream=ckpt, drain_stream=drain)
        drain.synchronize(); ckpt.synchronize()
        eng.precopy_direct_result()
        tl = eng.timeline(0)
        if e:
            out.append({"hash_waves_ms": round(eng.kernel_ms("hash_waves"), 4), "d2h_start_ms": tl["d2h"][0],
                        "d2h_end_ms": tl["d2h"][1]})
        eng.commit_epoch()
    eng.close()
    med = {k: sorted(o[k] for o in out)[len(out) // 2] for k in out[0]}
    print(name, json.dumps(med), flush=True)

run("c5like_8GB_w1", [125_000_000] * 64, 1)
run("c5like_8GB_w4", [125_000_000] * 64, 4)
import json as _j
t = _j.load(open(os.path.join(ROOT, "tests", "golden", "c2_resnet_trace.json")))
run("c2like", t["sizes"], 1)
run("c2like_sms74", t["sizes"], 1, hash_sms=74)
run("c2like_sms37", t["sizes"], 1, hash_sms=37)
