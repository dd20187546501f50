"""One wave of the config-5 direct pre-copy, standalone, for `ncu --set full`
(the bench's 120 GB state is too large for ncu's kernel replay to back up):
60 x 125 MB buffers (7.5 GB = one of the 16 waves), k_hash_chunks over
them exactly as a wave launches it (L2 flushed before each launch), then
the STW gather (k_copy_bulk) of 9 of them (1.125 GB, the bench's optimizer
tail) into the cache."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_12079_b200 as pd

N, SZ = 60, 125_000_000
stride = (SZ + 255) // 256 * 256
mem = pd.DeviceMemory(N * stride)
flush = pd.DeviceMemory(256 << 20)
bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * stride, size=SZ) for i in range(N)]
pd.fill_batch([(b.dev_ptr, b.size, 5000 + b.handle) for b in bufs])
pd.device_synchronize()
eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=2 << 30))
eng.register_buffers(bufs)
if "--digest2" in sys.argv:  # the O2 compare's second digest on
    eng.set_o2_digest2(True)
for i in range(4):
    pd.check(pd.lib().pos_memset(flush.ptr, i, flush.nbytes, None))
    pd.device_synchronize()
    eng.hash_chunks()
    pd.device_synchronize()
    print("hash ms", round(eng.kernel_ms("hash"), 4), "GB/s", round(N * SZ / eng.kernel_ms("hash") / 1e6, 1))
eng.commit_epoch()
eng.record_dirty(range(N - 8, N + 1))
for i in range(2):
    pd.check(pd.lib().pos_memset(flush.ptr, i, flush.nbytes, None))
    pd.device_synchronize()
    off, nb = eng.at_final_stop(stw_begin_slot=3, stw_end_slot=4)
    pd.device_synchronize()
    print("stw gather ms", round(eng.event_elapsed(3, 4), 4), "bytes", nb)
# restore-side scatter (materialize, cr.hpp:1026-1084) of that delta pack back
# into the buffers: k_pack_items + k_copy_bulk (the 3rd/4th k_copy_bulk launch)
cache_ptr, _ = eng.cache()
for i in range(2):
    pd.check(pd.lib().pos_memset(flush.ptr, i, flush.nbytes, None))
    pd.device_synchronize()
    eng.materialize(cache_ptr + off, nb)
    pd.device_synchronize()
    print("scatter ms", round(eng.kernel_ms("scatter"), 4), "GB/s (2x payload)",
          round(2 * 9 * SZ / eng.kernel_ms("scatter") / 1e6, 1))
eng.close()
