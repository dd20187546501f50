"""Parity at the BASELINE configs' full sizes (112 GB,
40 GB, 120 GB on one B200), against the C restatement of the reference.

The states are filled on the device with fill_bytes (rng.hpp:43-54, k_fill)
and the oracle regenerates any chunk at random access (or_fill_bytes_at), so
no host copy of the state is needed:
  * >= 4096 random chunk digests == crc32 of the oracle's chunk bytes
    (crc32.hpp:26-34), and 512 of those chunks byte-compared after download;
  * the FULL digest table folds (or_fold_digests) into every buffer's device
    whole-buffer CRC (O1's k_buffer_crc), and two whole buffers are
    CRC'd on the host from scratch;
  * an epoch of the workload's writes (c4: appends; c3/c5: the optimizer
    step) flags exactly the chunks the writes touch, and written chunks
    hash to the oracle's bytes of the overlaid writes.
"""
import os
import sys

import numpy as np
import pytest

import paper_2405_12079_b200 as pd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
CS = 65536


def chunk_bytes(orc, size, base_seed, writes, c):
    """Expected bytes of chunk c: the fill, then the epoch writes in order."""
    lo, hi = c * CS, min(size, (c + 1) * CS)
    out = np.empty(hi - lo, np.uint8)
    orc.or_fill_bytes_at(base_seed, lo, out.ctypes.data, out.size)
    for off, n, seed in writes:
        a, b = max(lo, off), min(hi, off + n)
        if a < b:
            tmp = np.empty(b - a, np.uint8)
            orc.or_fill_bytes_at(seed, a - off, tmp.ctypes.data, tmp.size)
            out[a - lo:b - lo] = tmp
    return out


@pytest.mark.parametrize("name", ["c4", "c5", "c3"])
def test_full_size_parity(orc, name):
    wl = bench.Workload(name)
    sizes = wl.sizes
    stride = [(n + 255) // 256 * 256 for n in sizes]
    offs = np.concatenate([[0], np.cumsum(stride)[:-1]]).astype(np.uint64)
    mem = pd.DeviceMemory(int(sum(stride)))
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + int(o), size=n) for i, (o, n) in enumerate(zip(offs, sizes))]
    seed = {b.handle: 5000 + b.handle for b in bufs}
    pd.fill_batch([(b.dev_ptr, b.size, seed[b.handle]) for b in bufs])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=CS, cache_capacity=64 << 20))
    eng.register_buffers(bufs)
    nch = np.array([(n + CS - 1) // CS for n in sizes], np.int64)
    base = np.concatenate([[0], np.cumsum(nch)[:-1]])
    total = int(nch.sum())
    assert eng.n_chunks == total

    def where(g):
        i = int(np.searchsorted(base, g, side="right") - 1)
        return i, int(g - base[i])

    def check_epoch(writes_by_buf, rng):
        eng.hash_chunks()
        eng.scan_dedup()
        dig = eng.digests()
        crcs, _ = eng.buffer_crcs()
        sample = rng.choice(total, 4096, replace=False)
        # the written chunks, if any, are all in the sample's pool
        wchunks = sorted({int(base[h - 1]) + c for h, ws in writes_by_buf.items()
                          for off, n, _ in ws for c in range(off // CS, (off + n - 1) // CS + 1)})
        pool = np.unique(np.concatenate([sample, np.array(wchunks[:4096], np.int64)]))
        for k, g in enumerate(pool):
            i, c = where(int(g))
            want = chunk_bytes(orc, sizes[i], seed[i + 1], writes_by_buf.get(i + 1, []), c)
            assert dig[g] == orc.or_crc32(want.ctypes.data, want.size), (i, c)
            if k % 8 == 0:  # 1/8 of them byte for byte
                got = mem.download(want.size, offset=int(offs[i]) + c * CS)
                assert np.array_equal(got, want), (i, c)
        for i, n in enumerate(sizes):  # the full table folds into every device buffer CRC
            d = np.ascontiguousarray(dig[base[i]:base[i] + nch[i]])
            assert orc.or_fold_digests(d.ctypes.data, n, CS) == crcs[i], i
        for i in (0, len(sizes) - 1):  # whole buffers on the host, from scratch
            full = np.empty(sizes[i], np.uint8)
            orc.or_fill_bytes(seed[i + 1], full.ctypes.data, full.size)
            for off, n, s in writes_by_buf.get(i + 1, []):
                tmp = np.empty(n, np.uint8)
                orc.or_fill_bytes(s, tmp.ctypes.data, n)
                full[off:off + n] = tmp
            assert orc.or_crc32(full.ctypes.data, full.size) == crcs[i], i
        return dig

    rng = np.random.default_rng(12345)
    d0 = check_epoch({}, rng)
    eng.commit_epoch()
    # one epoch of the workload's writes (the optimizer tail included)
    writes = list(wl.epoch_writes(1)) + [(h, 0, sizes[h - 1], s) for k in wl.window(1) for h, s in k]
    pd.fill_batch([(bufs[h - 1].dev_ptr + o, n, s) for h, o, n, s in writes])
    pd.device_synchronize()
    by_buf: dict = {}
    for h, o, n, s in writes:
        by_buf.setdefault(h, []).append((o, n, s))
    for h, ws in by_buf.items():  # a whole-buffer rewrite replaces the base fill
        if any(o == 0 and n == sizes[h - 1] for o, n, _ in ws):
            last = max(k for k, (o, n, _) in enumerate(ws) if o == 0 and n == sizes[h - 1])
            seed[h] = ws[last][2]
            by_buf[h] = ws[last + 1:]
    check_epoch(by_buf, rng)
    flags = eng.flags()
    want = np.zeros(total, bool)
    for h, o, n, _ in writes:
        want[int(base[h - 1]) + o // CS:int(base[h - 1]) + (o + n - 1) // CS + 1] = True
    assert np.array_equal(flags.astype(bool), want)
    eng.close()
    mem.close()
    del d0


def test_buffers_beyond_4gib(orc):
    """64-bit offsets everywhere (buffer.hpp sizes are uint64_t): two buffers
    larger than 4 GiB and a tiny one.  Chunk digests past the 4 GiB mark ==
    crc32 of the oracle's bytes, the digest table folds into each buffer's
    device CRC, a sparse epoch's direct pre-copy lands every written chunk
    at image + ci * chunk_size beyond 4 GiB, and the STW gather of a 5 GiB
    DAG-dirty buffer (a > 4 GiB delta pack) drains into the image intact."""
    G = 1 << 30
    sizes = [5 * G + 12345, 3, 4 * G + 2 * CS + 7]
    stride = [(n + 255) // 256 * 256 for n in sizes]
    offs = [0, stride[0], stride[0] + stride[1]]
    mem = pd.DeviceMemory(sum(stride))
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + o, size=n) for i, (o, n) in enumerate(zip(offs, sizes))]
    seeds = {1: 61, 2: 62, 3: 63}
    pd.fill_batch([(b.dev_ptr, b.size, seeds[b.handle]) for b in bufs])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=CS, cache_capacity=6 * G))
    eng.register_buffers(bufs)
    img = pd.PinnedHost(sum(stride), image=True)
    image = [img.array[o:o + n] for o, n in zip(offs, sizes)]
    eng.register_image(image)
    nch = [(n + CS - 1) // CS for n in sizes]
    base = [0, nch[0], nch[0] + nch[1]]
    s, d = pd.Stream(), pd.Stream()
    eng.precopy_direct(waves=2, stream=s, drain_stream=d)
    eng.precopy_direct_result()
    d.synchronize()
    dig = eng.digests()
    eng.scan_dedup()
    crcs, _ = eng.buffer_crcs()
    rng = np.random.default_rng(7)
    for i in (0, 2):
        hi = np.arange((4 * G) // CS - 2, nch[i])  # the chunks around and past 4 GiB, all of them
        for c in np.concatenate([hi, rng.choice(nch[i], 256, replace=False)]):
            want = chunk_bytes(orc, sizes[i], seeds[i + 1], [], int(c))
            assert dig[base[i] + c] == orc.or_crc32(want.ctypes.data, want.size), (i, c)
            if c % 64 == 0 or c == nch[i] - 1:
                assert np.array_equal(image[i][c * CS:c * CS + want.size], want), (i, c)
        dd = np.ascontiguousarray(dig[base[i]:base[i] + nch[i]])
        assert orc.or_fold_digests(dd.ctypes.data, sizes[i], CS) == crcs[i], i
    eng.commit_epoch()
    # epoch 1: sparse writes past 4 GiB in buffer 3; buffer 1 rewritten whole by the "window" (DAG-dirty)
    writes3 = [(4 * G + 100, 5000, 71), (4 * G + CS + 3, CS + 4, 72), (17 * CS, 9, 73)]  # the 2nd ends at the buffer end
    pd.fill_batch([(bufs[2].dev_ptr + o, n, sd) for o, n, sd in writes3])
    eng.record_dirty([1])
    pd.fill_batch([(bufs[0].dev_ptr, sizes[0], 81)])
    pd.device_synchronize()
    eng.precopy_direct(waves=2, stream=s, drain_stream=d)
    nship, _ = eng.precopy_direct_result()
    touched = sorted({c for o, n, _ in writes3 for c in range(o // CS, (o + n - 1) // CS + 1)})
    assert nship == len(touched)
    off, m = eng.at_final_stop(stream=s)
    assert m > 5 * G
    d.wait(s)
    eng.delta_drain(stream=d)
    d.synchronize()
    s.synchronize()
    for c in touched:
        want = chunk_bytes(orc, sizes[2], seeds[3], writes3, c)
        assert np.array_equal(image[2][c * CS:c * CS + want.size], want), c
    for c in list(range(0, nch[0], 997)) + [(4 * G) // CS, nch[0] - 1]:
        want = chunk_bytes(orc, sizes[0], 81, [], c)
        assert np.array_equal(image[0][c * CS:c * CS + want.size], want), c
    eng.close()
    img.close()
    mem.close()
