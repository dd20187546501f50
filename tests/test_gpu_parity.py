"""GPU parity: every kernel of the dump path through the C ABI, against the
C restatement (oracle/) on the same seeded inputs.  Integer/byte work, so
every comparison is bit-exact.

Edge cases follow the reference: short tails (buffer.hpp:46-49), chunk_size
of any positive value (config.hpp:70-71), 1-byte buffers (buffer.hpp:109),
unknown handles / out-of-range writes (buffer.hpp:80-86), corrupt input.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2405_12079_b200 as pd
from oracle_ctypes import or_buffer_t

pytestmark = pytest.mark.gpu


def mb(orc, seed, n):
    out = np.empty(n, np.uint8)
    orc.or_fill_bytes(seed, out.ctypes.data, n)
    return out


def ocrc(orc, a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return orc.or_crc32(a.ctypes.data, a.nbytes)


def odigests(orc, a, cs):
    n = orc.or_chunk_count(a.size, cs)
    out = np.empty(n, np.uint32)
    orc.or_chunk_digests(a.ctypes.data, a.size, cs, out.ctypes.data)
    return out


def opack(orc, bufs, cs, flags, epoch=0, pflags=0):
    arr = (or_buffer_t * len(bufs))(*[or_buffer_t(h, a.ctypes.data, a.size) for h, a in bufs])
    n = orc.or_build_pack(arr, len(bufs), cs, flags.ctypes.data, epoch, pflags, None)
    out = np.empty(n, np.uint8)
    orc.or_build_pack(arr, len(bufs), cs, flags.ctypes.data, epoch, pflags, out.ctypes.data)
    return out


class Proc:
    """A set of device buffers with a host mirror (the oracle's view)."""

    def __init__(self, orc, sizes, seed0=100, handles=None, align=256, offsets=None):
        self.orc = orc
        self.sizes = list(sizes)
        self.handles = list(handles or range(1, len(sizes) + 1))
        offsets = offsets or [0] * len(sizes)
        self.mem = []
        self.bufs = []
        self.host = []
        for i, (n, off) in enumerate(zip(self.sizes, offsets)):
            m = pd.DeviceMemory(n + off + align)
            ptr = m.ptr + off
            self.mem.append(m)
            self.bufs.append(pd.GpuBuffer(handle=self.handles[i], dev_ptr=ptr, size=n))
            pd.fill_bytes(ptr, n, seed0 + i)
            self.host.append(mb(orc, seed0 + i, n))
        pd.device_synchronize()

    def write(self, i, off, n, seed):
        pd.fill_bytes(self.bufs[i].dev_ptr + off, n, seed)
        self.host[i][off:off + n] = mb(self.orc, seed, n)

    def read(self, i):
        b = self.bufs[i]
        out = np.empty(b.size, np.uint8)
        pd.check(pd.lib().pos_memcpy(out.ctypes.data, b.dev_ptr, b.size, 2, None))
        pd.device_synchronize()
        return out

    def zero(self, i):
        b = self.bufs[i]
        pd.check(pd.lib().pos_memset(b.dev_ptr, 0, b.size, None))


def download_cache(eng, offset, n):
    pin = pd.PinnedHost(n)
    eng.d2h_async(pin.ptr, offset, n, slice_bytes=1 << 16)
    pd.device_synchronize()
    out = pin.array.copy()
    pin.close()
    return out


# ---------------------------------------------------------------------------

def test_device_fill_matches_fill_bytes(orc):
    for n, off in [(1, 0), (7, 3), (16, 0), (17, 1), (1000, 5), (65536 + 9, 0)]:
        m = pd.DeviceMemory(n + off + 16)
        pd.fill_bytes(m.ptr + off, n, 12345 + n)
        pd.device_synchronize()
        assert np.array_equal(m.download(n, off), mb(orc, 12345 + n, n))


@pytest.mark.parametrize("n", [1, 2, 15, 16, 17, 100, 511, 512, 513, 4095, 4096, 65535, 65536,
                               65537, 1 << 20, (3 << 20) + 7])
def test_crc32_device_matches_reference(orc, n):
    m = pd.DeviceMemory(n + 64)
    pd.fill_bytes(m.ptr, n + 64, 7 + n)
    pd.device_synchronize()
    host = mb(orc, 7 + n, n + 64)
    for off in (0, 1, 3, 8, 15):
        assert pd.crc32(m.ptr + off, n) == ocrc(orc, host[off:off + n]), (n, off)


def test_crc32_known_vector_and_update(orc):  # test_memory.cpp:10-17
    m = pd.DeviceMemory(16)
    m.upload(np.frombuffer(b"123456789", np.uint8))
    assert pd.crc32(m.ptr, 9) == 0xCBF43926
    c = pd.crc32_update(0, m.ptr, 4)
    c = pd.crc32_update(c, m.ptr + 4, 5)
    assert c == 0xCBF43926
    assert pd.crc32(m.ptr, 0) == 0


@pytest.mark.parametrize("cs", [4096, 65536, 1000, 7, 16, 65537, 1 << 20])
def test_chunk_digests_and_epoch_bitmap(orc, cs):
    sizes = [3 * cs, 10000, 1, 2 * cs + 5, 70001]
    p = Proc(orc, sizes)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=8 << 20))
    eng.register_buffers(p.bufs)
    eng.hash_chunks()
    want = np.concatenate([odigests(orc, h, cs) for h in p.host])
    assert np.array_equal(eng.digests(), want)
    assert eng.flags().all()  # fresh epoch: everything ships
    eng.commit_epoch()
    # epoch 1: rewrite a few ranges (straddling chunk boundaries, and one no-op)
    p.write(0, cs - 3, 10, 999)
    p.write(3, 2 * cs, 5, 998)
    p.write(4, 0, 1, 997)
    pd.device_synchronize()
    prev = want
    eng.hash_chunks()
    cur = np.concatenate([odigests(orc, h, cs) for h in p.host])
    assert np.array_equal(eng.digests(), cur)
    oflags = np.zeros(cur.size, np.uint8)
    orc.or_dirty_flags(prev.ctypes.data, cur.ctypes.data, cur.size, 1, oflags.ctypes.data)
    assert np.array_equal(eng.flags(), oflags)
    bm = np.zeros((cur.size + 31) // 32, np.uint32)
    orc.or_pack_bitmap(oflags.ctypes.data, cur.size, bm.ctypes.data)
    assert np.array_equal(eng.bitmap(), bm)
    eng.close()


def _digest_layout(kind):
    rng = np.random.default_rng(hash(kind) & 0xFFFF)
    if kind == "tiny512":      # 1-6 warp steps per chunk
        return 512, [int(x) for x in rng.integers(1, 3000, 200)]
    if kind == "mixed64k":     # ResNet-like mix: scalars, tails, multi-chunk buffers
        return 65536, [int(x) for x in rng.integers(1, 4 << 20, 40)] + [1, 4, 65536, 65537, 3 * 65536]
    if kind == "big1m":        # 1 MiB chunks: few chunks, segmented over warps
        return 1 << 20, [4 << 20, (1 << 20) + 3, 7, (3 << 20) - 100, 2 << 20]
    if kind == "many4k":       # one 64 MiB buffer of 4 KiB chunks: many rounds per warp
        return 4096, [64 << 20]
    if kind == "sparse2k":     # 2 KiB chunks over 300 small buffers
        return 2048, [int(x) for x in rng.integers(1, 5000, 300)]
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["tiny512", "mixed64k", "big1m", "many4k", "sparse2k"])
def test_chunk_digest_layouts(orc, kind):
    """The O2 hash gives the reference's chunk digests (chunk_digests,
    buffer.hpp:117-128) for chunk/buffer layouts from 1-step chunks over
    hundreds of buffers to 1 MiB chunks (segmented across warps), epoch after
    epoch."""
    cs, sizes = _digest_layout(kind)
    p = Proc(orc, sizes)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20))
    eng.register_buffers(p.bufs)
    rng = np.random.default_rng(5)
    for epoch in range(3):
        if epoch:
            for _ in range(8):
                i = int(rng.integers(0, len(sizes)))
                off = int(rng.integers(0, sizes[i]))
                p.write(i, off, int(min(sizes[i] - off, rng.integers(1, 3 * cs))), 700 + epoch * 10 + i)
            pd.device_synchronize()
        eng.hash_chunks()
        want = np.concatenate([odigests(orc, h, cs) for h in p.host])
        got = eng.digests()
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (kind, epoch, bad[:10], got.size)
        eng.commit_epoch()
    eng.close()


@pytest.mark.parametrize("cs", [4096, 65536])
def test_unaligned_buffers(orc, cs):
    p = Proc(orc, [5000, 12345, 3, 3 * cs + 77], offsets=[1, 7, 13, 5])
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20))
    eng.register_buffers(p.bufs)
    n = eng.plan_precopy()
    want = np.concatenate([odigests(orc, h, cs) for h in p.host])
    assert np.array_equal(eng.digests(), want)
    pack = download_cache(eng, 0, n)
    flags = np.ones(want.size, np.uint8)
    assert np.array_equal(pack, opack(orc, list(zip(p.handles, p.host)), cs, flags))
    eng.close()


def test_buffer_crc_and_dedup_verdicts(orc):
    """scan_dedup (cr.hpp:416-425) + finalize_image gate (cr.hpp:720):
    clean -> ok, rewritten -> not ok, host touched -> not ok, no upstream ->
    absent, DAG-written -> not ok (mirrors test_cr.cpp:375-415)."""
    cs = 65536
    sizes = [65536, 100000, 65536 * 3, 4096, 777]
    p = Proc(orc, sizes, seed0=300)
    crcs = [ocrc(orc, h) for h in p.host]
    p.bufs[0].upstream = pd.Upstream(crcs[0], True)        # clean
    p.bufs[1].upstream = pd.Upstream(crcs[1], True)        # rewritten below
    p.bufs[2].upstream = pd.Upstream(crcs[2], False)       # host touched
    p.bufs[3].upstream = None                              # no provenance
    p.bufs[4].upstream = pd.Upstream(crcs[4], True)        # DAG-flagged
    p.write(1, 500, 3, 42)
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=8 << 20))
    eng.register_buffers(p.bufs)
    eng.record_dirty([5, 999])  # 999 is not in the snapshot: ignored (cr.hpp:904)
    eng.hash_chunks()
    eng.scan_dedup()
    got, ver = eng.buffer_crcs()
    assert [int(x) for x in got] == [ocrc(orc, h) for h in p.host]
    assert eng.dedup_verdicts() == {1: True, 2: False, 3: False, 5: False}
    for i, b in enumerate(p.bufs):
        want = orc.or_dedup_verdict(b.upstream is not None, ocrc(orc, p.host[i]),
                                    b.upstream.crc if b.upstream else 0,
                                    b.upstream.host_untouched if b.upstream else 0)
        assert bool(ver[i]) == (bool(want) and b.handle != 5)
    # dedup disabled (config.hpp:36): no verdict is ok
    eng2 = pd.DumpEngine(pd.SimConfig(chunk_size=cs, dedup=False, cache_capacity=8 << 20))
    eng2.register_buffers(p.bufs)
    eng2.hash_chunks()
    eng2.scan_dedup()
    assert not any(eng2.dedup_verdicts().values())
    eng.close()
    eng2.close()


@pytest.mark.parametrize("cs", [4096, 65536, 1000])
def test_compact_pack_is_bit_exact(orc, cs):
    """O3 pack == oracle pack for the eligible chunks: dirty, not dedup-ok,
    not DAG-dirty (chunk_copied abandons those, cr.hpp:487)."""
    sizes = [4 * cs, 3 * cs + 11, 17, 5 * cs, 9000]
    p = Proc(orc, sizes, seed0=500)
    crcs = [ocrc(orc, h) for h in p.host]
    p.bufs[2].upstream = pd.Upstream(crcs[2], True)  # dedup-ok: never packed
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=16 << 20))
    eng.register_buffers(p.bufs)
    eng.hash_chunks()
    eng.commit_epoch()
    rng = np.random.default_rng(cs)
    for i, n in enumerate(sizes):
        for _ in range(2):
            off = int(rng.integers(0, n))
            p.write(i, off, min(n - off, int(rng.integers(1, 300))), int(rng.integers(1, 1 << 40)))
    pd.device_synchronize()
    eng.record_dirty([4])
    prev = np.concatenate([odigests(orc, h, cs) for h in p.host])  # placeholder, recomputed below
    n = eng.plan_precopy(exclude_dag_dirty=True)
    cur = np.concatenate([odigests(orc, h, cs) for h in p.host])
    flags = eng.flags()
    # eligibility mask
    g = 0
    elig = flags.copy()
    for i, b in enumerate(p.bufs):
        nc = b.chunk_count(cs)
        if b.handle == 4 or (b.upstream is not None and ocrc(orc, p.host[i]) == b.upstream.crc):
            elig[g:g + nc] = 0
        g += nc
    want = opack(orc, list(zip(p.handles, p.host)), cs, elig, epoch=1)
    got = download_cache(eng, 0, n)
    assert n == want.size
    assert np.array_equal(got, want)
    assert np.array_equal(eng.digests(), cur)
    del prev
    eng.close()


@pytest.mark.parametrize("cs,offsets,window", [(4096, None, False), (65536, None, False),
                                                (65536, [0, 3, 0, 9], False), (65536, [0, 3, 0, 9], True)])
def test_delta_copy_pack_and_digests(orc, cs, offsets, window):
    """at_final_stop (cr.hpp:599-621): whole DAG-flagged buffers, after the
    pre-copy pack, ascending handle; digests refreshed from what was copied.
    window: the engine-delimited STW window (pos_final_stop)."""
    sizes = [3 * cs, 5000, 100, 2 * cs + 33]
    p = Proc(orc, sizes, seed0=700, handles=[2, 4, 6, 8], offsets=offsets)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=4 << 20))
    eng.register_buffers(p.bufs)
    n0 = eng.plan_precopy()
    eng.record_dirty([8, 4])
    p.write(1, 10, 4000, 31)   # the app writes while the pre-copy drains
    p.write(3, 0, 2 * cs, 32)
    pd.device_synchronize()
    assert eng.prepare_final_stop() == eng.prepare_final_stop()  # idempotent staging
    pd.device_synchronize()
    off, n1 = eng.at_final_stop(stw_begin_slot=3, stw_end_slot=4) if window else eng.at_final_stop()
    assert off == (n0 + 255) // 256 * 256
    if window:
        assert 0 < eng.event_elapsed(3, 4) == pytest.approx(eng.kernel_ms("delta"))
    got = download_cache(eng, off, n1)
    g_flags = np.concatenate([np.full(b.chunk_count(cs), b.handle in (4, 8), np.uint8) for b in p.bufs])
    want = opack(orc, list(zip(p.handles, p.host)), cs, g_flags, epoch=0, pflags=1)
    assert np.array_equal(got, want)
    cur = np.concatenate([odigests(orc, h, cs) for h in p.host])
    assert np.array_equal(eng.digests()[g_flags == 1], cur[g_flags == 1])
    eng.close()


def test_final_stop_window_errors(orc):
    """pos_final_stop validates its event slots (InvalidArgument) before
    touching the delta; a valid window then works on the same engine."""
    cs = 4096
    p = Proc(orc, [3 * cs, 100], seed0=900)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20))
    eng.register_buffers(p.bufs)
    eng.plan_precopy()
    eng.record_dirty([1])
    for begin, end in [(3, 3), (3, -1), (1000, 4), (3, 1000)]:
        with pytest.raises(pd.SimError):
            eng.at_final_stop(stw_begin_slot=begin, stw_end_slot=end)
    off, n = eng.at_final_stop(stw_begin_slot=3, stw_end_slot=4)
    assert n > 0 and eng.event_elapsed(3, 4) > 0
    eng.close()


def test_scatter_restores_state(orc):
    """materialize/load_complete (cr.hpp:1026-1084): packs applied in order
    reproduce the buffers."""
    cs = 4096
    sizes = [3 * cs, 5000, 1, 2 * cs + 100]
    p = Proc(orc, sizes, seed0=900)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=4 << 20))
    eng.register_buffers(p.bufs)
    n = eng.plan_precopy()
    full = download_cache(eng, 0, n)
    eng.commit_epoch()
    p.write(3, cs + 7, 20, 5)
    p.write(0, 0, 1, 6)
    pd.device_synchronize()
    n2 = eng.plan_precopy()
    delta = download_cache(eng, 0, n2)
    assert n2 < n
    for i in range(len(sizes)):
        p.zero(i)
    for pack in (full, delta):
        dev = pd.DeviceMemory(pack.size)
        dev.upload(pack)
        eng.materialize(dev.ptr, pack.size)
    pd.device_synchronize()
    for i in range(len(sizes)):
        assert np.array_equal(p.read(i), p.host[i])
    # corrupt input
    bad = full.copy()
    bad[:4] = 0
    dev = pd.DeviceMemory(bad.size)
    dev.upload(bad)
    with pytest.raises(pd.CorruptImageError):
        eng.materialize(dev.ptr, bad.size)
    # entry for an unknown handle -> InvalidLocator (buffer.hpp:80)
    bad = full.copy()
    bad[64:72] = np.frombuffer(np.uint64(12345).tobytes(), np.uint8)
    dev.upload(bad)
    with pytest.raises(pd.SimError) as e:
        eng.materialize(dev.ptr, bad.size)
    assert e.value.errc == "InvalidLocator"
    eng.close()


def test_staging_exhausted(orc):
    cs = 4096
    p = Proc(orc, [64 * cs], seed0=11)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=16 * cs))
    eng.register_buffers(p.bufs)
    with pytest.raises(pd.SimError) as e:
        eng.plan_precopy()
    assert e.value.errc == "StagingExhausted"
    eng.close()


def test_host_image_end_to_end(orc, ref):
    """Epoch 0 full pack + epoch 1 pre-copy + STW delta applied to the host
    image reproduce the device state; the POSI bytes equal the reference's
    write_image over the same Inline contents."""
    from oracle_ctypes import ref_image  # noqa: F401
    cs = 65536
    sizes = [1 << 20, 300000, 65536, 12345]
    p = Proc(orc, sizes, seed0=1200)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=8 << 20))
    eng.register_buffers(p.bufs)
    image = [np.zeros(n, np.uint8) for n in sizes]
    n = eng.plan_precopy()
    pd.apply_pack_host(download_cache(eng, 0, n), p.handles, image)
    eng.commit_epoch()
    p.write(0, 3 * cs + 5, 100, 77)
    p.write(1, 0, 10, 78)
    pd.device_synchronize()
    eng.record_dirty([3])
    n = eng.plan_precopy()
    pd.apply_pack_host(download_cache(eng, 0, n), p.handles, image)
    p.write(2, 100, 100, 79)
    pd.device_synchronize()
    off, n2 = eng.at_final_stop()
    pd.apply_pack_host(download_cache(eng, off, n2), p.handles, image)
    for i in range(len(sizes)):
        assert np.array_equal(image[i], p.host[i])
    img = pd.CheckpointImage()
    img.gpu_records = [pd.GpuBufferRec(h, 0, inline_bytes=image[i]) for i, h in enumerate(p.handles)]
    img.allocs = [(h, 0x7000_0000_0000 + 0x100000 * i, sizes[i]) for i, h in enumerate(p.handles)]
    ours = pd.write_image(img)
    # reference writer over the oracle's view of the device
    from oracle_ctypes import Rec, Alloc
    recs = (Rec * 4)()
    for i, h in enumerate(p.handles):
        recs[i].handle, recs[i].kind = h, 0
        recs[i].inline_bytes, recs[i].inline_len = p.host[i].ctypes.data, sizes[i]
    allocs = (Alloc * 4)(*[Alloc(*a) for a in img.allocs])
    args = [4096, None, 0, recs, 4, allocs, 4, None, 0, 0, 1, 0x7000_0000_0000, None, 0]
    nref = ref.ref_write_image(*args, None, 0)
    out = np.empty(nref, np.uint8)
    ref.ref_write_image(*args, out.ctypes.data, nref)
    assert ours == out.tobytes()
    eng.close()


@pytest.mark.slow
def test_c1_full_size_properties(orc):
    """BASELINE config 1 at full size (1 GiB, 64 x 16 MiB, 64 KiB chunks):
    golden digests of buffers 0 and 63, fold == whole CRC for every buffer
    (checksum of checksums), 10% random rewrite -> exactly those chunks dirty,
    pack -> scatter into zeroed buffers -> digests identical."""
    import json
    import os
    kat = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kat.json")))
    cs, nb, size = 65536, 64, 16 << 20
    mem = pd.DeviceMemory(nb * size)
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * size, size=size) for i in range(nb)]
    pd.fill_batch([(b.dev_ptr, size, 1000 + i) for i, b in enumerate(bufs)])
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=512 << 20))
    eng.register_buffers(bufs)
    eng.hash_chunks()
    eng.scan_dedup()
    d = eng.digests().reshape(nb, 256)
    for k, g in kat["c1_buffers"].items():
        i = int(k)
        assert f"{d[i, 0]:08x}" == g["chunk0"] and f"{d[i, 255]:08x}" == g["chunk255"]
        assert f"{ocrc(orc, d[i].copy().view(np.uint8)):08x}" == g["digests_crc"]
    crcs, _ = eng.buffer_crcs()
    for i in range(nb):
        assert crcs[i] == orc.or_fold_digests(d[i].copy().ctypes.data, size, cs)
    assert f"{crcs[0]:08x}" == kat["c1_buffers"]["0"]["whole"]
    assert f"{crcs[63]:08x}" == kat["c1_buffers"]["63"]["whole"]
    eng.commit_epoch()
    rng = np.random.default_rng(1)
    dirty = rng.choice(nb * 256, 1638, replace=False)
    pd.fill_batch([(bufs[g // 256].dev_ptr + (g % 256) * cs, cs, orc.or_mix64(1, int(g))) for g in dirty])
    n = eng.plan_precopy()
    flags = eng.flags()
    assert set(np.nonzero(flags)[0]) == set(int(g) for g in dirty)
    assert n == (64 + 32 * 1638 + 255) // 256 * 256 + 1638 * cs
    before = eng.digests().copy()
    cache_ptr, _ = eng.cache()
    # zero the dirty chunks, scatter the pack back, re-hash: identical digests
    for g in dirty:
        pd.check(pd.lib().pos_memset(bufs[g // 256].dev_ptr + (g % 256) * cs, 0, cs, None))
    pack = pd.DeviceMemory(n)
    pd.check(pd.lib().pos_memcpy(pack.ptr, cache_ptr, n, 3, None))
    eng.materialize(pack.ptr, n)
    eng.hash_chunks()
    assert np.array_equal(eng.digests(), before)
    eng.close()


@pytest.mark.parametrize("waves", [1, 3, 16])
def test_pipelined_precopy_matches_single_pack(orc, waves):
    """Wave-pipelined pre-copy: per-wave packs, chained in the cache and copied
    to the same host offsets, carry exactly the single pack's entries and
    payload; digests/flags/bitmap identical."""
    cs = 65536
    sizes = [3 * cs, 10000, 1, 2 * cs + 5, 70001, 5 * cs, 300, cs]
    p = Proc(orc, sizes, seed0=4000)
    p.bufs[2].upstream = pd.Upstream(ocrc(orc, p.host[2]), True)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=32 << 20))
    eng.register_buffers(p.bufs)
    n = eng.plan_precopy()
    single = download_cache(eng, 0, n)
    eng.commit_epoch()
    p.write(0, 5, 100, 1)
    p.write(5, 2 * cs, cs, 2)
    p.write(7, cs - 1, 1, 3)
    pd.device_synchronize()
    n1 = eng.plan_precopy()
    one = download_cache(eng, 0, n1)
    d1, f1, b1 = eng.digests(), eng.flags(), eng.bitmap()
    # same epoch again, pipelined (digests identical -> same flags)
    host = pd.PinnedHost(16 << 20)
    copy = pd.Stream()
    packs = eng.precopy_pipelined(host.ptr, waves=waves, copy_stream=copy)
    copy.synchronize()
    pd.device_synchronize()
    assert np.array_equal(eng.digests(), d1) and np.array_equal(eng.flags(), f1)
    assert np.array_equal(eng.bitmap(), b1)
    assert 1 <= len(packs) <= waves
    ents = [pd.parse_pack(host.array[o:o + z]) for o, z in packs]
    ref = pd.parse_pack(one)
    for key in ("handle", "chunk", "len", "crc"):
        assert np.array_equal(np.concatenate([e[key] for e in ents]), ref[key])
    img = [np.zeros(n, np.uint8) for n in sizes]
    for o, z in packs:
        pd.apply_pack_host(host.array[o:o + z], p.handles, img)
    want = [np.zeros(n, np.uint8) for n in sizes]
    pd.apply_pack_host(one, p.handles, want)
    for a, b in zip(img, want):
        assert np.array_equal(a, b)
    # the STW delta lands after the last wave pack
    eng.record_dirty([4])
    off, m = eng.at_final_stop()
    assert off == (packs[-1][0] + packs[-1][1] + 255) // 256 * 256
    del single
    eng.close()


@pytest.mark.parametrize("profile,seed,mode,eager", [
    ("gpt2-infer-desk", 1, 3, False),    # inference: parameters H2D-loaded -> DedupRef records
    ("resnet-train-desk", 1, 3, False),  # training under DAG retention
    ("fuzz", 7, 3, False),
    ("fuzz", 8, 1, False),               # stop-the-world image
    ("ppo-train-desk", 2, 3, False),     # a Recompute record
    ("resnet-train-desk", 1, 3, True),   # eager delta capture: the same image
    ("ppo-train-desk", 2, 3, True),
])
def test_reference_engine_image_is_reproduced(orc, ref, profile, seed, mode, eager):
    """Drop-in parity at engine level (P3 + P4): the reference CrEngine
    checkpoints a trace (checkpoint_at's flow, scenario.hpp:63-78); the
    device state at its cut is loaded onto the GPU with the session's
    provenance and DAG decisions (dirty_set_, recompute eligibility, final
    stop re-copies).  OUR path then does the rest: O2 + O1 verdicts on the
    device, the direct pre-copy into a pinned image, the STW delta + drain,
    and pos_finalize_image picks every record kind from the device verdicts
    and writes the image -- byte for byte the reference's, with the same
    CrMetrics.  Nothing is read from the reference's output image except the
    host-side sections (host pages, DAG, meta)."""
    from oracle_ctypes import ref_session
    from posi import read_posi
    from test_finalize import host_side
    sess = ref_session(ref, profile, seed, mode)
    img = read_posi(sess["image"])
    mems, bufs = [], []
    for r in sess["bufs"]:
        m = pd.DeviceMemory(r["size"])
        m.upload(np.frombuffer(r["content"], np.uint8))
        b = pd.GpuBuffer(handle=r["handle"], dev_ptr=m.ptr, size=r["size"])
        if r["has_upstream"]:  # note_h2d_provenance's record (process.hpp:505-522)
            b.upstream = pd.Upstream(r["up_crc"], r["host_untouched"])
        mems.append(m)
        bufs.append(b)
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=64 << 20))
    eng.register_buffers(bufs)
    image = [np.zeros(b.size, np.uint8) for b in bufs]
    eng.register_image(image)
    by_h = {r["handle"]: r for r in sess["bufs"]}
    # the DAG's view: buffers re-copied at the final stop are dirty during the
    # pre-copy; recompute-eligible dirty ones are dirty AND skipped by the stop
    recopy = [h for h, r in by_h.items() if r["final_recopy"]]
    recompute = [h for h, r in by_h.items() if r["dirty"] and r["recompute_eligible"]]
    eng.record_dirty(recopy + recompute)
    eng.set_stop_exclusions(recompute)
    s, d = pd.Stream(), pd.Stream()
    eng.precopy_direct(waves=2, stream=s, drain_stream=d)
    eng.precopy_direct_result()
    d.synchronize()
    if eager:  # every re-copied buffer already holds its bytes at the cut: captured before the stop
        eng.prepare_final_stop(stream=s)
        eng.pregather(recopy, stream=s)
    eng.at_final_stop(stream=s)
    d.wait(s)
    eng.delta_drain(stream=d)
    d.synchronize()
    s.synchronize()
    verdicts = eng.dedup_verdicts()
    for h, r in by_h.items():  # P3: the device O1 verdict == scan_dedup's (cr.hpp:416-445)
        if r["dedup_ok"] >= 0 and not r["dirty"]:
            assert verdicts[h] == (r["dedup_ok"] == 1), h
    fb = [pd.FinalizeBuf(handle=r["handle"], base=r["base"], size=r["size"], inline_bytes=a,
                         upstream=(r["up_host_addr"], r["up_len"], r["up_crc"]) if r["has_upstream"] else None,
                         dedup_ok=None, dirty=r["dirty"], recompute_eligible=r["recompute_eligible"],
                         recompute_nodes=r["pending"], precopy_survived=r["precopy_survived"])
          for r, a in zip(sess["bufs"], image)]
    out, m = pd.finalize_image(host_side(img), fb, engine=eng)
    assert out == sess["image"]
    want = sess["metrics"]
    for k in ("bytes_precopy", "bytes_dirty", "bytes_dedup_saved", "bytes_recompute_saved", "image_bytes",
              "image_file_bytes"):
        assert m[k] == want[k], k
    assert eng.metrics()["image_file_bytes"] == len(out)
    if mode == 3:  # closure identity (tests/test_harness.cpp:99-112)
        assert m["bytes_precopy"] + m["bytes_dirty"] + m["bytes_dedup_saved"] == sum(b.size for b in bufs)
    eng.close()


@pytest.mark.parametrize("region,peer_slots", [(300_000, 0), (1 << 20, 0), (300_000, 1), (300_000, 3)])
def test_cache_cycled_precopy(orc, region, peer_slots):
    """States larger than the O3 cache (BASELINE configs 3/5): waves cycle two
    cache regions; the packs handed to the sink carry exactly the single-pack
    entries/payload, and verdicts of buffers spanning waves still apply."""
    cs = 65536
    sizes = [3 * cs, 10000, 1, 2 * cs + 5, 70001, 5 * cs, 300, cs, 9 * cs + 7]
    p = Proc(orc, sizes, seed0=4500)
    p.bufs[1].upstream = pd.Upstream(ocrc(orc, p.host[1]), True)  # dedup-ok
    p.bufs[8].upstream = pd.Upstream(ocrc(orc, p.host[8]), True)  # dedup-ok, spans waves
    big = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=64 << 20))
    big.register_buffers(p.bufs)
    one = download_cache(big, 0, big.plan_precopy())
    big.close()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=2 * region + 4096))
    eng.register_buffers(p.bufs)
    if peer_slots:  # peer-GPU cache (config 5); the peer is this device on a 1-GPU box
        eng.attach_peer_cache(pd.device_count() - 1, peer_slots * (region // 256 * 256))
    got = []
    s, c = pd.Stream(), pd.Stream()
    total, n = eng.precopy_stream(lambda arr, i: got.append((i, arr.copy())), region_bytes=region,
                                  stream=s, copy_stream=c)
    if peer_slots:
        cap, tot = eng.peer_cache_stats()
        assert cap > 0
    assert [i for i, _ in got] == list(range(n)) and n >= 2
    assert total == sum(a.size for _, a in got)
    ents = [pd.parse_pack(a) for _, a in got]
    ref = pd.parse_pack(one)
    # buffer 9 spans waves: its early chunks may ship before its verdict is known
    keep = [e["handle"] != 9 for e in ents]
    for key in ("handle", "chunk", "len", "crc"):
        a = np.concatenate([e[key][k] for e, k in zip(ents, keep)])
        assert np.array_equal(a, ref[key]), key
    img = [np.zeros(n_, np.uint8) for n_ in sizes]
    for _, a in got:
        pd.apply_pack_host(a, p.handles, img)
    for i in range(len(sizes)):
        if i not in (1, 8):
            assert np.array_equal(img[i], p.host[i])
    eng.close()


@pytest.mark.parametrize("pinned", [False, True])
def test_streaming_restore_with_delta_replay(orc, pinned):
    """Restore = base image packs, then the incremental packs in order
    (delta-restore), through two cache regions: the restored buffers equal
    the live state; a pack naming an unknown handle is rejected before
    anything is written (all or nothing)."""
    cs = 65536
    sizes = [3 * cs, 10000, 1, 2 * cs + 5, 70001, 5 * cs]
    p = Proc(orc, sizes, seed0=6000)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=2 * 400_000 + 4096))
    eng.register_buffers(p.bufs)
    packs = []
    eng.precopy_stream(lambda a, i: packs.append(a.copy()), region_bytes=400_000)
    eng.commit_epoch()
    for e in range(3):  # appends: new bytes at a moving frontier
        p.write(5, e * cs + 100, 5000, 700 + e)
        p.write(0, e * 1000, 10, 800 + e)
        pd.device_synchronize()
        eng.precopy_stream(lambda a, i: packs.append(a.copy()), region_bytes=400_000)
        eng.commit_epoch()
    # fresh device buffers for the restored process (same handles)
    q = Proc(orc, sizes, seed0=9999)
    for i in range(len(sizes)):
        q.zero(i)
    rest = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=2 * 400_000 + 4096))
    rest.register_buffers(q.bufs)
    hostpacks = packs
    if pinned:
        hostpacks = []
        keep = []
        for a in packs:
            h = pd.PinnedHost(a.size)
            h.array[:] = a
            keep.append(h)
            hostpacks.append(h.array)
    rest.restore_packs(hostpacks, region_bytes=400_000)
    for i in range(len(sizes)):
        assert np.array_equal(q.read(i), p.host[i]), i
    bad = packs[-1].copy()
    if pd.parse_pack(bad)["n_entries"]:
        bad[64:72] = np.frombuffer(np.uint64(424242).tobytes(), np.uint8)
        before = [q.read(i) for i in range(len(sizes))]
        with pytest.raises(pd.SimError) as e:
            rest.restore_packs([packs[0], bad], region_bytes=400_000)
        assert e.value.errc == "InvalidLocator"
        assert all(np.array_equal(q.read(i), b) for i, b in enumerate(before))
    eng.close()
    rest.close()


@pytest.mark.parametrize("cs,waves,offsets,pageable", [
    (65536, 1, None, False),
    (65536, 3, None, True),          # pageable image: pinned + mapped by the context
    (4096, 2, [0, 5, 0, 3], False),  # unaligned buffers: the copy engine's byte-granular runs
    (1000, 1, None, False),          # chunk_size not a multiple of 16
])
def test_direct_precopy_into_image(orc, cs, waves, offsets, pageable):
    """Direct mode (pos_precopy_direct + pos_delta_drain): every shipped chunk
    lands at its place in the registered host image (chunk_copied,
    cr.hpp:499-501) -- epoch 0 ships everything, epoch 1 exactly the dirty
    chunks outside dirty_set_ plus the STW delta of dirty_set_; the image then
    equals the device, untouched image bytes are never written, and the index
    packs carry the oracle pack's entries."""
    sizes = [1 << 20, 300000, 65536 + 7, 12345]
    p = Proc(orc, sizes, seed0=4100, offsets=offsets)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=16 << 20))
    eng.register_buffers(p.bufs)
    if pageable:
        image = [np.zeros(n, np.uint8) for n in sizes]
    else:
        pin = pd.PinnedHost(sum((n + 255) // 256 * 256 for n in sizes))
        pin.array[:] = 0
        image, o = [], 0
        for n in sizes:
            image.append(pin.array[o:o + n])
            o += (n + 255) // 256 * 256
    eng.register_image(image)
    ckpt, drain = pd.Stream(), pd.Stream()
    eng.precopy_direct(waves=waves, stream=ckpt, drain_stream=drain)
    drain.synchronize()
    ckpt.synchronize()
    nch, pay = eng.precopy_direct_result()
    assert nch == sum((n + cs - 1) // cs for n in sizes)
    for i in range(len(sizes)):
        assert np.array_equal(image[i], p.host[i]), f"epoch 0 buffer {i}"
    d0 = eng.digests()
    eng.commit_epoch()
    # epoch 1: sparse rewrites; buffer 3 is DAG-dirty (left to the STW delta)
    p.write(0, 3 * cs + 5, 100, 77)
    p.write(1, 0, 10, 78)
    p.write(3, 7, 20, 79)
    pd.device_synchronize()
    flags = np.concatenate([odigests(orc, h, cs) for h in p.host]) != d0
    marker = image[2].copy()
    eng.record_dirty([4])
    eng.precopy_direct(waves=waves, stream=ckpt, drain_stream=drain)
    p.write(3, 100, 50, 80)  # written during the pre-copy window
    pd.device_synchronize()
    off, n = eng.at_final_stop(stream=ckpt)
    eng.delta_drain(stream=drain)  # no host-side ordering: the drain waits for the gather itself
    drain.synchronize()
    ckpt.synchronize()
    nch, pay = eng.precopy_direct_result()
    bounds = np.cumsum([0] + [(s + cs - 1) // cs for s in sizes])
    want = flags.copy()
    want[bounds[3]:bounds[4]] = False  # DAG-dirty buffer: not in the pre-copy
    assert nch == int(want.sum())
    for i in range(len(sizes)):
        assert np.array_equal(image[i], p.host[i]), f"epoch 1 buffer {i}"
    assert np.array_equal(image[2], marker)
    # index pack (cache offset 0, first wave): POSD header with the direct
    # flag; one wave -> its entries are the oracle pack's entries byte for byte
    idx = download_cache(eng, 0, 64)
    assert idx[:4].tobytes() == b"POSD" and (int(idx[20:24].view(np.uint32)[0]) & 2)
    if waves == 1:
        ne = int(idx[16:20].view(np.uint32)[0])
        assert ne == nch
        ours = download_cache(eng, 0, 64 + 32 * ne)[64:]
        ref = opack(orc, list(zip(p.handles, p.host)), cs, want.astype(np.uint8), 1)
        assert np.array_equal(ours, ref[64:64 + 32 * ne])
    eng.close()


def test_direct_runs_never_span_allocations(orc):
    """Separately allocated buffers that sit back to back in device memory,
    imaged into one pinned range back to back: the copy-engine runs may not
    be merged across the buffer boundary (a copy may not span two
    allocations) -- the pre-copy and the delta drain still land every byte."""
    cs = 4096
    sizes = [3 * cs, 2 * cs, 4 * cs, cs]
    mems = [pd.DeviceMemory(n) for n in sizes]
    host = []
    for i, (m, n) in enumerate(zip(mems, sizes)):
        pd.fill_bytes(m.ptr, n, 600 + i)
        host.append(mb(orc, 600 + i, n))
    pd.device_synchronize()
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=m.ptr, size=n) for i, (m, n) in enumerate(zip(mems, sizes))]
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20))
    eng.register_buffers(bufs)
    pin = pd.PinnedHost(sum(sizes))
    pin.array[:] = 0
    image, o = [], 0
    for n in sizes:
        image.append(pin.array[o:o + n])
        o += n
    eng.register_image(image)
    s, d = pd.Stream(), pd.Stream()
    eng.record_dirty([3, 4])  # adjacent buffers through the delta drain too
    eng.precopy_direct(waves=1, stream=s, drain_stream=d)
    eng.at_final_stop(stream=s)
    d.wait(s)
    eng.delta_drain(stream=d)
    d.synchronize()
    s.synchronize()
    for i, (img, h) in enumerate(zip(image, host)):
        assert np.array_equal(img, h), f"buffer {i + 1}"
    eng.close()


@pytest.mark.parametrize("cs", [4096, 1000])
def test_buffer_set_changes_mid_session(orc, cs):
    """A buffer freed and another allocated between checkpoints (cr.hpp:301-306,
    709-716): pos_update_buffer_set keeps the surviving buffers incremental
    (only their changed chunks ship), the new buffer ships whole, the freed
    one is never read, and the image equals the device afterwards; a
    committed epoch makes the new buffer incremental too."""
    sizes = [3 * cs + 5, 5000, 100, 2 * cs + 33]
    p = Proc(orc, sizes, seed0=5100)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=4 << 20))
    eng.register_buffers(p.bufs)
    image = [np.zeros(n, np.uint8) for n in sizes]
    eng.register_image(image)
    ckpt, drain = pd.Stream(), pd.Stream()

    def precopy():
        eng.precopy_direct(waves=1, stream=ckpt, drain_stream=drain)
        drain.synchronize()
        ckpt.synchronize()
        return eng.precopy_direct_result()[0]

    assert precopy() == sum((n + cs - 1) // cs for n in sizes)
    d0 = eng.digests()
    eng.commit_epoch()
    # buffer 2 is freed, buffer 5 allocated; buffer 1 rewritten in one chunk
    p.write(0, cs + 3, 10, 501)
    new = pd.DeviceMemory(3 * cs + 256)
    pd.fill_bytes(new.ptr, 3 * cs, 502)
    pd.device_synchronize()
    new_host = mb(orc, 502, 3 * cs)
    keep = [0, 2, 3]
    bufs = [p.bufs[i] for i in keep] + [pd.GpuBuffer(handle=5, dev_ptr=new.ptr, size=3 * cs)]
    eng.update_buffer_set(bufs)
    # surviving buffers keep their digests (now the previous epoch's table)
    nc = [(n + cs - 1) // cs for n in sizes]
    base = np.cumsum([0] + nc)
    kept_prev = np.concatenate([d0[base[i]:base[i + 1]] for i in keep])
    assert eng.n_chunks == kept_prev.size + 3
    with pytest.raises(pd.SimError):  # the new buffer has no image range yet
        eng.precopy_direct(waves=1, stream=ckpt, drain_stream=drain)
    image2 = [image[i] for i in keep] + [np.zeros(3 * cs, np.uint8)]
    eng.register_image(image2)
    assert precopy() == 1 + 3  # the rewritten chunk + the new buffer
    hosts = [p.host[i] for i in keep] + [new_host]
    for i, img in enumerate(image2):
        assert np.array_equal(img, hosts[i]), f"buffer {bufs[i].handle}"
    want = np.concatenate([odigests(orc, h, cs) for h in hosts])
    assert np.array_equal(eng.digests(), want)
    eng.commit_epoch()
    assert precopy() == 0  # nothing changed: every buffer incremental now
    eng.commit_epoch()
    # a fresh target (CheckpointTarget::fresh, cr.hpp:35,396) gets everything,
    # the round after is incremental again
    for im in image2:
        im[:] = 0
    eng.set_target_fresh()
    assert precopy() == eng.n_chunks
    for i, img in enumerate(image2):
        assert np.array_equal(img, hosts[i])
    eng.commit_epoch()
    assert precopy() == 0
    eng.commit_epoch()
    # same handle, moved allocation (re-allocated between checkpoints): fresh
    moved = pd.DeviceMemory(3 * cs + 256)
    pd.fill_bytes(moved.ptr, 3 * cs, 502)  # same bytes, new address
    pd.device_synchronize()
    bufs2 = bufs[:3] + [pd.GpuBuffer(handle=5, dev_ptr=moved.ptr, size=3 * cs)]
    eng.update_buffer_set(bufs2)
    eng.register_image(image2)
    assert precopy() == 3  # its digests are unchanged, but it ships whole
    assert np.array_equal(image2[3], new_host)
    eng.close()


@pytest.mark.parametrize("cs", [4096, 1000])
def test_h2d_provenance_on_device(orc, cs):
    """note_h2d_provenance (process.hpp:505-522) on the device, after
    test_api.cpp:76-98: a whole-buffer H2D records Upstream::crc ==
    crc32(payload) -- lane-tree fold for buffers past 33 chunks, shuffle chain
    below -- and the next pre-copy dedups the buffer (O1, cr.hpp:416-425);
    a partial H2D drops the provenance; an address outside every buffer is a
    plain copy."""
    sizes = [cs * 1, cs * 2 + 1, cs * 33, cs * 34 - 5, cs * 100 + 17, 7]
    p = Proc(orc, sizes, seed0=5200)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=8 << 20))
    eng.register_buffers(p.bufs)
    s = pd.Stream()
    payloads = [mb(orc, 9000 + i, n) for i, n in enumerate(sizes)]
    for i, b in enumerate(p.bufs):
        eng.h2d_provenance(b.dev_ptr, payloads[i], stream=s)
        p.host[i][:] = payloads[i]
    s.synchronize()
    for i, b in enumerate(p.bufs):
        assert np.array_equal(p.read(i), payloads[i])
        assert eng.upstream(b.handle) == ocrc(orc, payloads[i]), f"buffer {i}"
    # O1 at the next pre-copy: every buffer dedups, the pack is empty
    n = eng.plan_precopy()
    crcs, ver = eng.buffer_crcs()
    assert [int(c) for c in crcs] == [ocrc(orc, h) for h in p.host]
    assert all(ver), ver
    assert n == 256  # header only: no entries, payload at the 256-B aligned offset
    # partial H2D into buffer 2 drops its provenance (process.hpp:510-513)
    part = mb(orc, 9100, 100)
    eng.h2d_provenance(p.bufs[2].dev_ptr + 5, part, stream=s)
    s.synchronize()
    assert eng.upstream(p.bufs[2].handle) is None
    eng.commit_epoch()
    eng.plan_precopy()
    _, ver = eng.buffer_crcs()
    assert not ver[2] and all(ver[i] for i in range(len(sizes)) if i != 2)
    eng.close()


def test_o1_verdicts_many_candidates(orc):
    """O1 with more provenance candidates (1500) than the scan's candidate
    list (1024 slots): the overflow walk must give the same verdicts
    (crc == Upstream::crc, cr.hpp:419-421) -- every other buffer carries a
    wrong crc."""
    n, size, cs = 1500, 100, 64
    mem = pd.DeviceMemory(n * 128)
    host = [mb(orc, 7000 + i, size) for i in range(n)]
    bufs = []
    for i in range(n):
        mem.upload(host[i], offset=i * 128)
        crc = ocrc(orc, host[i]) ^ (i & 1)
        bufs.append(pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * 128, size=size,
                                 upstream=pd.Upstream(crc, True)))
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=4 << 20))
    eng.register_buffers(bufs)
    s, d = pd.Stream(), pd.Stream()
    pin = pd.PinnedHost(n * 128)
    pin.array[:] = 0
    img = [pin.array[i * 128:i * 128 + size] for i in range(n)]
    eng.register_image(img)
    eng.precopy_direct(waves=1, stream=s, drain_stream=d)
    d.synchronize()
    s.synchronize()
    nch, _ = eng.precopy_direct_result()
    crcs, ver = eng.buffer_crcs()
    assert [int(c) for c in crcs] == [ocrc(orc, h) for h in host]
    assert [bool(v) for v in ver] == [i % 2 == 0 for i in range(n)]
    assert nch == (n // 2) * ((size + cs - 1) // cs)  # only the non-dedup buffers ship
    for i in range(n):
        want = host[i] if i % 2 else np.zeros(size, np.uint8)
        assert np.array_equal(img[i], want)
    eng.close()


@pytest.mark.parametrize("pinned", [True, False])
def test_ondemand_restore_from_image(orc, pinned):
    """On-demand restore (restore / start_loads / gate_restore, cr.hpp:167-204,
    1043-1143) of a flat host image: loads follow `order`, a gated buffer is
    resident before a kernel enqueued behind the gate reads it (the device
    waits on the buffer's ready event), and every buffer ends byte-exact."""
    sizes = [3 << 20, 1 << 20, 700001, 12345, 5 << 20]
    p = Proc(orc, sizes, seed0=6100)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=8 << 20))
    eng.register_buffers(p.bufs)
    if pinned:
        pin = pd.PinnedHost(sum((n + 255) // 256 * 256 for n in sizes))
        image, o = [], 0
        for h in p.host:
            image.append(pin.array[o:o + h.size])
            image[-1][:] = h
            o += (h.size + 255) // 256 * 256
    else:
        image = [h.copy() for h in p.host]
    for i in range(len(sizes)):
        p.zero(i)
    pd.device_synchronize()
    h2d, app = pd.Stream(), pd.Stream()
    eng.restore_image_begin(image, order=[5, 4, 3, 2, 1], slice_bytes=256 << 10, h2d_stream=h2d)
    # a "kernel" of the application touching buffer 1 (last in the load order)
    eng.restore_gate(1, stream=app)
    out = pd.DeviceMemory(sizes[0])
    pd.check(pd.lib().pos_memcpy(out.ptr, p.bufs[0].dev_ptr, sizes[0], 3, int(app)))
    app.synchronize()
    assert np.array_equal(out.download(), p.host[0])
    with pytest.raises(pd.SimError) as ei:
        eng.restore_want(99)
    assert ei.value.errc == "InvalidLocator"
    with pytest.raises(pd.SimError) as ei:  # the buffer set is pinned while the loader runs
        eng.update_buffer_set(p.bufs)
    assert ei.value.errc == "BadState"
    eng.restore_image_wait()
    for i in range(len(sizes)):
        assert np.array_equal(p.read(i), p.host[i]), f"buffer {i}"
    assert eng.restore_ready(1)  # no restore running: everything is ready
    eng.close()


@pytest.mark.parametrize("cs", [65536, 1000])
def test_cow_staging_keeps_prewrite_bytes(orc, cs):
    """CoW gate staging (stage_buffers, cr.hpp:858-888; after test_cr.cpp:
    106-127): a writer lands on buffer `a` before the epoch's pre-copy saved
    it; staging copies a's stop-point bytes into a staging pack, the kernel
    then overwrites the live buffer, and the checkpoint (pre-copy pack +
    staging pack) holds the pre-write payload while the other buffers ship
    normally.  The next epoch sees `a` as dirty against its staged digest.
    Staging more than the cache holds is StagingExhausted."""
    sizes = [1 << 20, 300001, 70000]
    p = Proc(orc, sizes, seed0=6600)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=3 << 20))
    eng.register_buffers(p.bufs)
    app = pd.Stream()
    snap = [h.copy() for h in p.host]
    off, n = eng.stage_buffers([1, 99], stream=app)  # unknown handle 99: not in the snapshot
    assert n > 0 and off + n <= 3 << 20
    # the kernel the gate let through, on the same (application) stream
    pd.fill_bytes(p.bufs[0].dev_ptr + 5, 4000, 4242, stream=app)
    p.host[0][5:4005] = mb(orc, 4242, 4000)
    pd.device_synchronize()
    m = eng.plan_precopy()
    image = [np.zeros(s, np.uint8) for s in sizes]
    pd.apply_pack_host(download_cache(eng, 0, m), p.handles, image)
    staged = download_cache(eng, off, n)
    assert int(staged[20:24].view(np.uint32)[0]) == 4  # staging pack flag
    pd.apply_pack_host(staged, p.handles, image)
    for i in range(len(sizes)):
        assert np.array_equal(image[i], snap[i]), f"buffer {i}"
    # the staging pack's entries carry the stop-point chunk crcs
    ent = pd.parse_pack(staged)
    assert list(ent["crc"]) == list(odigests(orc, snap[0], cs))
    eng.commit_epoch()
    # next epoch: `a` differs from its staged digest -> its written chunk ships
    m = eng.plan_precopy()
    ents = pd.parse_pack(download_cache(eng, 0, m))
    assert set(int(h) for h in ents["handle"]) == {1}
    assert set(int(c) for c in ents["chunk"]) == set(range(5 // cs, (5 + 4000 - 1) // cs + 1))
    eng.commit_epoch()
    eng.close()
    small = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20))
    small.register_buffers(p.bufs)
    assert small.stage_buffers([3], stream=app)[1] > 0  # 70 KB fits
    with pytest.raises(pd.SimError) as ei:
        small.stage_buffers([1], stream=app)  # 1 MiB + header does not
    assert ei.value.errc == "StagingExhausted"
    small.close()


_DRAIN_SCRIPT = r"""
import os, sys
import numpy as np
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import paper_2405_12079_b200 as pd
from oracle_ctypes import oracle
orc = oracle()
cs = 4096
sizes = [300000, 1 << 20, 12345, 70001]
mems, bufs, host = [], [], []
for i, n in enumerate(sizes):
    m = pd.DeviceMemory(n); pd.fill_bytes(m.ptr, n, 80 + i)
    h = np.empty(n, np.uint8); orc.or_fill_bytes(80 + i, h.ctypes.data, n)
    mems.append(m); host.append(h); bufs.append(pd.GpuBuffer(handle=i + 1, dev_ptr=m.ptr, size=n))
pd.device_synchronize()
eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=8 << 20))
eng.register_buffers(bufs)
pin = pd.PinnedHost(sum(sizes) + 1024); pin.array[:] = 0
img, o = [], 0
for n in sizes:
    img.append(pin.array[o:o + n]); o += (n + 255) // 256 * 256
eng.register_image(img)
s, d = pd.Stream(), pd.Stream()
for epoch in range(3):
    if epoch:
        for i, n in enumerate(sizes):
            off = (epoch * 7919 * (i + 1)) % n
            m = min(5000, n - off)
            pd.fill_bytes(bufs[i].dev_ptr + off, m, 900 + 10 * epoch + i)
            host[i][off:off + m] = 0
            t = np.empty(m, np.uint8); orc.or_fill_bytes(900 + 10 * epoch + i, t.ctypes.data, m); host[i][off:off + m] = t
        pd.device_synchronize()
        eng.record_dirty([3])
    eng.precopy_direct(waves=2, stream=s, drain_stream=d)
    eng.at_final_stop(stream=s); d.wait(s); eng.delta_drain(stream=d)
    d.synchronize(); s.synchronize()
    eng.precopy_direct_result()
    for i in range(len(sizes)):
        assert np.array_equal(img[i], host[i]), (epoch, i)
    eng.commit_epoch()
print("ok")
"""


def test_direct_precopy_fresh_process(tmp_path):
    """The direct pre-copy's first use in a fresh process (every kernel loaded
    at context creation: a lazily loaded kernel would wait for the copy
    engine) rebuilds the image byte for byte over three incremental epochs
    with a DAG-dirty buffer."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ROOT=root)
    r = subprocess.run([sys.executable, "-c", _DRAIN_SCRIPT], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_direct_tiled_scan_many_tiles(orc):
    """The tiled scan (decoupled look-back over ~200 CTAs) with 64-byte chunks
    over ~20 MB: index entries == the oracle pack's entries, the dirty bitmap
    == the digest comparison, the image == the device, across a fresh and an
    incremental epoch with provenance buffers and a DAG-dirty buffer."""
    rng = np.random.default_rng(11)
    cs = 64
    sizes = [int(x) for x in rng.integers(1, 900_000, 40)] + [1, 63, 64, 65]
    p = Proc(orc, sizes, seed0=8100)
    for i in (3, 17):  # dedup-ok provenance buffers
        p.bufs[i].upstream = pd.Upstream(ocrc(orc, p.host[i]), True)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=64 << 20))
    eng.register_buffers(p.bufs)
    pin = pd.PinnedHost(sum((n + 255) // 256 * 256 for n in sizes))
    pin.array[:] = 0
    img, o = [], 0
    for n in sizes:
        img.append(pin.array[o:o + n])
        o += (n + 255) // 256 * 256
    eng.register_image(img)
    s, d = pd.Stream(), pd.Stream()
    prev = None
    for epoch in range(2):
        if epoch:
            for i in rng.choice(len(sizes), 12, replace=False):
                n = sizes[i]
                off = int(rng.integers(0, n))
                m = int(min(n - off, rng.integers(1, 5000)))
                p.write(int(i), off, m, 7000 + int(i))
            pd.device_synchronize()
            eng.record_dirty([9])
        eng.precopy_direct(waves=1, stream=s, drain_stream=d)
        eng.at_final_stop(stream=s)
        d.wait(s)
        eng.delta_drain(stream=d)
        d.synchronize()
        s.synchronize()
        nch, _ = eng.precopy_direct_result()
        dig = np.concatenate([odigests(orc, h, cs) for h in p.host])
        assert np.array_equal(eng.digests(), dig)
        flags = np.ones(dig.size, bool) if prev is None else dig != prev
        bounds = np.cumsum([0] + [(n + cs - 1) // cs for n in sizes])
        bm = eng.bitmap()
        want_bm = np.zeros(bm.size, np.uint32)
        for g in np.nonzero(flags)[0]:
            want_bm[g >> 5] |= np.uint32(1 << (int(g) & 31))
        assert np.array_equal(bm, want_bm)
        elig = flags.copy()
        for i in (3, 17):
            elig[bounds[i]:bounds[i + 1]] = False  # O1: dedup
        if epoch:
            elig[bounds[8]:bounds[9]] = False  # DAG-dirty handle 9: the STW delta ships it
        assert nch == int(elig.sum())
        idx = download_cache(eng, 0, 64 + 32 * nch)
        ref = opack(orc, list(zip(p.handles, p.host)), cs, elig.astype(np.uint8), epoch)
        assert np.array_equal(idx[64:], ref[64:64 + 32 * nch])
        for i in range(len(sizes)):
            if i in (3, 17):
                continue  # dedup'd: the image keeps whatever the target had (DedupRef)
            assert np.array_equal(img[i], p.host[i]), f"epoch {epoch} buffer {i}"
        prev = dig
        eng.commit_epoch()
    eng.close()


@pytest.mark.parametrize("profile,seed,mode", [("gpt2-infer-desk", 1, 3), ("resnet-train-desk", 1, 3)])
def test_restore_from_reference_image(orc, ref, profile, seed, mode):
    """Restore from a POSI image the reference's CrEngine wrote (read_image +
    materialize, cr.hpp:1026-1030; dedup_content image.hpp:364-376): every
    Inline / DedupRef buffer lands byte for byte on the device, Recompute
    records are left to replay, and a corrupted copy of the image is rejected
    with the reference's offset before anything is written."""
    import ctypes as C
    from posi import dedup_bytes, read_posi
    n = ref.ref_checkpoint_image(profile.encode(), 0, seed, mode, None, 0)
    buf = C.create_string_buffer(n)
    ref.ref_checkpoint_image(profile.encode(), 0, seed, mode, buf, n)
    data = buf.raw[:n]
    img = read_posi(data)
    allocs = {h: size for h, base, size in img["meta"]["allocs"]}
    mems, bufs, want = [], [], {}
    for h in sorted(allocs):
        m = pd.DeviceMemory(allocs[h])
        pd.check(pd.lib().pos_memset(m.ptr, 0, allocs[h], None))
        mems.append(m)
        bufs.append(pd.GpuBuffer(handle=h, dev_ptr=m.ptr, size=allocs[h]))
    for r in img["recs"]:
        if r["kind"] == 0:
            want[r["handle"]] = r["inline"]
        elif r["kind"] == 1:
            want[r["handle"]] = dedup_bytes(img, r, allocs[r["handle"]])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=8 << 20))
    eng.register_buffers(bufs)
    # corrupt copy first: rejected with the reference's offset, nothing written
    bad = bytearray(data)
    bad[100] ^= 0x40  # inside the host pages / first records, before the (opaque) DAG
    wbad = np.frombuffer(bytes(bad), np.uint8)
    code = ref.ref_read_image_check(wbad.ctypes.data, wbad.size)
    if code:
        with pytest.raises(pd.CorruptImageError) as ei:
            eng.restore_image(bytes(bad))
        assert ei.value.offset == code - 1
        for m in mems:
            assert not m.download().any()
    loaded, recompute = eng.restore_image(data)
    assert loaded == len(want)
    assert recompute == sum(1 for r in img["recs"] if r["kind"] == 2)
    by_h = {b.handle: m for b, m in zip(bufs, mems)}
    for h, content in want.items():
        assert by_h[h].download().tobytes() == bytes(content), h
    eng.close()


# ---------------------------------------------------------------------------
# session-state hygiene (advisor round 1)

def test_reregister_clears_image_and_pending_state(orc):
    """register_image, then a new buffer set: the old image is gone, so a
    direct pre-copy is BAD_STATE until an image is registered again."""
    p = Proc(orc, [4096 * 3, 5000])
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=4096, cache_capacity=1 << 20))
    eng.register_buffers(p.bufs)
    eng.register_image([np.zeros(b.size, np.uint8) for b in p.bufs])
    eng.register_buffers(p.bufs)
    with pytest.raises(pd.SimError) as ei:
        eng.precopy_direct(waves=1)
    assert ei.value.errc == "BadState"
    img = [np.zeros(b.size, np.uint8) for b in p.bufs]
    eng.register_image(img)
    s, d = pd.Stream(), pd.Stream()
    eng.precopy_direct(waves=1, stream=s, drain_stream=d)
    eng.precopy_direct_result()
    d.synchronize()
    for a, h in zip(img, p.host):
        assert np.array_equal(a, h)
    eng.close()


def test_restore_begin_failure_leaves_no_loader(orc):
    """A rejected on-demand restore leaves the context usable (no half-built
    loader blocking buffer-set changes, no dangling gate)."""
    p = Proc(orc, [4096 * 2, 4096])
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=4096, cache_capacity=1 << 20))
    eng.register_buffers(p.bufs)
    bad = [np.zeros(p.bufs[0].size, np.uint8), np.zeros(p.bufs[1].size + 1, np.uint8)]
    with pytest.raises(pd.SimError) as ei:
        eng.restore_image_begin(bad)
    assert ei.value.errc == "InvalidArgument"
    eng.restore_gate(p.bufs[0].handle)  # no restore running: a no-op
    eng.register_buffers(p.bufs)        # not BAD_STATE
    good = [h.copy() for h in p.host]
    for i in range(2):
        p.zero(i)
    eng.restore_image_begin(good)
    eng.restore_image_wait()
    for i in range(2):
        assert np.array_equal(p.read(i), p.host[i])
    eng.close()


def test_scatter_rejects_misaligned_payloads(orc):
    """POSD payloads are 16-B padded by format; a pack whose payload offset or
    entry offset breaks that is CorruptImage, not a misaligned bulk copy."""
    cs = 4096
    p = Proc(orc, [cs * 2])
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20))
    eng.register_buffers(p.bufs)
    good = opack(orc, [(1, p.host[0])], cs, np.ones(2, np.uint8))
    for mutate in ("payload_off", "entry_off"):
        bad = good.copy()
        if mutate == "payload_off":
            v = bad[24:32].view(np.uint64)
            v[0] += 8
        else:  # second entry's payload offset
            v = bad[64 + 32 + 8:64 + 32 + 16].view(np.uint64)
            v[0] += 4
        dev = pd.DeviceMemory(bad.size)
        dev.upload(bad)
        with pytest.raises(pd.SimError) as ei:
            eng.materialize(dev.ptr, bad.size)
        assert ei.value.errc == "CorruptImage", mutate
        with pytest.raises(pd.SimError) as ei:
            eng.restore_packs([bad])
        assert ei.value.errc == "CorruptImage", mutate
    eng.close()


@pytest.mark.parametrize("trust", [True, False])
def test_buffer_level_o2_skip(orc, trust):
    """plan_precopy's O2 branch (cr.hpp:396-401) with trust_written_bit: in an
    incremental round a buffer with written_since_ckpt == 0 is neither hashed
    nor shipped (its digests carry over), even if its bytes changed behind
    the engine's back -- the bit is trusted, as the reference trusts it.
    finalize clears the bit (cr.hpp:745); a written buffer is hashed at chunk
    granularity.  Without trust every chunk is hashed (the CRC decides)."""
    cs = 4096
    p = Proc(orc, [cs * 8, cs * 8 + 100, cs * 3], seed0=7100)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20, trust_written_bit=trust))
    eng.register_buffers(p.bufs)
    eng.hash_chunks()
    d0 = eng.digests()
    eng.commit_epoch()                      # epoch 0 done: every written bit cleared
    p.write(0, cs * 2, cs, 7200)            # buffer 0: written and reported
    p.bufs[0].written_since_ckpt = True
    eng.update_buffer(p.bufs[0])
    p.write(1, cs * 5, 10, 7201)            # buffer 1: changed, NOT reported
    pd.device_synchronize()
    eng.hash_chunks()
    flags = eng.flags()
    dig = eng.digests()
    base1, base2 = 8, 8 + 9
    want0 = odigests(orc, p.host[0], cs)
    assert np.array_equal(dig[:8], want0) and list(np.nonzero(flags[:8])[0]) == [2]
    if trust:  # buffer 1 was not hashed: previous digests, nothing to ship
        assert np.array_equal(dig[base1:base2], d0[base1:base2]) and not flags[base1:base2].any()
    else:
        assert np.array_equal(dig[base1:base2], odigests(orc, p.host[1], cs))
        assert list(np.nonzero(flags[base1:base2])[0]) == [5]
    assert not flags[base2:].any()
    eng.commit_epoch()
    eng.hash_chunks()  # nothing written since: with trust, nothing hashed at all
    assert not eng.flags().any() or not trust
    eng.close()


@pytest.mark.parametrize("waves", [1, 2])
def test_direct_precopy_trust_written_bit(orc, waves):
    """The direct pre-copy (hash -> O1 -> tiled scan -> copy-engine runs) with
    the buffer-level O2 skip (cr.hpp:396-401): a clean
    buffer is neither hashed nor shipped even though its bytes changed, a
    written buffer ships exactly its changed chunks (short tails included)."""
    cs = 4096
    sizes = [cs * 40 + 100, cs * 33, cs * 5, cs * 70 + 7, cs]
    p = Proc(orc, sizes, seed0=7300)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=4 << 20, trust_written_bit=True))
    eng.register_buffers(p.bufs)
    pin = pd.PinnedHost(sum((n + 255) // 256 * 256 for n in sizes) + 256)
    pin.array[:] = 0
    image, o = [], 0
    for n in sizes:
        image.append(pin.array[o:o + n])
        o += (n + 255) // 256 * 256
    eng.register_image(image)
    ckpt, drain = pd.Stream(), pd.Stream()
    eng.precopy_direct(waves=waves, stream=ckpt, drain_stream=drain)
    drain.synchronize()
    ckpt.synchronize()
    eng.precopy_direct_result()
    for i in range(len(sizes)):
        assert np.array_equal(image[i], p.host[i])
    eng.commit_epoch()
    before = [im.copy() for im in image]
    p.write(0, cs * 2, cs * 3, 7400)      # buffer 0: chunks 2-4, reported
    p.write(0, cs * 40 - 50, 100, 7401)   # ... and its last two chunks (tail)
    p.bufs[0].written_since_ckpt = True
    eng.update_buffer(p.bufs[0])
    p.write(1, cs * 5, 10, 7402)          # buffer 1: changed, NOT reported
    p.write(3, cs * 69, cs + 7, 7403)     # buffer 3: reported, last two chunks
    p.bufs[3].written_since_ckpt = True
    eng.update_buffer(p.bufs[3])
    pd.device_synchronize()
    eng.precopy_direct(waves=waves, stream=ckpt, drain_stream=drain)
    drain.synchronize()
    ckpt.synchronize()
    nch, pay = eng.precopy_direct_result()
    assert nch == 3 + 2 + 2
    assert pay == 3 * cs + cs + 112 + cs + 16  # padded to 16 B in the index pack
    assert np.array_equal(image[0], p.host[0]) and np.array_equal(image[3], p.host[3])
    assert np.array_equal(image[1], before[1]) and not np.array_equal(image[1], p.host[1])
    assert np.array_equal(image[2], p.host[2]) and np.array_equal(image[4], p.host[4])
    eng.close()


@pytest.mark.parametrize("profile,seed,mode", [
    ("gpt2-infer-desk", 1, 3),    # DedupRef records, nothing pending
    ("resnet-train-desk", 1, 3),  # 35 retained kernels to replay
    ("fuzz", 7, 3),               # opaque + known kernels pending
    ("fuzz", 8, 1),               # stop-the-world image
    ("ppo-train-desk", 2, 3),     # a Recompute record, 591 kernels pending
])
def test_restore_state_parity(ref, profile, seed, mode):
    """P5: the state after OUR restore (pos_image_restore:
    Inline + DedupRef scattered onto device buffers, Recompute left to the
    replay) followed by the delta-restore replay of the image's pending
    kernels (replay_pending, cr.hpp:1099-1101; each kernel's effect =
    apply_kernel_effect, process.hpp:244-261: FNV-1a of name, seq and the
    read set's DEVICE bytes, then k_fill of every write with
    mix64(digest, h)) hashes (StateSnapshot::hash, process.hpp:76-89) to
    restore_state(img, Full) AND to plain_final_state(trace, cursor)
    (scenario.hpp:51-90)."""
    import ctypes as C
    from oracle_ctypes import ref_replay_plan
    from posi import read_posi
    n = ref.ref_checkpoint_image(profile.encode(), 0, seed, mode, None, 0)
    raw = C.create_string_buffer(n)
    ref.ref_checkpoint_image(profile.encode(), 0, seed, mode, raw, n)
    img_bytes = raw.raw[:n]
    im = read_posi(img_bytes)
    allocs = sorted(im["meta"]["allocs"])
    mems, bufs, dev = [], [], {}
    for h, base, size in allocs:
        m = pd.DeviceMemory(size)
        pd.check(pd.lib().pos_memset(m.ptr, 0, size, None))
        mems.append(m)
        bufs.append(pd.GpuBuffer(handle=h, dev_ptr=m.ptr, size=size))
        dev[h] = m
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=1 << 20))
    eng.register_buffers(bufs)
    loaded, recompute = eng.restore_image(img_bytes)
    kinds = [r["kind"] for r in im["recs"]]
    assert loaded == kinds.count(0) + kinds.count(1) and recompute == kinds.count(2)
    plan = ref_replay_plan(ref, img_bytes)
    assert all(p["kind"] in ("LaunchKnown", "LaunchOpaque") for p in plan)
    for p in plan:  # the application's replay of its pending kernels
        digest = ref.ref_fnv1a(p["name"], len(p["name"]), ref.ref_fnv1a_u64(p["seq"], 0xCBF29CE484222325))
        for h in sorted(p["reads"]):
            c = dev[h].download()
            digest = ref.ref_fnv1a_u64(h, digest)
            digest = ref.ref_fnv1a(c.ctypes.data, c.size, digest)
        pd.fill_batch([(dev[h].ptr, dev[h].nbytes, ref.ref_mix64(digest, h)) for h in sorted(p["writes"])])
        pd.device_synchronize()
    contents = [dev[h].download() for h, _, _ in allocs]
    handles = np.array([h for h, _, _ in allocs], np.uint64)
    bases = np.array([b for _, b, _ in allocs], np.uint64)
    sizes = np.array([s for _, _, s in allocs], np.uint64)
    cptrs = (C.c_void_p * max(len(allocs), 1))(*[c.ctypes.data for c in contents])
    pages = [np.frombuffer(b, np.uint8) for _, b in im["pages"]]
    pidx = np.array([i for i, _ in im["pages"]], np.uint64)
    pptrs = (C.c_void_p * max(len(pages), 1))(*[p.ctypes.data for p in pages])
    ours = ref.ref_snapshot_hash(len(allocs), handles.ctypes.data, bases.ctypes.data, sizes.ctypes.data, cptrs,
                                 len(pages), pidx.ctypes.data if pages else None, pptrs, im["page_size"])
    src = C.create_string_buffer(img_bytes, len(img_bytes))
    assert ours == ref.ref_restore_hash(src, len(img_bytes))
    assert ours == ref.ref_plain_hash(profile.encode(), 0, seed, im["meta"]["cursor"])
    eng.close()


def test_app_copy_overtakes_checkpoint_host_leg(orc):
    """CopyEngine priority (engines.hpp:153-159, test_engines.cpp:62-74): an
    application D2H issued during a direct pre-copy of 2 GB goes ahead of
    the checkpoint slices still to come -- it completes in a small fraction
    of the pre-copy (a plain copy on another stream waited for nearly all of
    it: tools/probe_app_copy.py) -- and both the application's bytes and
    the image are exact."""
    import time
    n, sz = 16, 125_000_000
    stride = (sz + 255) // 256 * 256
    mem = pd.DeviceMemory(n * stride)
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * stride, size=sz) for i in range(n)]
    pd.fill_batch([(b.dev_ptr, b.size, 8100 + b.handle) for b in bufs])
    app_dev = pd.DeviceMemory(16 << 20)
    pd.fill_bytes(app_dev.ptr, 16 << 20, 8200)
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=256 << 20))
    eng.register_buffers(bufs)
    img = pd.PinnedHost(n * stride, image=True)
    eng.register_image([img.array[i * stride:i * stride + sz] for i in range(n)])
    app_host = pd.PinnedHost(16 << 20)
    ckpt, drain, app = pd.Stream(priority=1), pd.Stream(priority=1), pd.Stream()
    eng.event_record(0, ckpt)
    eng.precopy_direct(waves=4, stream=ckpt, drain_stream=drain)
    time.sleep(0.005)
    eng.event_record(20, app)
    eng.app_copy(app_host.ptr, app_dev.ptr, 16 << 20, 2, stream=app)
    eng.event_record(21, app)
    eng.precopy_direct_result()
    eng.event_record(1, drain)
    drain.synchronize()
    app.synchronize()
    app_ms, pre_ms = eng.event_elapsed(20, 21), eng.event_elapsed(0, 1)
    assert pre_ms > 20 and app_ms < 0.25 * pre_ms, (app_ms, pre_ms)
    assert eng.host_leg_stats()[1] >= 1  # the leg yielded to it
    assert np.array_equal(app_host.array, mb(orc, 8200, 16 << 20))
    for i in (0, 7, n - 1):
        assert np.array_equal(img.array[i * stride:i * stride + sz], mb(orc, 8100 + i + 1, sz))
    eng.close()


def test_record_dirty_cancels_queued_host_leg_copies(orc):
    """record_dirty during the pre-copy cancels the buffer's copies still to
    be submitted (cr.hpp:909-918, CopyEngine::cancel): the last of 16 x 125 MB
    buffers, flagged while the host leg is still on the first ones, is not
    shipped by the pre-copy; the final stop re-copies it and the image is
    exact -- including the bytes an application kernel wrote meanwhile."""
    n, sz = 16, 125_000_000
    stride = (sz + 255) // 256 * 256
    mem = pd.DeviceMemory(n * stride)
    bufs = [pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + i * stride, size=sz) for i in range(n)]
    pd.fill_batch([(b.dev_ptr, b.size, 8300 + b.handle) for b in bufs])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=512 << 20))
    eng.register_buffers(bufs)
    img = pd.PinnedHost(n * stride, image=True)
    eng.register_image([img.array[i * stride:i * stride + sz] for i in range(n)])
    ckpt, drain, app = pd.Stream(priority=1), pd.Stream(priority=1), pd.Stream()
    eng.precopy_direct(waves=1, stream=ckpt, drain_stream=drain)
    eng.record_dirty([n])                      # the application's kernel on buffer n is submitted
    pd.fill_bytes(bufs[-1].dev_ptr, sz, 8400, stream=app)
    eng.event_record(2, app)
    eng.stream_wait_event(2, ckpt)             # drain the application
    eng.at_final_stop(stream=ckpt)             # waits for the pre-copy's last slice by itself
    drain.wait(ckpt)
    eng.delta_drain(stream=drain)
    eng.precopy_direct_result()
    drain.synchronize()
    ckpt.synchronize()
    _, _, cancelled = eng.host_leg_stats()
    assert cancelled >= sz // 2, cancelled
    assert np.array_equal(img.array[(n - 1) * stride:(n - 1) * stride + sz], mb(orc, 8400, sz))
    for i in (0, n - 2):
        assert np.array_equal(img.array[i * stride:i * stride + sz], mb(orc, 8300 + i + 1, sz))
    eng.close()


def test_ondemand_restore_recompute_handoff(orc):
    """The delta-restore hand-off (replay_pending / buffer_ready,
    cr.hpp:1099-1119) on the on-demand loader: buffer 2 is a Recompute record
    (not loaded); a reader gated on it waits -- on the host until its writer
    is enqueued (pos_restore_replayed), on the device until the writer ran --
    and sees the regenerated bytes; loaded buffers are exact; the restore
    cannot end while a Recompute buffer awaits its replay."""
    import threading
    import time
    cs = 65536
    p = Proc(orc, [cs * 40, cs * 30 + 7, cs * 20], seed0=8500)
    image = [h.copy() for h in p.host]
    for i in range(3):
        p.zero(i)
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20))
    eng.register_buffers(p.bufs)
    h2d, app, replay = pd.Stream(), pd.Stream(), pd.Stream()
    eng.restore_image_begin([image[0], None, image[2]], order=[3, 1], h2d_stream=h2d)
    scratch = pd.DeviceMemory(p.bufs[1].size)
    gated = threading.Event()

    def reader():  # a replayed kernel that reads buffer 2
        eng.restore_gate(2, stream=app)
        pd.check(pd.lib().pos_memcpy(scratch.ptr, p.bufs[1].dev_ptr, p.bufs[1].size, 3, int(app)))
        gated.set()

    t = threading.Thread(target=reader)
    t.start()
    time.sleep(0.2)
    assert not gated.is_set()  # buffer_ready(2) is false until its writer replays
    with pytest.raises(pd.SimError) as ei:
        eng.restore_image_wait()
    assert ei.value.errc == "BadState"
    pd.fill_bytes(p.bufs[1].dev_ptr, p.bufs[1].size, 8600, stream=replay)  # the writer, replayed
    eng.restore_replayed(2, stream=replay)
    t.join(10)
    assert gated.is_set()
    app.synchronize()
    eng.restore_image_wait()
    assert np.array_equal(scratch.download(), mb(orc, 8600, p.bufs[1].size))
    assert np.array_equal(p.read(0), image[0]) and np.array_equal(p.read(2), image[2])
    eng.close()


@pytest.mark.parametrize("offsets", [None, [0, 3, 0, 5, 0]])
def test_direct_host_leg_short_and_long_runs(orc, offsets):
    """The host leg's two engines in one pre-copy: runs of >= 4 MiB as
    copy-engine slices, shorter runs as k_ship_runs batches (more than
    kShipMaxRuns = 2048 runs per wave, so several batches; runs split between
    CTAs mid-run; unaligned buffers take the byte path).  Every shipped chunk
    lands in the image (chunk_copied, cr.hpp:499-501), clean chunks are never
    written."""
    cs = 4096
    sizes = [6 << 20, 24 << 20, 4 << 20, 9 << 20, 4097]
    p = Proc(orc, sizes, seed0=6100, offsets=offsets)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=64 << 20))
    eng.register_buffers(p.bufs)
    pin = pd.PinnedHost(sum((n + 255) // 256 * 256 for n in sizes))
    pin.array[:] = 0
    image, o = [], 0
    for n in sizes:
        image.append(pin.array[o:o + n])
        o += (n + 255) // 256 * 256
    eng.register_image(image)
    ckpt, drain = pd.Stream(), pd.Stream()
    eng.precopy_direct(waves=1, stream=ckpt, drain_stream=drain)
    drain.synchronize()
    ckpt.synchronize()
    eng.precopy_direct_result()
    for i in range(len(sizes)):
        assert np.array_equal(image[i], p.host[i]), f"epoch 0 buffer {i}"
    eng.commit_epoch()
    # epoch 1: buffer 0 wholly rewritten (one long run), buffer 1 every
    # other chunk (3072 one-chunk runs), buffer 3 random chunks, the tail
    # buffer's last byte
    p.write(0, 0, sizes[0], 91)
    for c in range(0, sizes[1] // cs, 2):
        p.write(1, c * cs + 17, 40, 1000 + c)
    rng = np.random.default_rng(5)
    for c in rng.choice(sizes[3] // cs, 300, replace=False):
        p.write(3, int(c) * cs, 8, 5000 + int(c))
    p.write(4, 4096, 1, 92)
    pd.device_synchronize()
    marker = [im.copy() for im in image]
    eng.precopy_direct(waves=1, stream=ckpt, drain_stream=drain)
    drain.synchronize()
    ckpt.synchronize()
    nch, pay = eng.precopy_direct_result()
    assert nch == sizes[0] // cs + sizes[1] // cs // 2 + 300 + 1
    for i in range(len(sizes)):
        assert np.array_equal(image[i], p.host[i]), f"epoch 1 buffer {i}"
    assert np.array_equal(image[2], marker[2])
    eng.close()


@pytest.mark.parametrize("cs,offsets", [(4096, None), (65536, [0, 3, 0, 9, 0])])
def test_delta_pregather_equals_stop_gather(orc, cs, offsets):
    """Eager delta capture (pos_delta_pregather): buffers gathered behind
    their last writer before the stop, one of them written again and
    re-recorded dirty (a later writer), the rest gathered at the stop -- the
    delta pack is byte-identical to the reference's at_final_stop re-copy of
    the final contents (cr.hpp:599-621), and the post-stop digests match."""
    sizes = [3 * cs, 5000, 100, 2 * cs + 33, 4 * cs]
    p = Proc(orc, sizes, seed0=7700, handles=[2, 4, 6, 8, 10], offsets=offsets)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=4 << 20))
    eng.register_buffers(p.bufs)
    n0 = eng.plan_precopy()
    dirty = [4, 8, 10]
    eng.record_dirty(dirty)
    eng.prepare_final_stop()
    ckpt = pd.Stream()
    # the window's writers on the application stream, each buffer captured behind its writer
    p.write(1, 10, 4000, 31)
    p.write(3, 0, 2 * cs, 32)
    eng.pregather([4, 8], after_stream=None, stream=ckpt)
    p.write(4, 7, 3 * cs, 33)
    eng.pregather([10], after_stream=None, stream=ckpt)
    # a later writer of buffer 8: re-recorded dirty -> gathered again at the stop
    p.write(3, 5, 100, 34)
    eng.record_dirty([8])
    eng.pregather([4], after_stream=None, stream=ckpt)  # already captured: no-op
    pd.device_synchronize()
    off, n1 = eng.at_final_stop(stream=ckpt, stw_begin_slot=3, stw_end_slot=4)
    ckpt.synchronize()
    assert off == (n0 + 255) // 256 * 256
    got = download_cache(eng, off, n1)
    g_flags = np.concatenate([np.full(b.chunk_count(cs), b.handle in dirty, np.uint8) for b in p.bufs])
    want = opack(orc, list(zip(p.handles, p.host)), cs, g_flags, epoch=0, pflags=1)
    assert np.array_equal(got, want)
    cur = np.concatenate([odigests(orc, h, cs) for h in p.host])
    assert np.array_equal(eng.digests()[g_flags == 1], cur[g_flags == 1])
    # the stop consumed the preparation: a new pregather needs a new one
    with pytest.raises(pd.SimError):
        eng.pregather([4], stream=ckpt)
    eng.close()


def test_empty_buffer_set_checkpoint(orc, ref):
    """A process with no live allocation (test_image.cpp:86-95's empty image):
    the pre-copy pack and the STW delta are header-only, the scatter of an
    empty pack is a no-op, and finalize writes the reference's 64-byte
    image."""
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=65536, cache_capacity=1 << 20))
    eng.register_buffers([])
    n = eng.plan_precopy()
    pack = download_cache(eng, 0, n)
    assert pack[:4].tobytes() == b"POSD" and int(pack[16:20].view(np.uint32)[0]) == 0
    eng.record_dirty([1, 2])  # handles outside the (empty) snapshot are ignored (cr.hpp:904)
    off, m = eng.at_final_stop()
    delta = download_cache(eng, off, m)
    assert int(delta[16:20].view(np.uint32)[0]) == 0
    dev = pd.DeviceMemory(max(n, 256))
    dev.upload(pack)
    eng.materialize(dev.ptr, n)
    pd.device_synchronize()
    out, metrics = pd.finalize_image(pd.CheckpointImage(page_size=4096), [], engine=eng)
    assert len(out) == 64 and out == pd.write_image(pd.CheckpointImage(page_size=4096))
    assert metrics["bytes_precopy"] == metrics["bytes_dirty"] == 0
    eng.close()


@pytest.mark.parametrize("trial", range(24))
def test_direct_checkpoint_random_sessions(orc, trial):
    """Randomised direct-mode sessions against the host mirror: chunk sizes
    (incl. not a multiple of 16), buffer sizes from 1 B to 12 MB at odd
    offsets, 1-4 waves, random sparse and whole-buffer writes, a random DAG
    dirty set (some written during the pre-copy, some pregathered), three
    epochs.  After every final stop + drain the image equals the device
    state, and image bytes between the buffers' ranges are never written
    (chunk_copied / at_final_stop, cr.hpp:447-621)."""
    rng = np.random.default_rng(1000 + trial)
    cs = int(rng.choice([1000, 4096, 16384, 65536]))
    nb = int(rng.integers(3, 12))
    sizes = [int(rng.choice([1, 17, cs - 1, cs, cs + 1, 3 * cs + 5])) if rng.random() < 0.4
             else int(rng.integers(1, 12 << 20)) for _ in range(nb)]
    offsets = [int(rng.integers(0, 16)) for _ in range(nb)]
    p = Proc(orc, sizes, seed0=20000 + 100 * trial, offsets=offsets)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=sum(sizes) + (64 << 20)))
    eng.register_buffers(p.bufs)
    gap = 64
    pin = pd.PinnedHost(sum(n + gap for n in sizes))
    pin.array[:] = 0xAB
    image, o = [], 0
    for n in sizes:
        image.append(pin.array[o:o + n])
        o += n + gap
    eng.register_image(image)
    ckpt, drain = pd.Stream(), pd.Stream()
    for epoch in range(3):
        if epoch:
            for _ in range(int(rng.integers(1, 3 * nb))):
                i = int(rng.integers(nb))
                off = int(rng.integers(sizes[i]))
                n = int(rng.integers(1, sizes[i] - off + 1))
                p.write(i, off, n, int(rng.integers(1 << 30)))
        pd.device_synchronize()
        dag = sorted({int(h) for h in rng.choice(p.handles, int(rng.integers(0, nb)), replace=False)})
        eng.record_dirty(dag)
        eng.precopy_direct(waves=int(rng.integers(1, 5)), stream=ckpt, drain_stream=drain)
        late = [h for h in dag if rng.random() < 0.5]  # written during the pre-copy window
        for h in late:
            i = p.handles.index(h)
            off = int(rng.integers(sizes[i]))
            p.write(i, off, int(rng.integers(1, sizes[i] - off + 1)), int(rng.integers(1 << 30)))
        pd.device_synchronize()
        eng.prepare_final_stop(stream=ckpt)
        early = [h for h in dag if h not in late and rng.random() < 0.5]
        if early:
            eng.pregather(early, stream=ckpt)
        eng.at_final_stop(stream=ckpt)
        eng.delta_drain(stream=drain)
        drain.synchronize()
        ckpt.synchronize()
        eng.precopy_direct_result()
        for i in range(nb):
            assert np.array_equal(image[i], p.host[i]), (trial, epoch, i, sizes[i], cs)
        o = 0
        for n in sizes:  # the gaps between image ranges: untouched
            assert np.all(pin.array[o + n:o + n + gap] == 0xAB), (trial, epoch)
            o += n + gap
        eng.commit_epoch()
        eng.clear_dirty()
    eng.close()


@pytest.mark.parametrize("trial", range(16))
def test_pack_and_delta_random_vs_oracle(orc, trial):
    """Randomised O2 + O3 + STW delta against the C oracle (P2 + P4): random
    chunk size, buffer sizes and offsets, sparse writes, a random DAG dirty
    set.  The pre-copy pack == the oracle's pack of the chunks whose digest
    changed outside the dirty set (bytes, entries, crcs); the dirty flags ==
    the oracle's digest compare; the delta pack == the oracle's pack of the
    dirty set's every chunk (at_final_stop)."""
    rng = np.random.default_rng(5000 + trial)
    cs = int(rng.choice([512, 1000, 4096, 65536]))
    nb = int(rng.integers(2, 10))
    sizes = [int(rng.integers(1, 2 << 20)) if rng.random() < 0.7 else int(rng.choice([1, cs, cs + 1, 7 * cs - 3]))
             for _ in range(nb)]
    handles = sorted(int(h) for h in rng.choice(np.arange(1, 1000), nb, replace=False))
    p = Proc(orc, sizes, seed0=30000 + 100 * trial, handles=handles,
             offsets=[int(rng.integers(0, 32)) * 16 for _ in range(nb)])
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=2 * sum(sizes) + (32 << 20)))
    eng.register_buffers(p.bufs)
    eng.hash_chunks()
    prev = np.concatenate([odigests(orc, h, cs) for h in p.host])
    assert np.array_equal(eng.digests(), prev)
    eng.commit_epoch()
    for _ in range(int(rng.integers(1, 4 * nb))):
        i = int(rng.integers(nb))
        off = int(rng.integers(sizes[i]))
        p.write(i, off, int(rng.integers(1, min(sizes[i] - off, 3 * cs) + 1)), int(rng.integers(1 << 40)))
    pd.device_synchronize()
    dag = sorted(int(h) for h in rng.choice(handles, int(rng.integers(0, nb)), replace=False))
    eng.record_dirty(dag)
    n = eng.plan_precopy(exclude_dag_dirty=True)
    cur = np.concatenate([odigests(orc, h, cs) for h in p.host])
    oflags = np.zeros(cur.size, np.uint8)
    orc.or_dirty_flags(prev.ctypes.data, cur.ctypes.data, cur.size, 1, oflags.ctypes.data)
    assert np.array_equal(eng.flags(), oflags)
    elig, g = oflags.copy(), 0
    for b in p.bufs:
        nc = b.chunk_count(cs)
        if b.handle in dag:
            elig[g:g + nc] = 0
        g += nc
    want = opack(orc, list(zip(p.handles, p.host)), cs, elig, epoch=1)
    assert n == want.size and np.array_equal(download_cache(eng, 0, n), want)
    off, m = eng.at_final_stop()
    dflags = np.concatenate([np.full(b.chunk_count(cs), b.handle in dag, np.uint8) for b in p.bufs])
    wantd = opack(orc, list(zip(p.handles, p.host)), cs, dflags, epoch=1, pflags=1)
    assert m == wantd.size and np.array_equal(download_cache(eng, off, m), wantd)
    # restore scatter (materialize, cr.hpp:1026-1084) of both packs onto zeroed
    # buffers: exactly the packed chunks come back, nothing else is written
    packs = [download_cache(eng, 0, n), download_cache(eng, off, m)]
    for i in range(nb):
        p.zero(i)
    dev = pd.DeviceMemory(max(n, m))
    for pk in packs:
        dev.upload(pk)
        eng.materialize(dev.ptr, pk.size)
        pd.device_synchronize()
    g = 0
    for i, b in enumerate(p.bufs):
        got, nc = p.read(i), b.chunk_count(cs)
        for c in range(nc):
            lo, hi = c * cs, min(sizes[i], (c + 1) * cs)
            shipped = elig[g + c] or dflags[g + c]
            assert np.array_equal(got[lo:hi], p.host[i][lo:hi] if shipped else np.zeros(hi - lo, np.uint8)), (i, c)
        g += nc
    eng.close()


def crc_null_change(orc, n, start):
    """A nonzero byte pattern E of length n (bits in bytes [start, start+8))
    with crc32(A ^ E) == crc32(A) for every A of length n: CRC-32 is affine
    in its input, so a GF(2) dependency among the CRC effects of 64 single
    bits is a change it cannot see."""
    zeros = np.zeros(n, np.uint8)
    z = orc.or_crc32(zeros.ctypes.data, n)
    basis = {}
    for i in range(64):
        e = zeros.copy()
        e[start + i // 8] ^= 1 << (i % 8)
        v, m = orc.or_crc32(e.ctypes.data, n) ^ z, 1 << i
        while v:
            h = v.bit_length() - 1
            if h not in basis:
                basis[h] = (v, m)
                break
            v, m = v ^ basis[h][0], m ^ basis[h][1]
        if v == 0:
            out = zeros.copy()
            for k in range(64):
                if m >> k & 1:
                    out[start + k // 8] ^= 1 << (k % 8)
            return out
    raise AssertionError("no dependency among 64 bits")


@pytest.mark.parametrize("d2", [False, True])
def test_o2_second_digest_catches_crc_preserving_change(orc, d2):
    """The chunk-level O2 compare's blind spot, and its guard: a change that
    leaves a chunk's CRC-32 unchanged (XOR of a multiple of the polynomial)
    is invisible to a CRC-32-only compare (the documented residual risk) and
    caught by the second digest (pos_set_o2_digest2).  The reported digest
    stays the reference's CRC-32 either way."""
    cs = 65536
    p = Proc(orc, [4 * cs, 3 * cs + 100], seed0=8800)
    E = crc_null_change(orc, cs, 1000)
    a = p.host[0][cs:2 * cs]
    assert E.any() and orc.or_crc32(a.ctypes.data, cs) == orc.or_crc32((a ^ E).ctypes.data, cs)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=1 << 20))
    eng.register_buffers(p.bufs)
    eng.set_o2_digest2(d2)
    eng.hash_chunks()
    d0 = eng.digests().copy()
    eng.commit_epoch()
    changed = a ^ E
    p.mem[0].upload(changed, offset=cs)
    p.host[0][cs:2 * cs] = changed
    pd.device_synchronize()
    eng.hash_chunks()
    assert np.array_equal(eng.digests(), d0)  # the CRC-32s did not move
    flags = eng.flags()
    want = np.zeros(d0.size, np.uint8)
    if d2:
        want[1] = 1
    assert np.array_equal(flags, want)
    eng.close()


@pytest.mark.parametrize("cs,offsets", [(65536, None), (4096, [0, 3, 0, 9, 5]), (1000, [0, 1, 2, 3, 4])])
def test_o2_second_digest_is_exact_on_ordinary_writes(orc, cs, offsets):
    """With the second digest on, the dirty flags of ordinary writes equal
    the CRC-32 compare's (the oracle's) across three epochs and varying wave
    counts, through the direct pre-copy into an image, at unaligned buffer
    starts and a chunk size that is not a multiple of 16, and a buffer-set
    change carries the second digests along."""
    sizes = [3 * cs + 7, 17, cs, 9 * cs, 5 * cs + 1]
    p = Proc(orc, sizes, seed0=8900, offsets=offsets)
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=cs, cache_capacity=16 << 20))
    eng.register_buffers(p.bufs)
    eng.set_o2_digest2(True)
    pin = pd.PinnedHost(sum(sizes))
    image, o = [], 0
    for n in sizes:
        image.append(pin.array[o:o + n])
        o += n
    eng.register_image(image)
    s, d = pd.Stream(), pd.Stream()
    rng = np.random.default_rng(cs)
    prev = None
    for epoch in range(3):
        if epoch:
            for _ in range(6):
                i = int(rng.integers(len(sizes)))
                off = int(rng.integers(sizes[i]))
                p.write(i, off, int(rng.integers(1, min(sizes[i] - off, 300) + 1)), int(rng.integers(1 << 30)))
            pd.device_synchronize()
        eng.precopy_direct(waves=int(rng.integers(1, 3)), stream=s, drain_stream=d)
        eng.precopy_direct_result()
        d.synchronize()
        cur = np.concatenate([odigests(orc, h, cs) for h in p.host])
        if prev is not None:
            oflags = np.zeros(cur.size, np.uint8)
            orc.or_dirty_flags(prev.ctypes.data, cur.ctypes.data, cur.size, 1, oflags.ctypes.data)
            assert np.array_equal(eng.flags(), oflags), epoch
        for i in range(len(sizes)):
            assert np.array_equal(image[i], p.host[i]), (epoch, i)
        prev = cur
        eng.commit_epoch()
    # a buffer-set change keeps the surviving buffers' digests (both kinds): nothing ships
    eng.update_buffer_set(p.bufs)
    eng.register_image(image)
    eng.precopy_direct(waves=1, stream=s, drain_stream=d)
    nch, _ = eng.precopy_direct_result()
    assert nch == 0
    eng.close()
