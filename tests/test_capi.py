"""CPU: the C-ABI library loads, exports every symbol include/posdump.h
declares, maps errors onto the reference's Errc, refuses to run without a
device (no CPU fallback), and its host-side logic -- the streaming POSI writer
and the host pack applier -- is byte-identical to the reference / oracle."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2405_12079_b200 as pd
from paper_2405_12079_b200 import _lib
from oracle_ctypes import or_buffer_t

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BASE = 0x7000_0000_0000


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert lib.pos_abi_version() == 3


def test_error_codes_mirror_errc():
    lib = _lib.load()
    errc = ["PastTime", "Livelock", "OutOfDeviceMemory", "InvalidLocator", "UseAfterFree",
            "FreedBuffer", "BadState", "PendingKernels", "UnknownApi", "InvalidArgument",
            "CorruptDag", "CorruptImage", "InvariantViolation", "StagingExhausted", "OracleMismatch"]
    for i, name in enumerate(errc):  # errors.hpp:9-25 order
        assert lib.pos_strerror(i + 1).decode() == name
    assert lib.pos_strerror(0).decode() == "OK"


def test_no_cpu_fallback():
    if pd.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(pd.NoDeviceError):
        pd.DumpEngine(pd.SimConfig(chunk_size=4096))
    with pytest.raises(pd.NoDeviceError):
        pd.crc32(0x1000, 16)


def test_invalid_config_rejected_before_device():
    with pytest.raises(pd.SimError) as e:  # config.hpp:70-71
        pd.DumpEngine(pd.SimConfig(chunk_size=0))
    assert e.value.errc == "InvalidArgument"


def test_null_context_is_invalid_argument():
    """Every context entry point checks its arguments before touching a
    device: a null context is InvalidArgument (1 + Errc index 9)."""
    lib = _lib.load()
    inval = 1 + 9
    assert lib.pos_update_buffer_set(None, None, 0) == inval
    assert lib.pos_set_target_fresh(None, 1) == inval
    assert lib.pos_final_stop(None, None, 3, 4, None, None) == inval
    assert lib.pos_commit_epoch(None) == inval
    assert lib.pos_record_dirty(None, None, 0) == inval


def _mb(orc, seed, n):
    out = np.empty(n, np.uint8)
    orc.or_fill_bytes(seed, out.ctypes.data, n)
    return out


def _image_from_desc(orc, d):
    img = pd.CheckpointImage(page_size=d["page_size"])
    img.host_pages = [(idx, _mb(orc, seed, d["page_size"]).tobytes()) for idx, seed in d["pages"]]
    for r in d["recs"]:
        if r["kind"] == 0:
            img.gpu_records.append(pd.GpuBufferRec(r["handle"], 0, inline_bytes=_mb(orc, r["seed"], r["len"])))
        elif r["kind"] == 1:
            img.gpu_records.append(pd.GpuBufferRec(r["handle"], 1, dedup_first_page=r["first_page"],
                                                   dedup_page_count=r["page_count"],
                                                   dedup_offset=r["offset"], dedup_crc=r["crc"]))
        else:
            img.gpu_records.append(pd.GpuBufferRec(r["handle"], 2, recompute_nodes=r["nodes"]))
    img.allocs = [tuple(a) for a in d["allocs"]]
    img.stream_ids = list(d["streams"])
    img.cursor, img.next_handle, img.next_base = d["cursor"], d["next_handle"], d["next_base"]
    img.dag_bytes = bytes.fromhex(d["dag"])
    return img


def test_write_image_matches_reference_golden(orc):
    """image.hpp:136-207; golden bytes produced by the reference's write_image."""
    for g in json.load(open(os.path.join(GOLD, "images.json"))):
        got = pd.write_image(_image_from_desc(orc, g["desc"]))
        assert got.hex() == g["posi_hex"], g["desc"]["name"]
    empty = json.load(open(os.path.join(GOLD, "images.json")))[0]
    assert len(bytes.fromhex(empty["posi_hex"])) == 64  # test_image.cpp:86-95


def test_write_image_rejects_record_without_alloc():  # image.hpp:152-154
    img = pd.CheckpointImage()
    img.gpu_records.append(pd.GpuBufferRec(7, 0, inline_bytes=np.zeros(4, np.uint8)))
    with pytest.raises(pd.SimError) as e:
        pd.write_image(img)
    assert e.value.errc == "InvariantViolation"


def _random_desc(rng):
    """Random valid image description, shaped like test_image.cpp:12-78."""
    ps = int(rng.choice([64, 256, 4096]))
    pages = [(int(i), int(rng.integers(1, 1 << 30))) for i in rng.choice(100, int(rng.integers(0, 5)), replace=False)]
    handles = sorted(int(h) for h in rng.choice(np.arange(1, 50), int(rng.integers(0, 6)), replace=False))
    recs, allocs, base = [], [], BASE
    for h in rng.permutation(handles):
        size = int(rng.integers(1, 3000))
        allocs.append((int(h), base, size))
        base += (size + 255) // 256 * 256
        k = int(rng.integers(0, 3))
        if k == 0:
            recs.append({"handle": int(h), "kind": 0, "seed": int(rng.integers(1, 1 << 30)), "len": size})
        elif k == 1:
            recs.append({"handle": int(h), "kind": 1, "first_page": int(rng.integers(0, 9)),
                         "page_count": int(rng.integers(1, 4)), "offset": int(rng.integers(0, ps)),
                         "crc": int(rng.integers(0, 1 << 32))})
        else:
            recs.append({"handle": int(h), "kind": 2, "nodes": [int(x) for x in rng.integers(0, 1 << 40, int(rng.integers(1, 4)))]})
    meta_default = rng.random() < 0.3 and not allocs
    return {"name": "rand", "page_size": ps, "pages": pages, "recs": recs, "allocs": allocs,
            "streams": [] if meta_default else [int(x) for x in rng.integers(0, 9, int(rng.integers(0, 3)))],
            "cursor": 0 if meta_default else int(rng.integers(0, 1000)),
            "next_handle": 1 if meta_default else 50, "next_base": BASE if meta_default else base,
            "dag": "" if rng.random() < 0.5 else bytes(rng.integers(0, 256, int(rng.integers(1, 40)), dtype=np.uint8)).hex()}


def test_write_image_random_vs_reference(orc, ref):
    """200 random images through both writers: byte-identical."""
    from oracle_ctypes import ref_image
    rng = np.random.default_rng(2024)
    for _ in range(200):
        d = _random_desc(rng)
        want = ref_image(ref, d)
        assert pd.write_image(_image_from_desc(orc, d)) == want


def test_pack_apply_host_matches_oracle(orc):
    cs = 1000
    bufs = [(2, _mb(orc, 1, 5000)), (5, _mb(orc, 2, 2345)), (9, _mb(orc, 3, 7))]
    nch = sum(orc.or_chunk_count(a.size, cs) for _, a in bufs)
    flags = (np.random.default_rng(0).random(nch) < 0.6).astype(np.uint8)
    arr = (or_buffer_t * 3)(*[or_buffer_t(h, a.ctypes.data, a.size) for h, a in bufs])
    n = orc.or_build_pack(arr, 3, cs, flags.ctypes.data, 0, 0, None)
    pack = np.empty(n, np.uint8)
    orc.or_build_pack(arr, 3, cs, flags.ctypes.data, 0, 0, pack.ctypes.data)
    for threads in (1, 4):
        mine = [np.zeros_like(a) for _, a in bufs]
        theirs = [np.zeros_like(a) for _, a in bufs]
        pd.apply_pack_host(pack, [h for h, _ in bufs], mine, threads=threads)
        ptrs = (C.c_void_p * 3)(*[t.ctypes.data for t in theirs])
        hs = np.array([h for h, _ in bufs], np.uint64)
        sz = np.array([a.size for _, a in bufs], np.uint64)
        assert orc.or_apply_pack(pack.ctypes.data, pack.size, ptrs, hs.ctypes.data, sz.ctypes.data, 3) == 0
        for m, t in zip(mine, theirs):
            assert np.array_equal(m, t)
    with pytest.raises(pd.SimError) as e:  # unknown handle -> InvalidLocator
        pd.apply_pack_host(pack, [2, 5], [np.zeros(5000, np.uint8), np.zeros(2345, np.uint8)])
    assert e.value.errc == "InvalidLocator"
    bad = pack.copy()
    bad[:4] = 0
    with pytest.raises(pd.CorruptImageError):
        pd.apply_pack_host(bad, [h for h, _ in bufs], [np.zeros_like(a) for _, a in bufs])


def _ours_check(data: bytes) -> int:
    """0 if valid, else 1 + the CorruptImageError offset (ref_read_image_check's encoding)."""
    try:
        pd.read_image_check(data)
        return 0
    except pd.CorruptImageError as e:
        return 1 + e.offset


def test_read_image_check_dag_section_matches_reference(ref):
    """read_image's DAG validation (image.hpp:309-319 -> KernelDag::deserialize,
    dag.hpp:322-387; recompute nodes, :355-356): the reference engine's own
    images (real KDAG sections, Recompute records) and ~3000 mutations
    confined to their DAG section or the recompute node ids -- same
    accept/reject, same CorruptImageError offset (DAG-relative for a
    truncated read, 0 for a structural error, the image end for the
    cross-section checks).  Plus 300 images with random DAG bytes."""
    import struct
    from oracle_ctypes import ref_image
    from posi import read_posi
    rng = np.random.default_rng(91)
    cases = []
    for prof, seed, mode in [("resnet-train-desk", 1, 3), ("fuzz", 7, 3), ("ppo-train-desk", 2, 3),
                             ("gpt2-infer-desk", 1, 3)]:
        n = ref.ref_checkpoint_image(prof.encode(), 0, seed, mode, None, 0)
        buf = C.create_string_buffer(n)
        ref.ref_checkpoint_image(prof.encode(), 0, seed, mode, buf, n)
        data = buf.raw[:n]
        cases.append(data)
        dag_len, meta_len = struct.unpack_from("<QQ", data, 40)
        dag_lo = n - meta_len - dag_len
        for _ in range(700 if dag_len else 0):
            b = bytearray(data)
            k = int(rng.integers(0, 4))
            i = dag_lo + int(rng.integers(0, dag_len))
            if k == 0:
                b[i] ^= 1 << int(rng.integers(0, 8))
            elif k == 1:  # small length fields: make a count/len word large or small
                b[i] = int(rng.integers(0, 256))
            elif k == 2:  # a word of the header region of a node record
                j = dag_lo + int(rng.integers(0, min(dag_len, 64)))
                b[j] ^= 0xFF
            else:  # a recompute node id (Recompute records only exist in ppo)
                im = read_posi(data)
                rec = [r for r in im["recs"] if r["kind"] == 2]
                if not rec:
                    continue
                pos = data.index(struct.pack("<Q", rec[0]["nodes"][0]), 64)
                b[pos] ^= 1
            cases.append(bytes(b))
    for _ in range(300):
        d = _random_desc(rng)
        d["dag"] = bytes(rng.integers(0, 256, int(rng.integers(1, 40)), dtype=np.uint8)).hex()
        cases.append(ref_image(ref, d))
    n_bad = 0
    for c in cases:
        arr = np.frombuffer(c, np.uint8)
        want = ref.ref_read_image_check(arr.ctypes.data, arr.size)
        assert _ours_check(c) == want, len(c)
        n_bad += want != 0
    assert n_bad > 500


def test_read_image_check_matches_reference(orc, ref):
    """read_image (image.hpp:209-361): on 300 writer-generated images and ~4000
    corruptions of them -- byte flips, truncations, appended bytes -- our
    validator accepts exactly what the reference accepts and reports the
    same CorruptImageError offset (DAG sections: the test above)."""
    from oracle_ctypes import ref_image
    rng = np.random.default_rng(77)
    n_valid = n_checked = 0
    for _ in range(300):
        d = _random_desc(rng)
        d["dag"] = ""
        if rng.random() < 0.5:  # make the dedup checksums right so some images are valid
            for r in d["recs"]:
                if r["kind"] == 1:
                    r["page_count"] = 1
                    r["first_page"] = 0
                    r["offset"] = 0
            d["pages"] = [(0, 99)] + [p for p in d["pages"] if p[0] != 0]
            d["pages"].sort()
        data = ref_image(ref, d)
        cases = [data]
        for _ in range(12):
            b = bytearray(data)
            k = int(rng.integers(0, 3))
            if k == 0 and b:
                i = int(rng.integers(0, len(b)))
                b[i] ^= 1 << int(rng.integers(0, 8))
            elif k == 1 and b:
                del b[int(rng.integers(0, len(b))):]
            else:
                b += bytes(rng.integers(0, 256, int(rng.integers(1, 9)), dtype=np.uint8))
            cases.append(bytes(b))
        for c in cases:
            buf = np.frombuffer(c, np.uint8)
            want = ref.ref_read_image_check(buf.ctypes.data if buf.size else None, buf.size)
            assert _ours_check(c) == want, (d, len(c))
            n_valid += want == 0
            n_checked += 1
    assert n_valid > 50 and n_checked > 3500


def test_write_image_large_payloads_vs_reference(orc, ref):
    """Inline payloads of 1-70 MiB (copied by the writer's thread pool in
    64 MiB pieces after its layout pass) and 1 MiB host pages: byte-identical
    to the reference's write_image."""
    from oracle_ctypes import ref_image
    rng = np.random.default_rng(77)
    sizes = [1 << 20, (1 << 20) - 1, 3 * (1 << 20) + 5, 70 * (1 << 20) + 3, 200]
    recs, allocs, base = [], [], BASE
    for h, size in zip([9, 2, 5, 7, 11], sizes):
        allocs.append((h, base, size))
        base += (size + 255) // 256 * 256
        recs.append({"handle": h, "kind": 0, "seed": int(rng.integers(1, 1 << 30)), "len": size})
    d = {"name": "large", "page_size": 1 << 20, "pages": [(3, 11), (0, 12)], "recs": recs, "allocs": allocs,
         "streams": [1], "cursor": 5, "next_handle": 12, "next_base": base, "dag": ""}
    assert pd.write_image(_image_from_desc(orc, d)) == ref_image(ref, d)
