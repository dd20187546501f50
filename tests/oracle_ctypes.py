"""ctypes access to the test-only checkers (never imported by the product):
oracle/liboracle.so (C restatement) and oracle/_ref/libgpucrsim_ref.so (the
reference's own headers compiled from /root/reference)."""
from __future__ import annotations

import ctypes as C
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libgpucrsim_ref.so")

P, U64, U32, I32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int


class or_buffer_t(C.Structure):
    _fields_ = [("handle", U64), ("content", P), ("size", U64)]


_ORACLE = {
    "or_crc32_update": (U32, [U32, P, C.c_size_t]),
    "or_crc32": (U32, [P, C.c_size_t]),
    "or_crc32_combine": (U32, [U32, U32, U64]),
    "or_splitmix_next": (U64, [C.POINTER(U64)]),
    "or_mix64": (U64, [U64, U64]),
    "or_fill_bytes": (None, [U64, P, C.c_size_t]),
    "or_fill_bytes_at": (None, [U64, U64, P, C.c_size_t]),
    "or_fnv1a": (U64, [P, C.c_size_t, U64]),
    "or_chunk_count": (U32, [U64, U64]),
    "or_chunk_bytes": (U64, [U64, U64, U32]),
    "or_chunk_digests": (U32, [P, U64, U64, P]),
    "or_dirty_flags": (U64, [P, P, U64, I32, P]),
    "or_pack_bitmap": (None, [P, U64, P]),
    "or_fold_digests": (U32, [P, U64, U64]),
    "or_dedup_verdict": (I32, [I32, U32, U32, I32]),
    "or_build_pack": (U64, [C.POINTER(or_buffer_t), U32, U64, P, U64, U32, P]),
    "or_apply_pack": (I32, [P, U64, P, P, P, U32]),
}

_REF = {
    "ref_crc32": (U32, [P, U64]),
    "ref_crc32_update": (U32, [U32, P, U64]),
    "ref_mix64": (U64, [U64, U64]),
    "ref_fnv1a": (U64, [P, U64, U64]),
    "ref_make_bytes": (None, [U64, P, U64]),
    "ref_chunk_geometry": (U32, [U64, U64, P]),
    "ref_write_image": (U64, [U64, P, U32, P, U32, P, U32, P, U32, U64, U64, U64, P, U64, P, U64]),
    "ref_read_image_check": (U64, [P, U64]),
    "ref_state_create": (P, [U32, P, P, U64]),
    "ref_state_destroy": (None, [P]),
    "ref_state_dump": (U64, [P, P, I32, P, P, U32]),
    "ref_state_write": (None, [P, U32, U64, P, U64]),
    "ref_state_captured": (None, [P, U32, P]),
    "ref_gen_workload": (U64, [C.c_char_p, U64, U64, U64, U64, P, U64]),
    "ref_checkpoint_image": (U64, [C.c_char_p, U64, U64, I32, P, U64]),
    "ref_checkpoint_session": (U64, [C.c_char_p, U64, U64, I32, P, U64]),
    "ref_fnv1a_u64": (U64, [U64, U64]),
    "ref_snapshot_hash": (U64, [U32, P, P, P, P, U32, P, P, U64]),
    "ref_restore_hash": (U64, [P, U64]),
    "ref_plain_hash": (U64, [C.c_char_p, U64, U64, U64]),
    "ref_replay_plan": (U64, [P, U64, P, U64]),
}


def _load(path, sigs):
    lib = C.CDLL(path)
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_cache: dict = {}


def oracle():
    if "o" not in _cache:
        if not os.path.exists(ORACLE_SO):
            import subprocess
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")], check=True)
        _cache["o"] = _load(ORACLE_SO, _ORACLE)
    return _cache["o"]


def reference():
    """The reference's own code, or None when oracle/_ref was never built."""
    if "r" not in _cache:
        _cache["r"] = _load(REF_SO, _REF) if os.path.exists(REF_SO) else None
    return _cache["r"]


class Rec(C.Structure):
    _fields_ = [("handle", C.c_uint64), ("kind", C.c_uint32), ("n_recompute", C.c_uint32),
                ("inline_bytes", C.c_void_p), ("inline_len", C.c_uint64),
                ("dedup_first_page", C.c_uint64), ("dedup_page_count", C.c_uint32),
                ("dedup_offset", C.c_uint32), ("dedup_crc", C.c_uint32), ("pad", C.c_uint32),
                ("recompute", C.c_void_p)]


class Alloc(C.Structure):
    _fields_ = [("handle", C.c_uint64), ("base", C.c_uint64), ("size", C.c_uint64)]


class Page(C.Structure):
    _fields_ = [("index", C.c_uint64), ("bytes", C.c_void_p)]


def ref_image(ref, desc):
    """Bytes of the reference's write_image for a JSON image description."""
    import numpy as np

    def mb(seed, n):
        out = np.empty(n, np.uint8)
        ref.ref_make_bytes(seed, out.ctypes.data, n)
        return out

    keep = []
    ps = desc["page_size"]
    pages = (Page * max(1, len(desc["pages"])))()
    for i, (idx, seed) in enumerate(desc["pages"]):
        a = mb(seed, ps)
        keep.append(a)
        pages[i].index, pages[i].bytes = idx, a.ctypes.data
    recs = (Rec * max(1, len(desc["recs"])))()
    for i, r in enumerate(desc["recs"]):
        recs[i].handle, recs[i].kind = r["handle"], r["kind"]
        if r["kind"] == 0:
            a = mb(r["seed"], r["len"])
            keep.append(a)
            recs[i].inline_bytes, recs[i].inline_len = a.ctypes.data, a.nbytes
        elif r["kind"] == 1:
            recs[i].dedup_first_page, recs[i].dedup_page_count = r["first_page"], r["page_count"]
            recs[i].dedup_offset, recs[i].dedup_crc = r["offset"], r["crc"]
        else:
            a = np.array(r["nodes"], np.uint64)
            keep.append(a)
            recs[i].recompute, recs[i].n_recompute = a.ctypes.data, a.size
    allocs = (Alloc * max(1, len(desc["allocs"])))(*[Alloc(*a) for a in desc["allocs"]])
    streams = np.array(desc["streams"], np.uint64)
    dag = np.frombuffer(bytes.fromhex(desc["dag"]), np.uint8) if desc["dag"] else np.zeros(0, np.uint8)
    args = [ps, pages, len(desc["pages"]), recs, len(desc["recs"]), allocs, len(desc["allocs"]),
            streams.ctypes.data if streams.size else None, streams.size, desc["cursor"],
            desc["next_handle"], desc["next_base"], dag.ctypes.data if dag.size else None, dag.size]
    n = ref.ref_write_image(*args, None, 0)
    out = np.empty(n, np.uint8)
    ref.ref_write_image(*args, out.ctypes.data, n)
    return out.tobytes()


def ref_session(ref, profile: str, seed: int, mode: int, total_bytes: int = 0) -> dict:
    """The reference CrEngine's finalize_image inputs for one checkpoint
    (ref_checkpoint_session): the image it wrote, its CrMetrics, and per
    allocation the device bytes, Upstream, O1 verdict, dirty bit,
    recompute eligibility and pending writers."""
    import struct
    n = ref.ref_checkpoint_session(profile.encode(), total_bytes, seed, mode, None, 0)
    buf = C.create_string_buffer(n)
    ref.ref_checkpoint_session(profile.encode(), total_bytes, seed, mode, buf, n)
    b = buf.raw[:n]
    assert b[:4] == b"SESS"
    nb, ilen = struct.unpack_from("<IQ", b, 4)
    o = 16
    image = b[o:o + ilen]
    o += ilen
    keys = ["bytes_precopy", "bytes_dirty", "bytes_dedup_saved", "bytes_recompute_saved", "image_bytes",
            "image_file_bytes", "dirty_count", "retention"]
    metrics = dict(zip(keys, struct.unpack_from("<8Q", b, o)))
    o += 64
    bufs = []
    for _ in range(nb):
        h, base, size, has_up, up_addr, up_len, up_crc, untouched, ok, dirty, rec, npw = struct.unpack_from(
            "<QQQIQQIIiIII", b, o)
        o += struct.calcsize("<QQQIQQIIiIII")
        pending = list(struct.unpack_from(f"<{npw}Q", b, o))
        o += 8 * npw
        (clen,) = struct.unpack_from("<Q", b, o)
        o += 8
        content = b[o:o + clen]
        o += clen
        bufs.append(dict(handle=h, base=base, size=size, has_upstream=bool(has_up), up_host_addr=up_addr,
                         up_len=up_len, up_crc=up_crc, host_untouched=bool(untouched), dedup_ok=ok,
                         dirty=bool(dirty), recompute_eligible=bool(rec & 1), final_recopy=bool(rec & 2),
                         precopy_survived=bool(rec & 4), pending=pending, content=content))
    return {"image": image, "metrics": metrics, "bufs": bufs}


API_KINDS = ["Malloc", "Free", "MemcpyH2D", "MemcpyD2H", "MemcpyD2D", "LaunchKnown", "LaunchOpaque",
             "StreamCreate", "StreamDestroy", "DeviceSynchronize", "StreamSynchronize", "GetDevice"]


def ref_replay_plan(ref, image: bytes) -> list:
    """Pending DAG nodes of an image, in replay order (replay_pending)."""
    import struct
    src = C.create_string_buffer(image, len(image))
    n = ref.ref_replay_plan(src, len(image), None, 0)
    buf = C.create_string_buffer(max(n, 1))
    ref.ref_replay_plan(src, len(image), buf, n)
    b, o, out = buf.raw[:n], 0, []
    while o < n:
        kind, ln = struct.unpack_from("<II", b, o)
        o += 8
        name = b[o:o + ln]
        o += ln
        seq, dst, srcp, nbytes = struct.unpack_from("<QQQQ", b, o)
        o += 32
        (nr,) = struct.unpack_from("<I", b, o)
        reads = list(struct.unpack_from(f"<{nr}Q", b, o + 4))
        o += 4 + 8 * nr
        (nw,) = struct.unpack_from("<I", b, o)
        writes = list(struct.unpack_from(f"<{nw}Q", b, o + 4))
        o += 4 + 8 * nw
        out.append(dict(kind=API_KINDS[kind], name=name, seq=seq, dst=dst, src=srcp, bytes=nbytes,
                        reads=reads, writes=writes))
    return out
