"""Host-side mirror of the reference's dump-path interface over libposdump.so.

Names follow the reference (proj/include/gpucrsim): ``crc32`` /
``crc32_update`` (crc32.hpp:26-34), ``GpuBuffer.chunk_count/chunk_bytes``
(buffer.hpp:44-49), and a ``DumpEngine`` exposing the hot-path members of
``CrEngine`` (cr.hpp:124-1322): ``plan_precopy`` / ``scan_dedup`` /
``dedup_verdicts`` / ``record_dirty`` / ``dirty_set`` / ``at_final_stop`` /
``finalize_image`` / ``materialize``.  Errors raise ``SimError`` with the
reference's Errc names.  Every byte-level operation is a CUDA kernel behind
the C ABI; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import SimError, CorruptImageError, NoDeviceError, check  # noqa: F401

kDeviceAddrBase = 0x7000_0000_0000  # config.hpp:14
H2D, D2H, D2D = 1, 2, 3


def lib():
    return _lib.load()


def _s(stream) -> Optional[int]:
    return None if stream is None else int(stream)


# ---------------------------------------------------------------------------
# plumbing

def device_count() -> int:
    n = C.c_int(0)
    check(lib().pos_device_count(C.byref(n)))
    return n.value


class DeviceMemory:
    """A raw device allocation (cudaMalloc), freed on close/GC."""

    def __init__(self, nbytes: int):
        p = C.c_uint64(0)
        check(lib().pos_dev_malloc(nbytes, C.byref(p)))
        self.ptr, self.nbytes = p.value, nbytes

    def close(self):
        if self.ptr:
            lib().pos_dev_free(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, data, offset: int = 0, stream=None):
        a = np.ascontiguousarray(np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data.view(np.uint8))
        check(lib().pos_memcpy(self.ptr + offset, a.ctypes.data, a.nbytes, H2D, _s(stream)))
        check(lib().pos_stream_sync(_s(stream)))

    def download(self, nbytes: Optional[int] = None, offset: int = 0, stream=None) -> np.ndarray:
        n = self.nbytes - offset if nbytes is None else nbytes
        out = np.empty(n, dtype=np.uint8)
        check(lib().pos_memcpy(out.ctypes.data, self.ptr + offset, n, D2H, _s(stream)))
        check(lib().pos_stream_sync(_s(stream)))
        return out


class PinnedHost:
    """Page-locked host memory viewed as a numpy array: cudaHostAlloc, or with
    image=True the huge-page image allocator (pos_host_image_alloc: pinned +
    mapped, zero-filled, ~10x faster to allocate at 100+ GB)."""

    def __init__(self, nbytes: int, image: bool = False, threads: int = 0):
        p = C.c_void_p(0)
        self.image = image
        if image:
            check(lib().pos_host_image_alloc(max(nbytes, 1), threads, C.byref(p)))
        else:
            check(lib().pos_host_malloc_pinned(max(nbytes, 1), C.byref(p)))
        self.ptr, self.nbytes = p.value, nbytes
        self.array = np.ctypeslib.as_array((C.c_uint8 * max(nbytes, 1)).from_address(self.ptr))[:nbytes]

    def close(self):
        if self.ptr:
            self.array = None
            if self.image:
                lib().pos_host_image_free(self.ptr)
            else:
                lib().pos_host_free_pinned(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Stream:
    def __init__(self, priority: int = 0):
        s = C.c_void_p(0)
        check(lib().pos_stream_create_prio(priority, C.byref(s)))
        self.handle = s.value

    def __int__(self):
        return self.handle

    def synchronize(self):
        check(lib().pos_stream_sync(self.handle))

    def wait(self, other: "Stream"):
        check(lib().pos_stream_wait(self.handle, int(other)))

    def close(self):
        if self.handle:
            lib().pos_stream_destroy(self.handle)
            self.handle = 0


def device_synchronize():
    check(lib().pos_device_sync())


# ---------------------------------------------------------------------------
# crc32 over device memory (crc32.hpp:26-34)

def crc32(dev_ptr: int, n: int, stream=None) -> int:
    out = C.c_uint32(0)
    check(lib().pos_crc32(dev_ptr, n, C.byref(out), _s(stream)))
    return out.value


def crc32_update(crc: int, dev_ptr: int, n: int, stream=None) -> int:
    out = C.c_uint32(0)
    check(lib().pos_crc32_update(crc, dev_ptr, n, C.byref(out), _s(stream)))
    return out.value


def fill_bytes(dev_ptr: int, n: int, seed: int, stream=None) -> None:
    """Device fill_bytes (rng.hpp:43-54); asynchronous on `stream`."""
    check(lib().pos_fill(dev_ptr, n, seed & 0xFFFFFFFFFFFFFFFF, _s(stream)))


def fill_batch(ranges: Sequence[tuple[int, int, int]], stream=None) -> None:
    if not ranges:
        return
    a = np.array([[p, n, s & 0xFFFFFFFFFFFFFFFF] for p, n, s in ranges], dtype=np.uint64)
    check(lib().pos_fill_batch(a.ctypes.data, len(ranges), _s(stream)))


# ---------------------------------------------------------------------------
# buffers

@dataclass
class Upstream:
    """buffer.hpp:20-25 (+ the cr.hpp:420 host watermark verdict)."""
    crc: int
    host_untouched: bool = True


@dataclass
class GpuBuffer:
    """The fields of gpucrsim::GpuBuffer (buffer.hpp:27-41) the path reads."""
    handle: int
    dev_ptr: int
    size: int
    upstream: Optional[Upstream] = None
    written_since_ckpt: bool = True

    def chunk_count(self, chunk_size: int) -> int:  # buffer.hpp:44, :119
        return (self.size + chunk_size - 1) // chunk_size

    def chunk_bytes(self, idx: int, chunk_size: int) -> int:  # buffer.hpp:46-49
        return min(chunk_size, self.size - idx * chunk_size)

    def desc(self) -> _lib.pos_buffer_desc:
        d = _lib.pos_buffer_desc()
        d.handle, d.dev_ptr, d.size = self.handle, self.dev_ptr, self.size
        d.has_upstream = 1 if self.upstream is not None else 0
        d.upstream_crc = self.upstream.crc if self.upstream else 0
        d.host_untouched = 1 if (self.upstream and self.upstream.host_untouched) else 0
        d.written_since_ckpt = 1 if self.written_since_ckpt else 0
        return d


# ---------------------------------------------------------------------------
# POSD packs

PACK_HEADER, PACK_ENTRY = 64, 32


def parse_pack(pack: np.ndarray) -> dict:
    """Header + entries of a POSD pack held in host memory."""
    b = pack.view(np.uint8)
    if b[:4].tobytes() != b"POSD":
        raise CorruptImageError(_lib.CODES["CorruptImage"], "bad pack magic")
    hdr = b[:64]
    n = int(hdr[16:20].view(np.uint32)[0])
    ents = b[64:64 + 32 * n].reshape(n, 32) if n else np.zeros((0, 32), np.uint8)
    return {
        "chunk_size": int(hdr[8:16].view(np.uint64)[0]),
        "n_entries": n,
        "flags": int(hdr[20:24].view(np.uint32)[0]),
        "payload_off": int(hdr[24:32].view(np.uint64)[0]),
        "payload_bytes": int(hdr[32:40].view(np.uint64)[0]),
        "epoch": int(hdr[40:48].view(np.uint64)[0]),
        "total": int(hdr[48:56].view(np.uint64)[0]),
        "handle": ents[:, 0:8].copy().view(np.uint64).ravel(),
        "offset": ents[:, 8:16].copy().view(np.uint64).ravel(),
        "chunk": ents[:, 16:20].copy().view(np.uint32).ravel(),
        "len": ents[:, 20:24].copy().view(np.uint32).ravel(),
        "crc": ents[:, 24:28].copy().view(np.uint32).ravel(),
    }


def apply_pack_host(pack: np.ndarray, handles: Sequence[int], hosts: Sequence[np.ndarray],
                    threads: int = 1) -> None:
    """Apply a POSD pack onto host copies of the buffers (cr.hpp:499-501)."""
    n = len(handles)
    h = np.ascontiguousarray(np.array(handles, dtype=np.uint64))
    ptrs = (C.c_void_p * max(n, 1))(*[x.ctypes.data for x in hosts])
    sizes = np.array([x.nbytes for x in hosts], dtype=np.uint64)
    check(lib().pos_pack_apply_host(pack.ctypes.data, pack.nbytes, h.ctypes.data, ptrs,
                                    sizes.ctypes.data, n, threads))


# ---------------------------------------------------------------------------
# the engine

@dataclass
class SimConfig:
    """The SimConfig keys of the path (config.hpp:18-45)."""
    chunk_size: int = 64 * 1024
    page_size: int = 4096
    device_capacity: int = 80_000_000_000
    staging_fraction: float = 1.0 / 16.0
    dedup: bool = True
    cache_capacity: int = 0  # explicit O3 cache size; 0 => staging_capacity of the device
    dirty_threshold_frac: float = 0.25  # DAG retention (config.hpp:32)
    trust_written_bit: bool = False  # buffer-level O2 first (cr.hpp:396-401): clean buffers are not hashed


class DumpEngine:
    """Hot-path members of gpucrsim::CrEngine over the CUDA path."""

    def __init__(self, cfg: SimConfig = SimConfig(), device: int = 0):
        self.cfg = cfg
        c = _lib.pos_config()
        c.chunk_size, c.page_size = cfg.chunk_size, cfg.page_size
        c.cache_capacity = cfg.cache_capacity
        c.staging_fraction = cfg.staging_fraction
        c.device, c.dedup = device, 1 if cfg.dedup else 0
        c.dirty_threshold_frac = cfg.dirty_threshold_frac
        c.trust_written_bit = 1 if cfg.trust_written_bit else 0
        ctx = C.c_void_p(0)
        check(lib().pos_ctx_create(C.byref(c), C.byref(ctx)))
        self.ctx = ctx.value
        self.buffers: list[GpuBuffer] = []
        self.precopy_bytes = 0

    def close(self):
        if getattr(self, "ctx", None):
            lib().pos_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # snapshot_buffers_ = active_handles() (cr.hpp:346)
    def register_buffers(self, bufs: Iterable[GpuBuffer]) -> None:
        self.buffers = sorted(bufs, key=lambda b: b.handle)
        arr = (_lib.pos_buffer_desc * max(len(self.buffers), 1))(*[b.desc() for b in self.buffers])
        check(lib().pos_register_buffers(self.ctx, arr, len(self.buffers)))

    def update_buffer_set(self, bufs: Iterable[GpuBuffer]) -> None:
        """The snapshot's buffers changed mid-session (cr.hpp:301-306,
        709-716): unchanged buffers keep their digest history and image
        range; new ones join fresh (all chunks dirty until commit_epoch);
        missing ones are dropped."""
        self.buffers = sorted(bufs, key=lambda b: b.handle)
        arr = (_lib.pos_buffer_desc * max(len(self.buffers), 1))(*[b.desc() for b in self.buffers])
        check(lib().pos_update_buffer_set(self.ctx, arr, len(self.buffers)))

    def update_buffer(self, b: GpuBuffer) -> None:
        d = b.desc()
        check(lib().pos_update_buffer(self.ctx, C.byref(d)))

    @property
    def n_chunks(self) -> int:
        n = C.c_uint64(0)
        check(lib().pos_num_chunks(self.ctx, C.byref(n)))
        return n.value

    # ---- O2
    def hash_chunks(self, stream=None) -> None:
        check(lib().pos_hash_chunks(self.ctx, _s(stream)))

    def set_target_fresh(self, fresh: bool = True) -> None:
        """CheckpointTarget::fresh (cr.hpp:35, 396): the next round ships
        every chunk (until commit_epoch)."""
        check(lib().pos_set_target_fresh(self.ctx, 1 if fresh else 0))

    def commit_epoch(self) -> None:
        check(lib().pos_commit_epoch(self.ctx))

    def digests(self, stream=None) -> np.ndarray:
        out = np.empty(self.n_chunks, dtype=np.uint32)
        check(lib().pos_read_digests(self.ctx, out.ctypes.data, out.size, _s(stream)))
        return out

    def flags(self, stream=None) -> np.ndarray:
        out = np.empty(self.n_chunks, dtype=np.uint8)
        check(lib().pos_read_flags(self.ctx, out.ctypes.data, out.size, _s(stream)))
        return out

    def bitmap(self, stream=None) -> np.ndarray:
        out = np.empty((self.n_chunks + 31) // 32, dtype=np.uint32)
        check(lib().pos_read_bitmap(self.ctx, out.ctypes.data, out.size, _s(stream)))
        return out

    # ---- O1 (scan_dedup, cr.hpp:416-425)
    def scan_dedup(self, stream=None) -> None:
        check(lib().pos_buffer_crc(self.ctx, _s(stream)))

    def buffer_crcs(self, stream=None) -> tuple[np.ndarray, np.ndarray]:
        n = len(self.buffers)
        crcs = np.empty(n, dtype=np.uint32)
        ver = np.empty(n, dtype=np.uint8)
        check(lib().pos_read_buffer_crcs(self.ctx, crcs.ctypes.data, ver.ctypes.data, n, _s(stream)))
        return crcs, ver

    def dedup_verdicts(self, stream=None) -> dict[int, bool]:
        """dedup_ok_ (cr.hpp:141): only buffers with upstream provenance."""
        _, ver = self.buffer_crcs(stream)
        return {b.handle: bool(v) for b, v in zip(self.buffers, ver) if b.upstream is not None}

    # ---- DAG write sets (record_dirty, cr.hpp:901-931)
    def app_copy(self, dst: int, src: int, nbytes: int, kind: int, stream=None) -> None:
        """An application memcpy during a checkpoint (CopyEngine::submit(App)):
        the host leg yields to it (app > ckpt at slice granularity)."""
        check(lib().pos_app_copy(self.ctx, dst, src, nbytes, kind, _s(stream)))

    def set_hash_sms(self, sms: int) -> None:
        """SMs the hash may occupy (0 = all): the rest stay with the application."""
        check(lib().pos_set_hash_sms(self.ctx, sms))

    def set_o2_digest2(self, on: bool = True) -> None:
        """A second, non-linear chunk digest in the O2 compare (pos_set_o2_digest2)."""
        check(lib().pos_set_o2_digest2(self.ctx, 1 if on else 0))

    def set_host_leg(self, slice_bytes: int = 16 << 20, window: int = 3) -> None:
        check(lib().pos_set_host_leg(self.ctx, slice_bytes, window))

    def host_leg_stats(self) -> tuple[int, int, int]:
        """(slices, app copies yielded to, bytes cancelled by record_dirty)."""
        a, b, c = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        check(lib().pos_host_leg_stats(self.ctx, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def metrics(self) -> dict:
        """CrMetrics of the session (cr.hpp:69-119): final stop + finalize."""
        m = _lib.pos_metrics()
        check(lib().pos_get_metrics(self.ctx, C.byref(m)))
        return {k: int(getattr(m, k)) for k in METRIC_KEYS}

    def set_stop_exclusions(self, handles: Iterable[int]) -> None:
        """at_final_stop's exclusions (cr.hpp:608-613)."""
        a = np.array(sorted(set(handles)), dtype=np.uint64)
        check(lib().pos_set_stop_exclusions(self.ctx, a.ctypes.data if a.size else None, a.size))

    def record_dirty(self, handles: Iterable[int]) -> None:
        a = np.array(list(handles), dtype=np.uint64)
        check(lib().pos_record_dirty(self.ctx, a.ctypes.data if a.size else None, a.size))

    def clear_dirty(self) -> None:
        check(lib().pos_clear_dirty(self.ctx))

    # ---- O3 compaction
    def compact(self, exclude_dag_dirty: bool = True, stream=None) -> int:
        n = C.c_uint64(0)
        check(lib().pos_compact(self.ctx, 1 if exclude_dag_dirty else 0, _s(stream), C.byref(n)))
        self.precopy_bytes = n.value
        return n.value

    def plan_precopy(self, stream=None, exclude_dag_dirty: bool = True) -> int:
        """hash -> O1 verdicts -> compaction into the cache (cr.hpp:377-406).
        Returns the pre-copy pack size (bytes at cache offset 0)."""
        self.launch_precopy(stream, exclude_dag_dirty)
        return self.precopy_size()

    def launch_precopy(self, stream=None, exclude_dag_dirty: bool = True) -> None:
        """Asynchronous pre-copy (pos_precopy); pair with precopy_size()."""
        check(lib().pos_precopy(self.ctx, 1 if exclude_dag_dirty else 0, _s(stream)))

    def precopy_pipelined(self, host_ptr: Optional[int], waves: int = 4, stream=None, copy_stream=None,
                          exclude_dag_dirty: bool = True, slice_bytes: int = 0) -> list[tuple[int, int]]:
        """Wave-pipelined pre-copy with D2H of each wave's pack into host_ptr
        (same offsets as in the cache).  Returns [(offset, size)] per pack."""
        offs = (C.c_uint64 * 16)()
        sizes = (C.c_uint64 * 16)()
        n = C.c_uint32(0)
        check(lib().pos_precopy_pipelined(self.ctx, 1 if exclude_dag_dirty else 0, waves, _s(stream),
                                          _s(copy_stream), host_ptr, slice_bytes, offs, sizes, C.byref(n)))
        packs = [(offs[i], sizes[i]) for i in range(n.value)]
        if packs:
            o, z = packs[-1]
            self.precopy_bytes = o + z
        return packs

    def precopy_stream(self, sink, region_bytes: int = 0, stream=None, copy_stream=None,
                       exclude_dag_dirty: bool = True) -> tuple[int, int]:
        """Cache-cycled pre-copy (pos_precopy_stream) for states larger than the
        O3 cache: sink(pack: np.ndarray view, index) is called per wave, in
        order, while the next wave drains.  Returns (total pack bytes, packs)."""
        def _cb(user, ptr, nbytes, index):
            arr = np.ctypeslib.as_array(ptr, shape=(nbytes,)) if nbytes else np.zeros(0, np.uint8)
            sink(arr, index)
        cb = _lib.PACK_SINK(_cb)
        total, n = C.c_uint64(0), C.c_uint32(0)
        check(lib().pos_precopy_stream(self.ctx, 1 if exclude_dag_dirty else 0, _s(stream), _s(copy_stream),
                                       region_bytes, C.cast(cb, C.c_void_p), None, C.byref(total), C.byref(n)))
        self.precopy_bytes = 0
        return total.value, n.value

    # ---- H2D provenance (note_h2d_provenance, process.hpp:505-522)
    def h2d_provenance(self, dst: int, host: Optional[np.ndarray] = None, nbytes: Optional[int] = None,
                       stream=None) -> None:
        """H2D of `host` into device address dst (skipped when host is None:
        the caller enqueued it on `stream`), then Upstream::crc on the device."""
        if host is not None:
            host = np.ascontiguousarray(host).view(np.uint8).reshape(-1)
            nbytes = host.nbytes if nbytes is None else nbytes
            check(lib().pos_h2d_provenance(self.ctx, dst, host.ctypes.data, nbytes, 1, _s(stream)))
            self._h2d_keep = host  # pageable sources are staged by the call; pinned must stay alive
        else:
            check(lib().pos_h2d_provenance(self.ctx, dst, None, nbytes or 0, 0, _s(stream)))

    def upstream(self, handle: int) -> Optional[int]:
        """Upstream::crc of a buffer, or None without provenance."""
        has, crc = C.c_uint32(0), C.c_uint32(0)
        check(lib().pos_read_upstream(self.ctx, handle, C.byref(has), C.byref(crc)))
        return crc.value if has.value else None

    # ---- direct pre-copy into a registered host image (zero-copy chunk_copied)
    def register_image(self, hosts: Sequence[np.ndarray]) -> None:
        """hosts[i]: the host image of registered buffer i (uint8, its size);
        pinned memory is used as is, pageable arrays are pinned here."""
        arrs = list(hosts)
        if any(a.dtype != np.uint8 or not a.flags.c_contiguous for a in arrs):
            raise SimError(10, "image ranges must be contiguous uint8 arrays")  # InvalidArgument
        n = len(arrs)
        ptrs = (C.c_void_p * max(n, 1))(*[a.ctypes.data for a in arrs])
        sizes = np.array([a.size for a in arrs], dtype=np.uint64)
        check(lib().pos_register_image(self.ctx, ptrs, sizes.ctypes.data, n))
        self._image = arrs  # keep the memory alive

    def precopy_direct(self, waves: int = 1, stream=None, drain_stream=None,
                       exclude_dag_dirty: bool = True) -> None:
        """Pre-copy straight into the registered image (pos_precopy_direct);
        asynchronous -- pair with precopy_direct_result()."""
        check(lib().pos_precopy_direct(self.ctx, 1 if exclude_dag_dirty else 0, waves, _s(stream),
                                       _s(drain_stream)))

    def precopy_direct_result(self) -> tuple[int, int]:
        """(chunks, payload bytes) shipped by the last direct pre-copy."""
        n, pay, idx = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        check(lib().pos_precopy_direct_result(self.ctx, C.byref(n), C.byref(pay), C.byref(idx)))
        self.precopy_bytes = idx.value
        return n.value, pay.value

    def delta_drain(self, stream=None) -> None:
        """STW delta payload (in the cache) -> host image (pos_delta_drain)."""
        check(lib().pos_delta_drain(self.ctx, _s(stream)))

    # ---- NVLink peer-GPU cache (config 5) for precopy_stream
    def attach_peer_cache(self, peer_device: int, nbytes: int) -> None:
        check(lib().pos_peer_cache_attach(self.ctx, peer_device, nbytes))

    def peer_cache_stats(self) -> tuple[float, float]:
        """(capture ms, total ms) of the last precopy_stream through the peer cache."""
        a, b = C.c_float(0), C.c_float(0)
        check(lib().pos_peer_cache_stats(self.ctx, C.byref(a), C.byref(b)))
        return a.value, b.value

    def precopy_size(self) -> int:
        n = C.c_uint64(0)
        check(lib().pos_precopy_size(self.ctx, C.byref(n)))
        self.precopy_bytes = n.value
        return n.value

    # ---- CoW staging (gate_cow / stage_buffers, cr.hpp:806-888)
    def stage_buffers(self, handles: Iterable[int], stream=None) -> tuple[int, int]:
        """Stage whole buffers (stop-point bytes) into a staging pack before a
        kernel overwrites them; returns (cache offset, pack bytes)."""
        hs = np.array(sorted(set(handles)), dtype=np.uint64)
        off, n = C.c_uint64(0), C.c_uint64(0)
        check(lib().pos_stage_buffers(self.ctx, hs.ctypes.data if hs.size else None, hs.size, _s(stream),
                                      C.byref(off), C.byref(n)))
        return off.value, n.value

    # ---- STW delta-copy (at_final_stop, cr.hpp:599-621)
    def at_final_stop(self, stream=None, stw_end_slot: int = -1, stw_begin_slot: int = -1) -> tuple[int, int]:
        """STW delta pack: bulk gather, then the post-stop hash of the gathered
        copy.  With stw_begin_slot >= 0 the window is exactly [event begin,
        gather, event end] (pos_final_stop); otherwise event stw_end_slot
        (when >= 0) is recorded after the gather (pos_delta_copy_ex)."""
        off, n = C.c_uint64(0), C.c_uint64(0)
        if stw_begin_slot >= 0:
            check(lib().pos_final_stop(self.ctx, _s(stream), stw_begin_slot, stw_end_slot, C.byref(off), C.byref(n)))
        else:
            check(lib().pos_delta_copy_ex(self.ctx, _s(stream), stw_end_slot, C.byref(off), C.byref(n)))
        return off.value, n.value

    def prepare_final_stop(self, stream=None) -> tuple[int, int]:
        """Stage the delta pack layout before the stop (pos_delta_prepare)."""
        off, n = C.c_uint64(0), C.c_uint64(0)
        check(lib().pos_delta_prepare(self.ctx, _s(stream), C.byref(off), C.byref(n)))
        return off.value, n.value

    def pregather(self, handles: Iterable[int], after_stream=None, stream=None) -> None:
        """Eager delta capture (pos_delta_pregather): gather these DAG-dirty
        buffers into the prepared delta pack behind after_stream's writers."""
        hs = np.array(sorted(handles), dtype=np.uint64)
        check(lib().pos_delta_pregather(self.ctx, hs.ctypes.data if hs.size else None, int(hs.size),
                                        _s(after_stream), _s(stream)))

    # ---- host leg
    def d2h_async(self, host_ptr: int, offset: int, nbytes: int, stream=None, slice_bytes: int = 0) -> None:
        check(lib().pos_d2h_async(self.ctx, host_ptr, offset, nbytes, slice_bytes, _s(stream)))

    def cache(self) -> tuple[int, int]:
        p, cap = C.c_uint64(0), C.c_uint64(0)
        check(lib().pos_cache_info(self.ctx, C.byref(p), C.byref(cap)))
        return p.value, cap.value

    # ---- restore scatter (materialize / load_complete, cr.hpp:1026-1084)
    def materialize(self, pack_dev_ptr: int, pack_bytes: int, stream=None) -> None:
        check(lib().pos_scatter(self.ctx, pack_dev_ptr, pack_bytes, _s(stream)))

    def restore_packs(self, packs: Sequence[np.ndarray], stream=None, h2d_stream=None,
                      region_bytes: int = 0) -> None:
        """Streaming restore of host-resident packs, in order (base image then
        deltas): H2D through two cache regions + scatter (pos_restore_packs)."""
        n = len(packs)
        arrs = [np.ascontiguousarray(p.view(np.uint8)) for p in packs]
        ptrs = (C.c_void_p * max(n, 1))(*[a.ctypes.data for a in arrs])
        sizes = np.array([a.nbytes for a in arrs], dtype=np.uint64)
        check(lib().pos_restore_packs(self.ctx, ptrs, sizes.ctypes.data, n, _s(h2d_stream), _s(stream),
                                      region_bytes))

    # ---- restore from a POSI image (read_image + materialize)
    def restore_image(self, data: bytes, stream=None) -> tuple[int, int]:
        """Returns (records loaded, recompute records left to replay)."""
        buf = np.frombuffer(bytes(data), np.uint8)
        off, nl, nr = C.c_uint64(0), C.c_uint32(0), C.c_uint32(0)
        rc = lib().pos_image_restore(self.ctx, buf.ctypes.data if buf.size else None, buf.size, _s(stream),
                                     C.byref(off), C.byref(nl), C.byref(nr))
        if rc != 0:
            err = _lib.error_from(rc)
            err.offset = off.value
            raise err
        return nl.value, nr.value

    # ---- on-demand restore of a flat host image (restore / gate_restore, cr.hpp:167-204, 1043-1143)
    def restore_image_begin(self, hosts: Sequence[Optional[np.ndarray]], order: Sequence[int] = (),
                            slice_bytes: int = 0, h2d_stream=None) -> None:
        """hosts[i] None: buffer i is a Recompute record (regenerated by the
        replay; see restore_replayed)."""
        arrs = [None if h is None else np.ascontiguousarray(h).view(np.uint8).reshape(-1) for h in hosts]
        n = len(arrs)
        ptrs = (C.c_void_p * max(n, 1))(*[a.ctypes.data if a is not None else None for a in arrs])
        sizes = np.array([a.size if a is not None else 0 for a in arrs], dtype=np.uint64)
        order_a = np.array(list(order), dtype=np.uint64)
        self._restore_keep = arrs
        check(lib().pos_restore_image_begin(self.ctx, ptrs, sizes.ctypes.data, n,
                                            order_a.ctypes.data if order_a.size else None, order_a.size,
                                            slice_bytes, _s(h2d_stream)))

    def restore_replayed(self, handle: int, stream=None) -> None:
        """buffer_ready for a Recompute buffer (cr.hpp:1105-1119): its writer
        is enqueued on `stream`."""
        check(lib().pos_restore_replayed(self.ctx, handle, _s(stream)))

    def restore_want(self, handle: int) -> None:
        check(lib().pos_restore_want(self.ctx, handle))

    def restore_gate(self, handle: int, stream=None) -> None:
        check(lib().pos_restore_gate(self.ctx, handle, _s(stream)))

    def restore_ready(self, handle: int) -> bool:
        r = C.c_int(0)
        check(lib().pos_restore_ready(self.ctx, handle, C.byref(r)))
        return bool(r.value)

    def restore_image_wait(self) -> None:
        check(lib().pos_restore_image_wait(self.ctx))
        self._restore_keep = None

    # ---- timing
    def event_record(self, slot: int, stream=None) -> None:
        check(lib().pos_event_record(self.ctx, slot, _s(stream)))

    def event_elapsed(self, a: int, b: int) -> float:
        ms = C.c_float(0)
        check(lib().pos_event_elapsed(self.ctx, a, b, C.byref(ms)))
        return ms.value

    def stamp(self, slot: int, stream=None) -> None:
        """globaltimer stamp in stream order (pos_stamp)."""
        check(lib().pos_stamp(self.ctx, slot, _s(stream)))

    def stamp_elapsed(self, a: int, b: int) -> float:
        ms = C.c_float(0)
        check(lib().pos_stamp_elapsed(self.ctx, a, b, C.byref(ms)))
        return ms.value

    def stream_wait_event(self, slot: int, stream=None) -> None:
        check(lib().pos_stream_wait_event(self.ctx, slot, _s(stream)))

    def timeline(self, slot: int = 0) -> dict:
        """ms from event `slot` to each internal timer's begin/end."""
        out = (C.c_float * 14)()
        check(lib().pos_timeline(self.ctx, slot, out))
        names = ["hash", "combine", "scan", "copy", "delta", "scatter", "d2h"]
        return {n: (round(out[2 * i], 4), round(out[2 * i + 1], 4)) for i, n in enumerate(names) if out[2 * i] >= 0}

    def kernel_ms(self, which: str) -> float:
        ms = C.c_float(0)
        check(lib().pos_last_kernel_ms(self.ctx, which.encode(), C.byref(ms)))
        return ms.value

    @property
    def launches(self) -> int:
        n = C.c_uint64(0)
        check(lib().pos_launch_count(self.ctx, C.byref(n)))
        return n.value


# ---------------------------------------------------------------------------
# POSI image (image.hpp:136-207)

@dataclass
class GpuBufferRec:
    handle: int
    kind: int = 0  # 0 Inline, 1 DedupRef, 2 Recompute
    inline_bytes: Optional[np.ndarray] = None
    dedup_first_page: int = 0
    dedup_page_count: int = 0
    dedup_offset: int = 0
    dedup_crc: int = 0
    recompute_nodes: list = field(default_factory=list)


@dataclass
class CheckpointImage:
    page_size: int = 4096
    host_pages: list = field(default_factory=list)  # [(index, bytes)]
    gpu_records: list = field(default_factory=list)
    dag_bytes: bytes = b""
    stream_ids: list = field(default_factory=list)
    allocs: list = field(default_factory=list)  # [(handle, base, size)]
    cursor: int = 0
    next_handle: int = 1
    next_base: int = kDeviceAddrBase


def read_image_check(data: bytes) -> int:
    """read_image's validation (image.hpp:209-361) on the host: 0 if valid,
    else raises CorruptImageError whose .offset is the reference's offset."""
    buf = np.frombuffer(bytes(data), np.uint8)
    off = C.c_uint64(0)
    rc = lib().pos_image_check(buf.ctypes.data if buf.size else None, buf.size, C.byref(off))
    if rc != 0:
        err = _lib.error_from(rc)
        err.offset = off.value
        raise err
    return 0


@dataclass
class FinalizeBuf:
    """finalize_image's per-buffer inputs (cr.hpp:715-746): the captured bytes
    and what the session decided about the buffer."""
    handle: int
    base: int
    size: int
    inline_bytes: Optional[np.ndarray] = None  # captured_[h]
    upstream: Optional[tuple] = None  # dedup_snapshot_: (host_addr, len, crc)
    dedup_ok: Optional[bool] = None  # None: the engine's device O1 verdict
    dirty: bool = False
    recompute_eligible: bool = False
    recompute_nodes: list = field(default_factory=list)  # pending_writers(h)
    precopy_survived: bool = False


METRIC_KEYS = ("bytes_precopy", "bytes_dirty", "bytes_dedup_saved", "bytes_recompute_saved", "image_bytes",
               "image_file_bytes", "dirty_count", "retention_dirty_count", "retention", "n_inline", "n_dedup",
               "n_recompute")


def _image_desc(img: CheckpointImage, keep: list, with_records: bool = True):
    pages = (_lib.pos_image_page * max(len(img.host_pages), 1))()
    for i, (idx, data) in enumerate(img.host_pages):
        a = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8))
        if a.nbytes != img.page_size:
            raise SimError(_lib.CODES["InvariantViolation"], "host page size mismatch")
        keep.append(a)
        pages[i].index, pages[i].bytes = idx, a.ctypes.data
    keep.append(pages)
    streams = np.array(img.stream_ids, dtype=np.uint64)
    dag = np.frombuffer(img.dag_bytes, dtype=np.uint8) if img.dag_bytes else np.zeros(0, np.uint8)
    keep += [streams, dag]
    d = _lib.pos_image_desc()
    d.page_size = img.page_size
    d.pages, d.n_pages = C.cast(pages, C.c_void_p), len(img.host_pages)
    d.stream_ids, d.n_streams = (streams.ctypes.data if streams.size else None), streams.size
    d.cursor, d.next_handle, d.next_base = img.cursor, img.next_handle, img.next_base
    d.dag_bytes, d.dag_len = (dag.ctypes.data if dag.size else None), dag.size
    return d


def finalize_image(host_side: CheckpointImage, bufs: Sequence[FinalizeBuf], engine=None) -> tuple[bytes, dict]:
    """finalize_image (cr.hpp:680-764) through pos_finalize_image: record kinds,
    dedup_consistent over the image's host pages, the POSI bytes and the
    session metrics.  host_side supplies the host pages, meta and DAG bytes."""
    keep: list = []
    d = _image_desc(host_side, keep)
    arr = (_lib.pos_finalize_buf * max(len(bufs), 1))()
    for i, b in enumerate(bufs):
        f = arr[i]
        f.handle, f.base, f.size = b.handle, b.base, b.size
        if b.inline_bytes is not None:
            a = np.ascontiguousarray(np.asarray(b.inline_bytes, dtype=np.uint8).ravel())
            keep.append(a)
            f.inline_bytes = a.ctypes.data
        if b.upstream is not None:
            f.up_host_addr, f.up_len, f.up_crc = b.upstream
            f.has_upstream = 1
        f.dedup_ok = -1 if b.dedup_ok is None else int(bool(b.dedup_ok))
        f.dirty, f.recompute_eligible = int(b.dirty), int(b.recompute_eligible)
        f.precopy_survived = int(b.precopy_survived)
        if b.recompute_nodes:
            a = np.array(b.recompute_nodes, dtype=np.uint64)
            keep.append(a)
            f.recompute_nodes, f.n_recompute = a.ctypes.data, a.size
    ctx = engine.ctx if engine is not None else None
    size = C.c_uint64(0)
    m = _lib.pos_metrics()
    check(lib().pos_finalize_image(ctx, C.byref(d), arr, len(bufs), None, 0, C.byref(size), C.byref(m)))
    out = np.empty(size.value, dtype=np.uint8)
    check(lib().pos_finalize_image(ctx, C.byref(d), arr, len(bufs), out.ctypes.data, out.nbytes, C.byref(size),
                                   C.byref(m)))
    return out.tobytes(), {k: int(getattr(m, k)) for k in METRIC_KEYS}


def write_image(img: CheckpointImage, out: Optional[np.ndarray] = None):
    """write_image (image.hpp:136-207) through pos_image_write: the POSI bytes,
    or -- with `out` (a uint8 array at least that large) -- written into
    `out` without a copy, returning the image size."""
    keep = []
    pages = (_lib.pos_image_page * max(len(img.host_pages), 1))()
    for i, (idx, data) in enumerate(img.host_pages):
        a = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8))
        if a.nbytes != img.page_size:
            raise SimError(_lib.CODES["InvariantViolation"], "host page size mismatch")
        keep.append(a)
        pages[i].index, pages[i].bytes = idx, a.ctypes.data
    recs = (_lib.pos_image_rec * max(len(img.gpu_records), 1))()
    for i, r in enumerate(img.gpu_records):
        recs[i].handle, recs[i].kind = r.handle, r.kind
        if r.kind == 0:
            a = np.ascontiguousarray(np.asarray(r.inline_bytes, dtype=np.uint8).ravel())
            keep.append(a)
            recs[i].inline_bytes, recs[i].inline_len = a.ctypes.data, a.nbytes
        recs[i].dedup_first_page = r.dedup_first_page
        recs[i].dedup_page_count = r.dedup_page_count
        recs[i].dedup_offset = r.dedup_offset
        recs[i].dedup_crc = r.dedup_crc
        if r.recompute_nodes:
            a = np.array(r.recompute_nodes, dtype=np.uint64)
            keep.append(a)
            recs[i].recompute, recs[i].n_recompute = a.ctypes.data, a.size
    allocs = (_lib.pos_image_alloc * max(len(img.allocs), 1))(*[_lib.pos_image_alloc(*a) for a in img.allocs])
    streams = np.array(img.stream_ids, dtype=np.uint64)
    dag = np.frombuffer(img.dag_bytes, dtype=np.uint8) if img.dag_bytes else np.zeros(0, np.uint8)
    d = _lib.pos_image_desc()
    d.page_size = img.page_size
    d.pages, d.n_pages = C.cast(pages, C.c_void_p), len(img.host_pages)
    d.recs, d.n_recs = C.cast(recs, C.c_void_p), len(img.gpu_records)
    d.allocs, d.n_allocs = C.cast(allocs, C.c_void_p), len(img.allocs)
    d.stream_ids, d.n_streams = (streams.ctypes.data if streams.size else None), streams.size
    d.cursor, d.next_handle, d.next_base = img.cursor, img.next_handle, img.next_base
    d.dag_bytes, d.dag_len = (dag.ctypes.data if dag.size else None), dag.size
    size = C.c_uint64(0)
    if out is not None:
        check(lib().pos_image_write(C.byref(d), out.ctypes.data, out.nbytes, C.byref(size)))
        return size.value
    check(lib().pos_image_write(C.byref(d), None, 0, C.byref(size)))
    buf = np.empty(size.value, dtype=np.uint8)
    check(lib().pos_image_write(C.byref(d), buf.ctypes.data, buf.nbytes, C.byref(size)))
    return buf.tobytes()
