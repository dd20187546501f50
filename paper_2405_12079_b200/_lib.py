"""ctypes binding of libposdump.so (the C ABI declared in include/posdump.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  Importing this module without it raises: there is no CPU
fallback for the dump path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libposdump.so")

# Errc (include/gpucrsim/errors.hpp:9-25), POS_E_<Errc> = 1 + index.
ERRC = [
    "PastTime", "Livelock", "OutOfDeviceMemory", "InvalidLocator", "UseAfterFree",
    "FreedBuffer", "BadState", "PendingKernels", "UnknownApi", "InvalidArgument",
    "CorruptDag", "CorruptImage", "InvariantViolation", "StagingExhausted", "OracleMismatch",
]
POS_OK = 0
POS_E_CUDA = 64
POS_E_NO_DEVICE = 65
CODES = {name: i + 1 for i, name in enumerate(ERRC)}


class SimError(RuntimeError):
    """Mirror of gpucrsim::SimError (errors.hpp:48-56): carries the Errc name."""

    def __init__(self, code: int, what: str):
        self.code = code
        self.errc = ERRC[code - 1] if 1 <= code <= len(ERRC) else (
            "CudaError" if code == POS_E_CUDA else "NoDevice" if code == POS_E_NO_DEVICE else "Unknown")
        super().__init__(f"{self.errc}: {what}")


class CorruptImageError(SimError):
    """Mirror of gpucrsim::CorruptImageError (errors.hpp:59-68)."""


class NoDeviceError(SimError):
    pass


class pos_config(C.Structure):
    _fields_ = [("chunk_size", C.c_uint64), ("page_size", C.c_uint64),
                ("cache_capacity", C.c_uint64), ("staging_fraction", C.c_double),
                ("device", C.c_int32), ("dedup", C.c_int32),
                ("dirty_threshold_frac", C.c_double), ("trust_written_bit", C.c_int32), ("pad", C.c_int32)]


class pos_buffer_desc(C.Structure):
    _fields_ = [("handle", C.c_uint64), ("dev_ptr", C.c_uint64), ("size", C.c_uint64),
                ("has_upstream", C.c_uint32), ("upstream_crc", C.c_uint32),
                ("host_untouched", C.c_uint32), ("written_since_ckpt", C.c_uint32)]


class pos_image_rec(C.Structure):
    _fields_ = [("handle", C.c_uint64), ("kind", C.c_uint32), ("n_recompute", C.c_uint32),
                ("inline_bytes", C.c_void_p), ("inline_len", C.c_uint64),
                ("dedup_first_page", C.c_uint64), ("dedup_page_count", C.c_uint32),
                ("dedup_offset", C.c_uint32), ("dedup_crc", C.c_uint32), ("reserved", C.c_uint32),
                ("recompute", C.c_void_p)]


class pos_image_alloc(C.Structure):
    _fields_ = [("handle", C.c_uint64), ("base", C.c_uint64), ("size", C.c_uint64)]


class pos_image_page(C.Structure):
    _fields_ = [("index", C.c_uint64), ("bytes", C.c_void_p)]


class pos_image_desc(C.Structure):
    _fields_ = [("page_size", C.c_uint64),
                ("pages", C.c_void_p), ("n_pages", C.c_uint32),
                ("recs", C.c_void_p), ("n_recs", C.c_uint32),
                ("allocs", C.c_void_p), ("n_allocs", C.c_uint32),
                ("stream_ids", C.c_void_p), ("n_streams", C.c_uint32),
                ("cursor", C.c_uint64), ("next_handle", C.c_uint64), ("next_base", C.c_uint64),
                ("dag_bytes", C.c_void_p), ("dag_len", C.c_uint64)]


class pos_finalize_buf(C.Structure):
    _fields_ = [("handle", C.c_uint64), ("base", C.c_uint64), ("size", C.c_uint64),
                ("inline_bytes", C.c_void_p), ("up_host_addr", C.c_uint64), ("up_len", C.c_uint64),
                ("up_crc", C.c_uint32), ("has_upstream", C.c_uint32), ("dedup_ok", C.c_int32),
                ("dirty", C.c_uint32), ("recompute_eligible", C.c_uint32), ("n_recompute", C.c_uint32),
                ("recompute_nodes", C.c_void_p), ("precopy_survived", C.c_uint32), ("pad", C.c_uint32)]


class pos_metrics(C.Structure):
    _fields_ = [("bytes_precopy", C.c_uint64), ("bytes_dirty", C.c_uint64), ("bytes_dedup_saved", C.c_uint64),
                ("bytes_recompute_saved", C.c_uint64), ("image_bytes", C.c_uint64),
                ("image_file_bytes", C.c_uint64), ("dirty_count", C.c_uint64),
                ("retention_dirty_count", C.c_uint64), ("retention", C.c_uint32), ("n_inline", C.c_uint32),
                ("n_dedup", C.c_uint32), ("n_recompute", C.c_uint32)]


P = C.c_void_p
U64 = C.c_uint64
U32 = C.c_uint32
I32 = C.c_int
PU64 = C.POINTER(C.c_uint64)
PU32 = C.POINTER(C.c_uint32)
PU8 = C.POINTER(C.c_uint8)

# name -> (argtypes); every function returns int unless listed in _RESTYPE.
SIGNATURES = {
    "pos_strerror": [I32],
    "pos_last_error": [],
    "pos_abi_version": [],
    "pos_ctx_create": [C.POINTER(pos_config), C.POINTER(P)],
    "pos_ctx_destroy": [P],
    "pos_register_buffers": [P, C.POINTER(pos_buffer_desc), U32],
    "pos_update_buffer_set": [P, C.POINTER(pos_buffer_desc), U32],
    "pos_update_buffer": [P, C.POINTER(pos_buffer_desc)],
    "pos_num_chunks": [P, PU64],
    "pos_hash_chunks": [P, P],
    "pos_commit_epoch": [P],
    "pos_set_target_fresh": [P, I32],
    "pos_read_digests": [P, P, U64, P],
    "pos_read_flags": [P, P, U64, P],
    "pos_read_bitmap": [P, P, U64, P],
    "pos_buffer_crc": [P, P],
    "pos_read_buffer_crcs": [P, P, P, U32, P],
    "pos_record_dirty": [P, P, U32],
    "pos_clear_dirty": [P],
    "pos_compact": [P, I32, P, PU64],
    "pos_precopy": [P, I32, P],
    "pos_precopy_size": [P, PU64],
    "pos_precopy_pipelined": [P, I32, U32, P, P, P, U64, P, P, P],
    "pos_precopy_stream": [P, I32, P, P, U64, P, P, PU64, PU32],
    "pos_register_image": [P, P, P, U32],
    "pos_image_check": [P, U64, PU64],
    "pos_image_restore": [P, P, U64, P, PU64, PU32, PU32],
    "pos_peer_cache_attach": [P, I32, U64],
    "pos_peer_cache_stats": [P, C.POINTER(C.c_float), C.POINTER(C.c_float)],
    "pos_h2d_provenance": [P, U64, P, U64, I32, P],
    "pos_read_upstream": [P, U64, PU32, PU32],
    "pos_precopy_direct": [P, I32, U32, P, P],
    "pos_precopy_direct_result": [P, PU64, PU64, PU64],
    "pos_delta_drain": [P, P],
    "pos_delta_copy": [P, P, PU64, PU64],
    "pos_stage_buffers": [P, P, U32, P, PU64, PU64],
    "pos_delta_copy_ex": [P, P, I32, PU64, PU64],
    "pos_final_stop": [P, P, I32, I32, PU64, PU64],
    "pos_delta_prepare": [P, P, PU64, PU64],
    "pos_d2h_async": [P, P, U64, U64, U64, P],
    "pos_cache_info": [P, PU64, PU64],
    "pos_scatter": [P, U64, U64, P],
    "pos_restore_packs": [P, P, P, U32, P, P, U64],
    "pos_restore_image_begin": [P, P, P, U32, P, U32, U64, P],
    "pos_restore_want": [P, U64],
    "pos_restore_gate": [P, U64, P],
    "pos_restore_ready": [P, U64, C.POINTER(C.c_int)],
    "pos_restore_image_wait": [P],
    "pos_crc32": [U64, U64, PU32, P],
    "pos_crc32_update": [U32, U64, U64, PU32, P],
    "pos_fill": [U64, U64, U64, P],
    "pos_fill_batch": [P, U32, P],
    "pos_delta_pregather": [P, P, U32, P, P],
    "pos_stream_begin_capture": [P],
    "pos_stream_end_capture": [P, C.POINTER(C.c_void_p)],
    "pos_graph_launch": [P, P],
    "pos_graph_destroy": [P],
    "pos_event_record": [P, U32, P],
    "pos_event_elapsed": [P, U32, U32, C.POINTER(C.c_float)],
    "pos_stream_wait_event": [P, U32, P],
    "pos_stamp": [P, U32, P],
    "pos_stamp_elapsed": [P, U32, U32, C.POINTER(C.c_float)],
    "pos_timeline": [P, U32, P],
    "pos_launch_count": [P, PU64],
    "pos_last_kernel_ms": [P, C.c_char_p, C.POINTER(C.c_float)],
    "pos_image_write": [C.POINTER(pos_image_desc), P, U64, PU64],
    "pos_app_copy": [P, U64, U64, U64, I32, P],
    "pos_set_hash_sms": [P, U32],
    "pos_set_o2_digest2": [P, I32],
    "pos_restore_replayed": [P, U64, P],
    "pos_set_host_leg": [P, U64, U32],
    "pos_host_leg_stats": [P, PU64, PU64, PU64],
    "pos_finalize_image": [P, C.POINTER(pos_image_desc), P, U32, P, U64, PU64, C.POINTER(pos_metrics)],
    "pos_get_metrics": [P, C.POINTER(pos_metrics)],
    "pos_set_stop_exclusions": [P, P, U32],
    "pos_pack_apply_host": [P, U64, P, P, P, U32, U32],
    "pos_device_count": [C.POINTER(C.c_int)],
    "pos_set_device": [I32],
    "pos_dev_malloc": [U64, PU64],
    "pos_dev_free": [U64],
    "pos_host_malloc_pinned": [U64, C.POINTER(P)],
    "pos_host_image_alloc": [U64, U32, C.POINTER(P)],
    "pos_host_image_free": [P],
    "pos_host_free_pinned": [P],
    "pos_memcpy": [U64, U64, U64, I32, P],
    "pos_memset": [U64, I32, U64, P],
    "pos_stream_create": [C.POINTER(P)],
    "pos_stream_create_prio": [I32, C.POINTER(P)],
    "pos_stream_destroy": [P],
    "pos_stream_sync": [P],
    "pos_device_sync": [],
    "pos_stream_wait": [P, P],
}
# void (*pos_pack_sink)(void* user, const uint8_t* pack, uint64_t bytes, uint32_t index)
PACK_SINK = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_uint8), C.c_uint64, C.c_uint32)

_RESTYPE = {"pos_strerror": C.c_char_p, "pos_last_error": C.c_char_p}


def header_symbols(header_path: str | None = None) -> list[str]:
    """Every function declared in include/posdump.h."""
    import re
    if header_path is None:
        header_path = os.path.join(os.path.dirname(_HERE), "include", "posdump.h")
    text = open(header_path).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(pos_\w+)\(", text, re.M)))


_lib = None


def load() -> C.CDLL:
    """Load libposdump.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the dump path)")
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    _lib = lib
    return lib


def error_from(rc: int) -> SimError:
    """The exception for return code rc (with pos_last_error's message)."""
    msg = load().pos_last_error().decode(errors="replace")
    if rc == CODES["CorruptImage"]:
        return CorruptImageError(rc, msg)
    if rc == POS_E_NO_DEVICE:
        return NoDeviceError(rc, msg)
    return SimError(rc, msg)


def check(rc: int) -> None:
    if rc == POS_OK:
        return
    raise error_from(rc)
