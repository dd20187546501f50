"""B200-native buffer-dump hot path of the POS checkpoint engine (arXiv 2405.12079).

The product is ``libposdump.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/posdump.h``); this package is the host-side mirror of the reference's
interface for that path (see ``posdump.py``).
"""
from .posdump import (  # noqa: F401
    CheckpointImage, CorruptImageError, DeviceMemory, DumpEngine, GpuBuffer, GpuBufferRec,
    NoDeviceError, PinnedHost, SimConfig, SimError, Stream, Upstream, apply_pack_host, crc32,
    crc32_update, device_count, device_synchronize, fill_batch, fill_bytes, parse_pack,
    read_image_check, write_image, lib, check, FinalizeBuf, finalize_image,
)
