"""Generate tests/golden/*.json from the reference's OWN code (oracle/_ref,
compiled from /root/reference/proj/include by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The outputs are committed; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_ctypes import reference  # noqa: E402

ref = reference()
assert ref is not None, "build oracle/_ref first (make -C oracle)"


def mb(seed, n):
    out = np.empty(n, np.uint8)
    ref.ref_make_bytes(seed, out.ctypes.data, n)
    return out


def crc(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return ref.ref_crc32(a.ctypes.data, a.nbytes)


def digests(a, cs):
    return [crc(a[o:o + cs]) for o in range(0, a.size, cs)]


kat = {}
kat["crc32_strings"] = {s: f"{crc(np.frombuffer(s.encode(), np.uint8)):08x}"
                        for s in ["", "a", "abc", "123456789", "The quick brown fox jumps over the lazy dog"]}
kat["crc32_zero_byte"] = f"{crc(np.zeros(1, np.uint8)):08x}"
kat["crc32_update_split_123456789"] = f"{ref.ref_crc32_update(ref.ref_crc32(b'1234', 4), b'56789', 5):08x}"
kat["make_bytes_1_16"] = mb(1, 16).tobytes().hex()
kat["make_bytes_7_13"] = mb(7, 13).tobytes().hex()
kat["crc32_make_bytes_1_65536"] = f"{crc(mb(1, 65536)):08x}"
b = mb(2, 10000)
kat["make_bytes_2_10000"] = {"crc": f"{crc(b):08x}", "digests_4096": [f"{d:08x}" for d in digests(b, 4096)]}
c1 = {}
for i in (0, 63):
    v = mb(1000 + i, 16 << 20)
    c1[str(i)] = {"seed": 1000 + i, "whole": f"{crc(v):08x}", "chunk0": f"{crc(v[:65536]):08x}",
                  "chunk255": f"{crc(v[255 * 65536:]):08x}"}
    d = np.array(digests(v, 65536), np.uint32)
    c1[str(i)]["digests_crc"] = f"{crc(d.view(np.uint8)):08x}"  # checksum of checksums
kat["c1_buffers"] = c1
# odd chunk sizes and tails (buffer.hpp:46-49)
odd = []
for seed, n, cs in [(3, 1, 7), (4, 100, 7), (5, 65537, 65536), (6, 200000, 1000), (8, 4096, 4096),
                    (9, 123457, 4093), (10, 70000, 16), (11, 1 << 20, 65536)]:
    a = mb(seed, n)
    odd.append({"seed": seed, "size": n, "chunk_size": cs, "crc": f"{crc(a):08x}",
                "digests_crc": f"{crc(np.array(digests(a, cs), np.uint32).view(np.uint8)):08x}",
                "first": [f"{d:08x}" for d in digests(a, cs)[:4]],
                "last": f"{digests(a, cs)[-1]:08x}"})
kat["odd_chunks"] = odd
geo = []
for size, cs in [(10000, 4096), (1, 65536), (65536, 65536), (65537, 65536), (16 << 20, 65536), (17, 7)]:
    n = ref.ref_chunk_geometry(size, cs, None)
    out = np.empty(n, np.uint64)
    ref.ref_chunk_geometry(size, cs, out.ctypes.data)
    geo.append({"size": size, "chunk_size": cs, "count": int(n), "first": int(out[0]), "last": int(out[-1])})
kat["geometry"] = geo
kat["mix64"] = {f"{a},{b}": f"{ref.ref_mix64(a, b):016x}" for a, b in [(1, 2), (0, 0), (5, 123456789), (2**64 - 1, 7)]}
kat["fnv1a_empty"] = f"{ref.ref_fnv1a(None, 0, 0xcbf29ce484222325):016x}"
kat["fnv1a_123456789"] = f"{ref.ref_fnv1a(b'123456789', 9, 0xcbf29ce484222325):016x}"
json.dump(kat, open(os.path.join(HERE, "kat.json"), "w"), indent=1, sort_keys=True)


# ---- POSI images written by the reference's write_image (image.hpp:136-207)
from oracle_ctypes import ref_image as _ref_image  # noqa: E402


def ref_image(desc):
    return _ref_image(ref, desc)


BASE = 0x7000_0000_0000
images = [
    {"name": "empty", "page_size": 4096, "pages": [], "recs": [], "allocs": [], "streams": [],
     "cursor": 0, "next_handle": 1, "next_base": BASE, "dag": ""},
    {"name": "inline_unsorted", "page_size": 256, "pages": [(9, 51), (2, 52)],
     "recs": [{"handle": 3, "kind": 0, "seed": 61, "len": 1000}, {"handle": 1, "kind": 0, "seed": 62, "len": 17}],
     "allocs": [(3, BASE + 256, 1000), (1, BASE, 17)], "streams": [2, 1], "cursor": 42,
     "next_handle": 4, "next_base": BASE + 2048, "dag": ""},
    {"name": "all_kinds", "page_size": 512, "pages": [(0, 71), (1, 72), (2, 73)],
     "recs": [{"handle": 5, "kind": 1, "first_page": 0, "page_count": 2, "offset": 12, "crc": 0xDEADBEEF},
              {"handle": 2, "kind": 2, "nodes": [7, 9, 11]},
              {"handle": 4, "kind": 0, "seed": 74, "len": 4096}],
     "allocs": [(2, BASE, 64), (4, BASE + 256, 4096), (5, BASE + 8192, 900)], "streams": [],
     "cursor": 7, "next_handle": 6, "next_base": BASE + 16384, "dag": "00112233445566778899"},
]
golden_images = []
for d in images:
    golden_images.append({"desc": d, "posi_hex": ref_image(d).hex()})
json.dump(golden_images, open(os.path.join(HERE, "images.json"), "w"), indent=1)
print("wrote", os.listdir(HERE))
