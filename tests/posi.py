"""Minimal POSI v1 reader for tests (layout: image.hpp:18-39, read_image
image.hpp:209-361 without the cross-section validation)."""
import struct


def read_posi(b: bytes) -> dict:
    assert b[:4] == b"POSI"
    ver, flags, n_pages, n_recs = struct.unpack_from("<HHII", b, 4)
    page_size, host_len, gpu_len, dag_len, meta_len, _ = struct.unpack_from("<QQQQQQ", b, 16)
    pos = 64
    pages = []
    for _ in range(n_pages):
        (idx,) = struct.unpack_from("<Q", b, pos)
        pages.append((idx, b[pos + 8:pos + 8 + page_size]))
        pos += 8 + page_size
    recs = []
    for _ in range(n_recs):
        h, kind = struct.unpack_from("<QB", b, pos)
        pos += 9
        r = {"handle": h, "kind": kind}
        if kind == 0:
            (n,) = struct.unpack_from("<Q", b, pos)
            r["inline"] = b[pos + 8:pos + 8 + n]
            pos += 8 + n
        elif kind == 1:
            r["first_page"], r["page_count"], r["offset"], r["crc"] = struct.unpack_from("<QIII", b, pos)
            pos += 20
        else:
            (n,) = struct.unpack_from("<I", b, pos)
            r["nodes"] = list(struct.unpack_from(f"<{n}Q", b, pos + 4))
            pos += 4 + 8 * n
        recs.append(r)
    dag = b[pos:pos + dag_len]
    pos += dag_len
    meta = {"streams": [], "allocs": [], "cursor": 0, "next_handle": 1, "next_base": 0x7000_0000_0000}
    if meta_len:
        (ns,) = struct.unpack_from("<I", b, pos)
        meta["streams"] = list(struct.unpack_from(f"<{ns}Q", b, pos + 4))
        pos += 4 + 8 * ns
        (na,) = struct.unpack_from("<I", b, pos)
        pos += 4
        for _ in range(na):
            meta["allocs"].append(struct.unpack_from("<QQQ", b, pos))
            pos += 24
        meta["cursor"], meta["next_handle"], meta["next_base"] = struct.unpack_from("<QQQ", b, pos)
        pos += 24
    assert pos == len(b)
    return {"page_size": page_size, "pages": pages, "recs": recs, "dag": dag, "meta": meta}


def dedup_bytes(img: dict, r: dict, size: int) -> bytes:
    """dedup_content (image.hpp:364-376): the referenced host bytes."""
    pages = dict(img["pages"])
    ps = img["page_size"]
    out = bytearray()
    for i in range(size):
        at = r["offset"] + i
        out.append(pages[r["first_page"] + at // ps][at % ps])
    return bytes(out)
