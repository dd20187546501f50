"""finalize_image (cr.hpp:680-764) through the C ABI (pos_finalize_image),
host side: the record kinds (DedupRef / Recompute / Inline), the
dedup_consistent recheck over the image's host pages (cr.hpp:692-708), the
POSI bytes and CrMetrics, against the reference CrEngine on the same
session.  The inputs are the engine's OWN decisions at finalize (O1 verdict,
dirty_set_, recompute eligibility, pending writers, captured bytes --
ref_checkpoint_session); nothing is read from the reference's output image
except the host-side sections (host pages, DAG bytes, meta) that the CPU
side contributes.  The GPU-verdict / GPU-dump variant is in
test_gpu_parity.py."""
import pytest

import paper_2405_12079_b200 as pd
from oracle_ctypes import ref_session
from posi import read_posi

TRACES = [
    ("gpt2-infer-desk", 1, 3),    # inference: parameters H2D-loaded -> DedupRef records
    ("resnet-train-desk", 1, 3),  # training, DAG retention
    ("fuzz", 7, 3),
    ("fuzz", 8, 1),               # stop-the-world image
    ("ppo-train-desk", 2, 3),     # a Recompute record
]


def host_side(img: dict) -> pd.CheckpointImage:
    m = img["meta"]
    return pd.CheckpointImage(page_size=img["page_size"], host_pages=img["pages"], dag_bytes=bytes(img["dag"]),
                              stream_ids=m["streams"], cursor=m["cursor"], next_handle=m["next_handle"],
                              next_base=m["next_base"])


def finalize_bufs(sess: dict, dedup_from_device: bool = False) -> list:
    out = []
    for b in sess["bufs"]:
        out.append(pd.FinalizeBuf(
            handle=b["handle"], base=b["base"], size=b["size"],
            inline_bytes=memoryview(b["content"]),
            upstream=(b["up_host_addr"], b["up_len"], b["up_crc"]) if b["has_upstream"] else None,
            dedup_ok=None if dedup_from_device else b["dedup_ok"] == 1,
            dirty=b["dirty"], recompute_eligible=b["recompute_eligible"], recompute_nodes=b["pending"],
            precopy_survived=b["precopy_survived"]))
    return out


@pytest.mark.parametrize("profile,seed,mode", TRACES)
def test_finalize_reproduces_reference_image(ref, profile, seed, mode):
    sess = ref_session(ref, profile, seed, mode)
    img = read_posi(sess["image"])
    out, m = pd.finalize_image(host_side(img), finalize_bufs(sess))
    assert out == sess["image"]
    want = sess["metrics"]
    for k in ("bytes_precopy", "bytes_dedup_saved", "bytes_recompute_saved", "image_bytes", "image_file_bytes"):
        assert m[k] == want[k], k
    kinds = [r["kind"] for r in img["recs"]]
    assert (m["n_inline"], m["n_dedup"], m["n_recompute"]) == (kinds.count(0), kinds.count(1), kinds.count(2))
    if mode == 3:  # dirty-bit closure (tests/test_harness.cpp:99-112); bytes_dirty = the final stop's re-copies
        dirty = sum(b["size"] for b in sess["bufs"] if b["final_recopy"])
        assert dirty == want["bytes_dirty"]
        assert m["bytes_precopy"] + dirty + m["bytes_dedup_saved"] == sum(b["size"] for b in sess["bufs"])


def test_dedup_consistent_rejects_touched_host_pages(ref):
    """A DedupRef needs the Upstream crc to match the host pages as they land
    in the image (cr.hpp:692-708): flip one byte of a referenced page and
    the record becomes Inline; drop the page and it does too."""
    sess = ref_session(ref, "gpt2-infer-desk", 1, 3)
    img = read_posi(sess["image"])
    bufs = finalize_bufs(sess)
    dedup = [b for b in bufs if b.dedup_ok and not b.dirty]
    assert dedup
    victim = dedup[0]
    ps = img["page_size"]
    first = victim.upstream[0] // ps
    hs = host_side(img)
    pages = dict(hs.host_pages)
    flipped = bytearray(pages[first])
    flipped[victim.upstream[0] % ps] ^= 1
    hs.host_pages = [(i, bytes(flipped) if i == first else p) for i, p in hs.host_pages]
    out, m = pd.finalize_image(hs, bufs)
    rec = {r["handle"]: r for r in read_posi(out)["recs"]}
    assert rec[victim.handle]["kind"] == 0 and rec[victim.handle]["inline"] == bytes(victim.inline_bytes)
    assert m["n_dedup"] == len(dedup) - 1
    hs.host_pages = [(i, p) for i, p in host_side(img).host_pages if i != first]
    out, m = pd.finalize_image(hs, bufs)
    assert {r["handle"]: r for r in read_posi(out)["recs"]}[victim.handle]["kind"] == 0


def test_finalize_needs_a_context_for_device_verdicts(ref):
    sess = ref_session(ref, "fuzz", 8, 1)
    with pytest.raises(pd.SimError) as ei:
        pd.finalize_image(host_side(read_posi(sess["image"])), finalize_bufs(sess, dedup_from_device=True))
    assert ei.value.errc == "InvalidArgument"
