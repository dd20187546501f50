"""CPU: the bench's synthetic workloads have the shapes BASELINE.json names
and are deterministic per epoch."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_c1_shape_and_dirty_fraction():
    wl = bench.Workload("c1")
    assert wl.sizes == [16 << 20] * 64 and wl.total == 1 << 30
    w = wl.epoch_writes(3)
    assert len(w) == (1 << 30) // bench.CHUNK // 10  # 10 % of the chunks
    assert len({(h, o) for h, o, _, _ in w}) == len(w)  # distinct chunks
    assert all(n == bench.CHUNK and o % bench.CHUNK == 0 for _, o, n, _ in w)
    assert w == wl.epoch_writes(3) and w != wl.epoch_writes(4)


def test_c2_trace_is_the_reference_resnet_desk():
    wl = bench.Workload("c2")
    assert len(wl.sizes) == 224 and wl.total == 100_000_000
    assert len(wl.params) > 0 and wl.window(1)
    hs = {h for k in wl.window(1) for h, _ in k}
    assert hs and all(1 <= h <= 224 for h in hs)


@pytest.mark.parametrize("name,total", [("c3", 112_423_657_472), ("c4", 40_000_000_000),
                                        ("c5", 120_000_000_000)])
def test_large_states(name, total):
    wl = bench.Workload(name)
    assert wl.total == total
    w = wl.epoch_writes(1)
    if name == "c4":  # 256 sequences append one 32 KiB block per layer tensor
        assert wl.window(1) == []
        assert len(w) == 256 * 64 and all(n == 32768 for _, _, n, _ in w)
        assert sum(n for _, _, n, _ in w) / total < 0.02
    else:  # an optimizer step rewrites every tensor; its tail (>= 1 GiB) runs during the pre-copy
        win = {h for k in wl.window(1) for h, _ in k}
        assert win == wl.win and sum(wl.sizes[h - 1] for h in win) >= 1 << 30
        assert sum(wl.sizes[h - 1] for h in win) < 0.03 * total
        assert {h for h, _, _, _ in w}.isdisjoint(win)
        assert sum(n for _, _, n, _ in w) + sum(wl.sizes[h - 1] for h in win) == total
        assert wl.window(1) != wl.window(2)  # fresh bytes every step


def test_both_arms_print_the_same_config():
    """The driver compares the two arms' config dicts."""
    for name in ("c1", "c5"):
        wl = bench.Workload(name)
        assert bench.bench_config(wl, 1) == bench.bench_config(bench.Workload(name), 1)
        assert "workload" in bench.bench_config(wl, 1)


def test_gpus_flag_must_match_world(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    with pytest.raises(SystemExit) as ei:
        bench.main()
    assert "WORLD_SIZE" in str(ei.value)


def test_aggregate_value_is_whole_job():
    assert bench.aggregate_value(8, 100_000_000, 1.0) == pytest.approx(800.0)


def test_reference_cpu_breakdown():
    """The reference arm's per-function CPU timings run the reference's own
    code (oracle/_ref) on a small sample and report positive rates."""
    from oracle_ctypes import reference
    if reference() is None:
        pytest.skip("oracle/_ref not built")
    out = bench.cpu_breakdown(bench.Workload("c2"), 2, 2 << 20)
    assert set(out) >= {"crc32_per_chunk", "dump_loop_all_dirty", "write_image", "read_image"}
    assert all(v > 0 for v in out["crc32_per_chunk"].values())
    assert all(v > 0 for v in out["dump_loop_all_dirty"].values())
    assert out["write_image"] > 0 and out["read_image"] > 0
