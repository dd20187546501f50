"""CPU, world_size 2 (gloo on 127.0.0.1): the N>1 plumbing of bench.py.

Each GPU checkpoints its own process's buffers (independent
units, no data-path collective); the only cross-rank traffic is the barrier
and the max-over-ranks of the step timings.  Covered here: all_max, the
barrier, the weak-scaling aggregate, and the reference arm under torchrun
(rank 0 alone runs and prints; the others exit 0).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.barrier(dist, rank)
    vals = bench.all_max(dist, [float(rank + 1), float(10 - rank), 0.5 * rank], rank)
    q.put((rank, vals))
    dist.destroy_process_group()


def _summary_worker(rank, world, port, q):
    """The GPU arm's rank logic with the engine stubbed out: each rank brings
    its own step / STW / e2e timings and host-link rate, rank_summary gives
    the job's max and every rank's row, aggregate_value the weak-scaling sum."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    step, stw, e2e, link = 2000.0 + 100 * rank, 0.4 - 0.1 * rank, 2100.0 + rank, 56.0 - rank
    m_step, m_stw, m_e2e, per_rank = bench.rank_summary(dist, rank, step, stw, e2e, link)
    q.put((rank, m_step, m_stw, m_e2e, per_rank, bench.aggregate_value(world, 120_000_000_000, m_step)))
    dist.destroy_process_group()


def test_rank_summary_over_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_summary_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {o[0]: o[1:] for o in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1]
    m_step, m_stw, m_e2e, per_rank, value = out[0]
    assert (m_step, m_stw, m_e2e) == (2100.0, 0.4, 2101.0)
    assert [r["rank"] for r in per_rank] == [0, 1]
    assert per_rank[1]["ms_per_step"] == 2100.0 and per_rank[1]["stw_ms"] == pytest.approx(0.3)
    assert per_rank[0]["host_link_gbps"] == 56.0 and per_rank[1]["host_link_gbps"] == 55.0
    assert value == pytest.approx(2 * 120.0 / 2.1)


def test_all_max_and_barrier_over_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1] == [2.0, 10.0, 0.5]


def test_weak_scaling_aggregate():
    sys.path.insert(0, ROOT)
    import bench
    # value = N * state bytes / max step time over ranks
    assert bench.aggregate_value(world=4, state_bytes=100_000_000, step_ms=1.25) == pytest.approx(320.0)


def test_reference_arm_under_torchrun(tmp_path):
    ref = os.path.join(ROOT, "oracle", "_ref", "libgpucrsim_ref.so")
    if not os.path.exists(ref):
        pytest.skip("oracle/_ref not built")
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3",
           "--ref-sample-bytes", "8000000"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0


def test_gpus_flag_relaunches_one_process_per_gpu(tmp_path):
    """`bench.py --gpus 2` outside torchrun re-executes itself as 2 ranks
    (torch.distributed.run on 127.0.0.1) instead of silently running one."""
    ref = os.path.join(ROOT, "oracle", "_ref", "libgpucrsim_ref.so")
    if not os.path.exists(ref):
        pytest.skip("oracle/_ref not built")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "1"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "3", "--ref-sample-bytes", "8000000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2
