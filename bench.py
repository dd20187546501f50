#!/usr/bin/env python3
"""Benchmark of the B200 buffer-dump hot path (POS checkpoint engine).

One step = one incremental dirty-bit checkpoint of the workload's buffer set
(BASELINE.json metric "checkpoint dump GB/s per GPU (hash+compact+D2H) and
stop-the-world ms"), default mode `direct`:

  ckpt stream : per wave of whole buffers: k_hash_chunks (O2 digests + dirty
                flags) -> k_buffer_crc (O1) -> k_scan_tiles (ballot/prefix-sum
                compaction of the shipped chunks into copy runs + a POSD index
                pack in the on-device cache) ... [final stop: the application
                drained AND the pre-copy complete] -> event, TMA bulk gather of
                the DAG-dirty buffers into the cache (STW delta-copy), event
                -> hash of the gathered copy
  copy stream : copy-engine copies of each wave's runs, live buffers ->
                pinned host image (the checkpoint target's captured_), then the
                delta's runs, cache -> image
  app stream  : the application's kernels of the pre-copy window (their
                write sets are the DAG dirty set), concurrent with the dump

value = checkpointed state bytes / step time (device time, CUDA events:
first dump operation -> last byte in the host image), aggregated over ranks
as sum(bytes) / max(time).  stw_ms = the final stop's window.  Inputs are
resident in HBM when the timed region starts; L2 is flushed (a 256 MiB
memset) before every step.

Workloads (--workload; BASELINE.json configs): c5 (default, configs[4], the
metric's own configuration): a 120 GB per-GPU training state, 960 x 125 MB,
every tensor rewritten per optimizer step, the step's last 1 GB written
during the pre-copy; c1 (configs[0]): 64 x 16 MiB, 10% random chunk rewrites;
c2 (configs[1]): the reference's own gen_workload trace of resnet-train-desk
rescaled to ~100 MB (tests/golden/c2_resnet_trace.json); c3 (configs[2]):
Llama-3-8B bf16 + fp32 Adam state, 112 GB; c4 (configs[3]): 40 GB paged KV
cache, append-only, then restore + delta replay.  Large states (c3-c5) are
verified end to end: the device state is dropped, restored from the host
image, and every chunk digest must equal the checkpoint's.

--gpus N: one process per GPU (re-executed under torch.distributed.run when
not already launched that way); each rank checkpoints its own state, no
collective on the data path ("scaling": "weak").

--impl reference times the reference's own CPU implementation of the path
(oracle/_ref: gpucrsim's crc32 per chunk + chunk_copied capture, compiled
from /root/reference) on all host cores, on a >= 1 GiB prefix of the same
state, same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CHUNK = 65536
METRIC = "checkpoint dump GB/s per GPU (hash+compact+D2H) and stop-the-world ms"
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (GB/s)


# ---------------------------------------------------------------------------
# workloads

def splitmix(seed: int, k: int) -> int:
    m = (1 << 64) - 1
    z = (seed + (k + 1) * 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def mix64(a: int, b: int) -> int:  # rng.hpp:35-40
    m = (1 << 64) - 1
    z = a ^ ((b + 0x9E3779B97F4A7C15 + ((a << 6) & m) + (a >> 2)) & m)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


class Workload:
    """sizes[i] belongs to handle i+1.  epoch_writes(e) -> [(handle, off, len, seed)]
    applied untimed before checkpoint e; window(e) -> kernels [(writes, seeds)]
    that run on the app stream during the pre-copy of checkpoint e."""

    def __init__(self, name: str):
        self.name = name
        if name == "c2":
            t = json.load(open(os.path.join(ROOT, "tests", "golden", "c2_resnet_trace.json")))
            self.sizes = t["sizes"]
            self.params = set(t["params"])
            self.phases = t["phases"]
            self.desc = ("ResNet-50 training buffer trace (gpucrsim gen_workload resnet-train-desk, "
                         f"{len(self.sizes)} buffers, {sum(self.sizes)} B, {sum(len(p) for p in self.phases)} kernels)")
        elif name == "c3":
            # Llama-3-8B training state: per-tensor bf16 params + fp32 master,
            # Adam m and v (4 buffers per parameter tensor), ~112 GB.
            V, H, I, L, KV = 128256, 4096, 14336, 32, 1024
            tensors = [V * H]
            for _ in range(L):
                tensors += [H * H, H * KV, H * KV, H * H, H * I, H * I, I * H, H, H]
            tensors += [H, H * V]
            self.sizes = [2 * t for t in tensors] + [4 * t for t in tensors] * 3
            self.params = set()
            self.phases = []
            self.desc = (f"Llama-3 8B bf16 training state (params bf16 + fp32 master + Adam m,v; "
                         f"{len(self.sizes)} buffers, {sum(self.sizes)} B), Adam step rewrites all; "
                         "the step's last >= 1 GB is written during the pre-copy")
        elif name == "c5":
            # config 5: a 120 GB per-GPU training state (960 tensors of 125 MB),
            # every tensor rewritten per step, checkpointed concurrently on
            # every rank through the NVLink peer-GPU cache (next GPU's HBM)
            self.sizes = [125_000_000] * 960
            self.params = set()
            self.phases = []
            self.desc = ("120 GB per-GPU training state (960 x 125 MB tensors), every tensor rewritten per "
                         "optimizer step; the step's last 1 GB is written during the pre-copy")
        elif name == "c4":
            # LLM inference KV cache: 32 layers x {K, V} paged tensors, 40 GB;
            # 16-token blocks of 8 KV heads x 128 dims bf16 = 32 KiB per block
            # per tensor; 256 sequences each append one block per epoch (one
            # 16-token decode burst) at ring-allocated block slots.
            self.sizes = [625_000_000] * 64
            self.params = set()
            self.phases = []
            self.block, self.seqs = 32768, 256
            self.nblocks = self.sizes[0] // self.block
            self.desc = ("LLM inference KV cache (32 layers x K/V paged, 40 GB, 32 KiB blocks), 256 sequences "
                         "append one block each per epoch (1.3% of the state)")
        elif name == "c1":
            self.sizes = [16 << 20] * 64
            self.params = set()
            self.phases = []
            self.desc = "synthetic single process: 1 GiB across 64 buffers, 64 KiB chunks, 10% random dirty per epoch"
        else:
            raise SystemExit(f"unknown workload {name}")
        self.total = sum(self.sizes)
        self.n_iter = max(1, len(self.phases) // 2)
        # Training states (c3/c5): the checkpoint is triggered while the tail
        # of the optimizer step is still running -- the last tensors (>= 1 GB)
        # are written by application kernels DURING the pre-copy.  They are
        # in the DAG from submission, so the pre-copy leaves them to the
        # stop-the-world delta-copy (record_dirty, cr.hpp:901-931; at_final_stop,
        # cr.hpp:599-621).
        self.win = set()
        if name in ("c3", "c5"):
            acc = 0
            for h in range(len(self.sizes), 0, -1):
                if acc >= 1 << 30:
                    break
                self.win.add(h)
                acc += self.sizes[h - 1]

    def epoch_writes(self, e: int):
        if self.name == "c4":  # append-only: block slots (e * S + s) mod nblocks
            out = []
            for s in range(self.seqs):
                blk = (e * self.seqs + s) % self.nblocks
                for h in range(1, len(self.sizes) + 1):
                    out.append((h, blk * self.block, self.block, mix64(mix64(e, s), h)))
            return out
        if self.name in ("c3", "c5"):  # the optimizer step rewrites every tensor (its tail: window())
            return [(h, 0, n, mix64(e, h)) for h, n in enumerate(self.sizes, start=1) if h not in self.win]
        if self.name == "c1":
            nch = self.total // CHUNK
            rng = np.random.default_rng(e)
            picks = rng.choice(nch, nch // 10, replace=False)
            return [(int(g) // 256 + 1, (int(g) % 256) * CHUNK, CHUNK, mix64(e, int(g))) for g in picks]
        # one training iteration: compute phase + optimizer phase, whole-buffer
        # rewrites of every kernel's true write set (apply_kernel_effect,
        # process.hpp:244-261)
        it = e % self.n_iter
        out = []
        for ph in self.phases[2 * it:2 * it + 2]:
            for k, (_, _, writes) in enumerate(ph):
                for h in writes:
                    out.append((h, 0, self.sizes[h - 1], mix64(mix64(e, k), h)))
        return out

    def window(self, e: int):
        """Kernels of the next iteration's compute phase (stream 1 and 2
        kernels are serialised on one app stream)."""
        if self.name in ("c3", "c5"):  # the optimizer step's tail: one kernel per tensor
            return [[(h, mix64(mix64(e + 1000003, h), h))] for h in sorted(self.win)]
        if self.name in ("c1", "c4"):
            return []
        it = (e + 1) % self.n_iter
        ph = self.phases[2 * it]
        return [[(h, mix64(mix64(e + 1000003, k), h)) for h in writes] for k, (_, _, writes) in enumerate(ph)]


# ---------------------------------------------------------------------------
# helpers

_T0 = time.time()


def log(msg: str) -> None:
    """Progress on stderr (the driver reads only stdout's JSON line)."""
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)

def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        nv = self.nv
        names = {
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup():
    """One process per GPU: (world, rank, device, dist).  NCCL carries only
    the barriers and the max of the timings.  Fewer GPUs than ranks (a
    plumbing check on a 1-GPU box) maps ranks onto GPUs round-robin and uses
    gloo, since NCCL refuses two ranks on one device."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        ngpu = torch.cuda.device_count()
        backend = "nccl" if ngpu >= world else "gloo"
        if ngpu:
            local = local % ngpu
        if backend == "nccl":
            torch.cuda.set_device(local)
        else:
            log(f"rank {rank}: {ngpu} GPU(s) for {world} ranks -> GPU {local}, gloo (plumbing check only)")
        dist.init_process_group(backend)
    return world, rank, local, dist


def all_max(dist, vals, device):
    if dist is None:
        return vals
    import torch
    dev = f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().tolist()


def gather_rows(dist, row, device):
    """Every rank's row of floats, on every rank (all_gather; NCCL or gloo)."""
    if dist is None:
        return [list(row)]
    import torch
    dev = f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(row, dtype=torch.float64, device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.cpu().tolist() for o in out]


def rank_summary(dist, device, step_ms, stw_ms, e2e_ms, link_gbps):
    """Max over ranks of the timings (the job's step) and each rank's own row:
    step, STW window and host-link GB/s of every GPU (each rank
    checkpoints its own state over its own link)."""
    rows = gather_rows(dist, [step_ms, stw_ms, e2e_ms, link_gbps], device)
    mx = [max(r[k] for r in rows) for k in range(3)]
    per_rank = [{"rank": i, "ms_per_step": round(r[0], 4), "stw_ms": round(r[1], 4), "e2e_ms": round(r[2], 3),
                 "host_link_gbps": round(r[3], 2)} for i, r in enumerate(rows)]
    return mx[0], mx[1], mx[2], per_rank


def aggregate_value(world: int, state_bytes: int, step_ms: float) -> float:
    """Whole-job GB/s: every rank checkpoints state_bytes; time = max over ranks."""
    return world * state_bytes / (step_ms * 1e-3) / 1e9


def barrier(dist, device):
    if dist is not None:
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[device])
        else:
            dist.barrier()


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref) -- the reference's own code on host cores

def cpu_reference_run(wl: Workload, steps: int, warmup: int, threads: int, sample_bytes: int):
    """Each step: the epoch's writes (untimed) then the reference dump loop
    (crc32 per chunk, chunk_copied capture of dirty chunks, cr.hpp:481-504)
    plus the STW re-capture of the window's buffers, on `threads` cores.
    Returns (GB/s, ms/step, sample description, kind)."""
    import ctypes as C
    from oracle_ctypes import oracle, reference
    ref = reference()
    kind = "reference"
    orc = oracle()
    # bounded sample: a prefix of the buffer set
    idx, acc = [], 0
    for i, n in enumerate(wl.sizes):
        if acc >= sample_bytes:
            break
        idx.append(i)
        acc += n
    sizes = [wl.sizes[i] for i in idx]
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(threads)  # untimed input generation (ctypes drops the GIL)
    contents = [np.empty(wl.sizes[i], np.uint8) for i in idx]
    list(pool.map(lambda ia: orc.or_fill_bytes(7000 + ia[0], ia[1].ctypes.data, ia[1].size), zip(idx, contents)))
    nch = sum((n + CHUNK - 1) // CHUNK for n in sizes)
    prev = np.zeros(nch, np.uint32)
    cur = np.zeros(nch, np.uint32)
    flags = np.zeros(nch, np.uint8)
    if ref is None:
        raise SystemExit("oracle/_ref missing: run __graft_entry__.build() where /root/reference exists")
    ptrs = (C.c_void_p * len(sizes))(*[c.ctypes.data for c in contents])
    sz = np.array(sizes, np.uint64)
    st = ref.ref_state_create(len(sizes), sz.ctypes.data, ptrs, CHUNK)
    ref.ref_state_dump(st, prev.ctypes.data, 0, cur.ctypes.data, flags.ctypes.data, threads)
    times = []
    sel = {i + 1 for i in idx}
    for e in range(1, warmup + steps + 1):
        prev[:] = cur
        groups: dict[int, list] = {}  # one host thread per buffer: write_content is per-buffer state
        for w in wl.epoch_writes(e):
            if w[0] in sel:
                groups.setdefault(w[0], []).append(w)

        def apply(ws):
            for h, off, n, seed in ws:
                buf = np.empty(n, np.uint8)
                orc.or_fill_bytes(seed, buf.ctypes.data, n)
                ref.ref_state_write(st, idx.index(h - 1), off, buf.ctypes.data, n)
        list(pool.map(apply, groups.values()))
        t0 = time.perf_counter()
        ref.ref_state_dump(st, prev.ctypes.data, 1, cur.ctypes.data, flags.ctypes.data, threads)
        t1 = time.perf_counter()
        if e > warmup:
            times.append(t1 - t0)
    ref.ref_state_destroy(st)
    pool.shutdown()
    ms = statistics.median(times) * 1e3
    return acc / (ms * 1e-3) / 1e9, ms, f"{len(sizes)} of {len(wl.sizes)} buffers ({acc} B) per step", kind


# ---------------------------------------------------------------------------
# GPU arm

def bind_numa_local(device: int) -> str:
    """Pin this process to the CPUs local to the GPU (pinned host buffers are
    then allocated on the GPU's NUMA node, the PCIe root it hangs off)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device)
        bus = pynvml.nvmlDeviceGetPciInfo(h).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        path = f"/sys/bus/pci/devices/{bus.lower()[-12:]}/local_cpulist"
        if not os.path.exists(path):
            path = f"/sys/bus/pci/devices/{bus.lower()}/local_cpulist"
        spec = open(path).read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        os.sched_setaffinity(0, cpus)
        return spec
    except Exception as ex:  # not fatal: report it
        return f"unbound ({type(ex).__name__})"


def run_gpu(args, wl: Workload, world, rank, local, dist):
    import ctypes as C
    import paper_2405_12079_b200 as pd
    from paper_2405_12079_b200.posdump import D2H
    numa = bind_numa_local(local)
    pd.check(pd.lib().pos_set_device(local))

    total = wl.total
    log(f"{wl.name}: {len(wl.sizes)} buffers, {total} B; allocating device state")
    mem = pd.DeviceMemory(total + 256 * len(wl.sizes))
    bufs, off = [], 0
    for i, n in enumerate(wl.sizes):
        bufs.append(pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + off, size=n))
        off += (n + 255) // 256 * 256
    # initial state: parameters H2D-loaded (upstream provenance), the rest
    # produced on the device
    pd.fill_batch([(b.dev_ptr, b.size, 5000 + b.handle) for b in bufs])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=CHUNK, cache_capacity=0), device=local)
    eng.register_buffers(bufs)
    if args.hash_sms:
        eng.set_hash_sms(args.hash_sms)
    if args.o2_digest2:
        eng.set_o2_digest2(True)
    if args.slice_mib or args.window:
        eng.set_host_leg(slice_bytes=(args.slice_mib or 16) << 20, window=args.window or 3)
    if wl.params:  # note_h2d_provenance (process.hpp:505-522): Upstream.crc on device
        eng.hash_chunks()
        eng.scan_dedup()
        crcs, _ = eng.buffer_crcs()
        for b, c in zip(bufs, crcs):
            if b.handle in wl.params:
                b.upstream = pd.Upstream(int(c), True)
                eng.update_buffer(b)
    cache_ptr, cache_cap = eng.cache()
    # Landing ring of pinned buffers: the host applies step e's packs out of
    # one buffer while step e+1 DMA-writes the next (DMA into lines the CPU
    # just read costs ~30% of the link).
    direct = args.mode == "direct"
    if direct:
        # The checkpoint image itself is pinned + mapped: the copy engine moves
        # every shipped chunk to its place (chunk_copied, cr.hpp:499-501).
        img_offs, o = [], 0
        align = args.image_align or 256
        for b in bufs:
            img_offs.append(o)
            o += (b.size + align - 1) // align * align
        log(f"allocating the pinned host image ({o} B)")
        img_pin = pd.PinnedHost(max(o, 1), image=True)  # zero-filled huge pages, pinned + mapped
        huge_gb = anon_huge_gb()
        log(f"host image ready ({huge_gb} GB of anonymous huge pages in the process)")
        host_image = [img_pin.array[a:a + b.size] for a, b in zip(img_offs, bufs)]
        eng.register_image(host_image)
        pins = []
    else:
        pins = [pd.PinnedHost(min(cache_cap, 2 * total + (64 << 20))) for _ in range(args.ring)]
        host_image = [np.zeros(b.size, np.uint8) for b in bufs]
    handles = [b.handle for b in bufs]
    flush = pd.DeviceMemory(256 << 20)
    ckpt, app = pd.Stream(priority=args.ckpt_priority), pd.Stream(priority=args.app_priority)
    copy = pd.Stream(priority=args.drain_priority if args.drain_priority >= 0 else
                     (args.ckpt_priority if args.mode == "direct" else 0))
    by_handle = {b.handle: b for b in bufs}

    class app_window:
        """The application's window as a callable: one pos_fill_batch launch
        per kernel, or (graph=True) all of them captured once into a CUDA
        graph launched as one stream operation."""

        def __init__(self, args_list, graph):
            self.args, self.exec = args_list, None
            if graph and args_list:
                pd.check(pd.lib().pos_stream_begin_capture(int(app)))
                for a in args_list:
                    pd.check(pd.lib().pos_fill_batch(a.ctypes.data, a.shape[0], int(app)))
                ge = C.c_void_p()
                pd.check(pd.lib().pos_stream_end_capture(int(app), C.byref(ge)))
                self.exec = ge.value

        def __call__(self):
            if self.exec:
                pd.check(pd.lib().pos_graph_launch(self.exec, int(app)))
            else:
                for a in self.args:
                    pd.lib().pos_fill_batch(a.ctypes.data, a.shape[0], int(app))

        def close(self):
            if self.exec:
                pd.check(pd.lib().pos_graph_destroy(self.exec))
                self.exec = None

    class AppThread:
        """Long-lived application host thread: submits a window of kernels
        (pos_fill_batch) on the app stream, records event 2, and -- like an
        interception layer on the application's own thread -- enqueues the
        final stop right behind its last kernel (once the dump's host side
        has staged the delta), so the stop-the-world gather starts the moment
        the window drains."""

        def __init__(self):
            self.q, self.done = [], threading.Event()
            self.go, self.staged = threading.Event(), threading.Event()
            self.fill, self.h = pd.lib().pos_fill_batch, int(app)
            self.stw = None
            self.loop, self.graph, self.stop_loop, self.iters = False, False, threading.Event(), 0
            self.submitted = threading.Event()
            threading.Thread(target=self.run, daemon=True).start()

        def run(self):
            pd.check(pd.lib().pos_set_device(local))  # the CUDA device is per host thread
            while True:
                self.go.wait()
                self.go.clear()
                try:
                    window = app_window(self.q, self.graph)
                    eng.event_record(9, app)  # the application's window: 9 -> 2
                    window()
                    self.submitted.set()
                    self.iters = 1
                    # app-load pass: the application keeps iterating its window for
                    # the whole pre-copy, at most two iterations queued ahead
                    if self.loop:
                        eng.event_record(20, app)  # end of iteration 1
                    while self.loop and not self.stop_loop.is_set():
                        window()
                        self.iters += 1
                        eng.event_record(20 + (self.iters - 1) % 2, app)
                        eng.event_elapsed(9, 20 + (self.iters - 2) % 2)  # host waits for the iteration before
                    eng.event_record(2, app)
                    window.close()
                except Exception as ex:  # never leave the main thread waiting: surfaced by wait()
                    self.stw_result, self.error = None, ex
                    self.submitted.set()
                    self.done.set()
                    continue
                self.staged.wait()  # the engine is not re-entrant: after prepare_final_stop
                self.staged.clear()
                try:
                    self.stw_result, self.error = self.stw(), None
                except Exception as ex:  # surfaced on the main thread
                    self.stw_result, self.error = None, ex
                self.done.set()

        def submit(self, args_list, stw, loop=False, graph=False):
            self.q, self.stw, self.loop, self.graph = args_list, stw, loop, graph
            self.stop_loop.clear()
            self.submitted.clear()
            self.done.clear()
            self.go.set()

        def wait(self):
            self.done.wait()

    app_thread = AppThread()
    apply_threads = max(1, min(32, len(os.sched_getaffinity(0))))
    # slots: 0 start, 1 compact done, 2 app drained, 3 stop, 4 stw end, 5 end
    def checkpoint(e: int, e2e: bool, app_load: bool = False, app_graph: bool = False, pregather: bool = False):
        pin = pins[e % len(pins)] if pins else None
        # untimed application iteration
        pd.fill_batch([(by_handle[h].dev_ptr + o, n, seed) for h, o, n, seed in wl.epoch_writes(e)])
        pd.check(pd.lib().pos_memset(flush.ptr, e & 0xFF, flush.nbytes, None))  # flush L2
        pd.device_synchronize()
        window = [] if args.no_window else wl.window(e)
        launches0 = eng.launches

        # The window's kernels, argument blocks prepared ahead (as an application
        # would have its launch arguments ready): [dev_ptr, bytes, seed] per write.
        app_args = [np.array([[by_handle[h].dev_ptr, by_handle[h].size, s & 0xFFFFFFFFFFFFFFFF]
                              for h, s in k], dtype=np.uint64) for k in window]
        dag_writes = sorted({h for k in window for h, _ in k})

        t0 = time.perf_counter()
        # The window's kernels are in the DAG from submission (their spec write
        # sets, process.hpp:313-344): their buffers are left to the STW pass,
        # as record_dirty's copy cancellation does (cr.hpp:909-918).
        eng.record_dirty(dag_writes)
        def final_stop():  # at_final_stop (cr.hpp:599-621): drain the app, STW gather
            # (direct mode: the engine itself holds the stop until the
            # pre-copy's last slice has landed -- check_precopy_done ->
            # final_stop, cr.hpp:532-597 -- the application never resumes
            # over chunks still being copied)
            eng.stream_wait_event(2, ckpt)
            if args.trace:  # device-clock cross-check of the window (adds two operations to it)
                eng.event_record(3, ckpt)
                eng.stamp(3, ckpt)
                return eng.at_final_stop(stream=ckpt, stw_end_slot=4)
            # the window is [event 3, gather, event 4] and nothing else
            return eng.at_final_stop(stream=ckpt, stw_begin_slot=3, stw_end_slot=4)

        app_thread.submit(app_args, final_stop, loop=app_load and bool(app_args),
                          graph=app_graph)  # the application's own host thread
        eng.event_record(0, ckpt)  # device clock starts with the dump's first operation
        if direct:  # hash -> O1 -> scan per wave; chunks stored into the image on `copy`
            eng.precopy_direct(waves=args.waves, stream=ckpt, drain_stream=copy)
            packs = []
        else:  # waves: hash/O1/compaction of wave k+1 overlaps the D2H of wave k
            packs = eng.precopy_pipelined(pin.ptr, waves=args.waves, stream=ckpt, copy_stream=copy)
        eng.event_record(1, ckpt)
        if not direct:
            eng.event_record(8, copy)
        # Stage the delta's layout now (write sets known at submission), so the
        # stop window holds only the gather; then the final stop: hold the app
        # (its window is fully submitted) and drain it.
        eng.prepare_final_stop(stream=ckpt)
        if pregather and dag_writes:  # eager delta capture behind the window's writers (not with app_load:
            app_thread.submitted.wait()  # its repeated writes are not re-recorded)
            if app_thread.done.is_set() and app_thread.error is not None:
                raise app_thread.error
            eng.pregather(dag_writes, after_stream=app, stream=ckpt)
        if app_load and direct:  # the application iterates until the host leg submitted its last slice
            eng.host_leg_stats()
            app_thread.stop_loop.set()
        app_thread.staged.set()
        app_thread.wait()
        if app_thread.error is not None:
            raise app_thread.error
        doff, dbytes = app_thread.stw_result
        if direct:
            eng.delta_drain(stream=copy)  # waits for the gather (not the post-stop hash) by itself
            copy.wait(ckpt)  # the step ends when the post-stop hash is done too
        else:
            copy.wait(ckpt)
            eng.d2h_async(pin.ptr + doff, doff, dbytes, stream=copy)
        eng.event_record(5, copy)
        copy.synchronize()
        ckpt.synchronize()
        if direct:
            _, pre_payload = eng.precopy_direct_result()
            dpay = sum(by_handle[h].size for h in dag_writes)
        # host image = the checkpoint target (captured_); inside the e2e wall
        # clock, always outside the device-timed region
        if not args.no_host_apply and not direct:
            for o, z in packs:
                pd.apply_pack_host(pin.array[o:o + z], handles, host_image, threads=apply_threads)
            pd.apply_pack_host(pin.array[doff:doff + dbytes], handles, host_image, threads=apply_threads)
        t1 = time.perf_counter()
        ms = eng.event_elapsed(0, 5)
        stw = eng.event_elapsed(3, 4)
        stw_dev = eng.stamp_elapsed(3, 4) if args.trace else None  # same window on the device clock

        def kms(name):
            try:
                return eng.kernel_ms(name)
            except pd.SimError:
                return 0.0
        hash_ms = kms("hash_waves")
        if args.trace:
            marks = {"precopy_enqueued": 1, "app_drained": 2, "stop": 3, "stw_end": 4, "end": 5}
            tl = {k: round(eng.event_elapsed(0, v), 4) for k, v in marks.items()}
            tl.update(eng.timeline(0))
            tl["packs_MB"] = [round(z / 1e6, 2) for _, z in packs] + [round(dbytes / 1e6, 2)]
            print(json.dumps(tl), file=sys.stderr)
        r = {"ms": ms, "stw_ms": stw, "stw_dev_ms": stw_dev, "hash_ms": hash_ms, "wall_ms": (t1 - t0) * 1e3,
             "app_ms": eng.event_elapsed(9, 2) if window else 0.0, "app_iters": app_thread.iters if window else 0,
             "precopy_bytes": pre_payload if direct else sum(z for _, z in packs),
             "delta_bytes": dpay if direct else dbytes, "launches": eng.launches - launches0 + len(window),
             "d2h_ms": kms("d2h"), "compact_ms": kms("copy"),
             "scan_ms": kms("scan"), "delta_ms": kms("delta") if dbytes > 0 else 0.0,
             "delta_hash_ms": kms("delta_hash") if dbytes > 0 else 0.0,
             "h2d_bytes": len(bufs) + 64 + (48 if direct else 16) * (dbytes // CHUNK + 1)}
        eng.commit_epoch()
        return r

    # epoch 0: fresh full checkpoint (untimed) seeds digests + host image
    log("epoch 0 (full checkpoint)")
    checkpoint(0, True)
    e = 1
    for _ in range(args.warmup):
        log(f"warm-up epoch {e}")
        checkpoint(e, False)
        e += 1
    # the application's window alone (no dump running): its slowdown beside the dump
    app_alone = []
    for k in range(3):
        win = wl.window(e + 100 + k)
        if not win:
            break
        args_list = [np.array([[by_handle[h].dev_ptr, by_handle[h].size, s & 0xFFFFFFFFFFFFFFFF] for h, s in kk],
                              dtype=np.uint64) for kk in win]
        pd.check(pd.lib().pos_memset(flush.ptr, k, flush.nbytes, None))
        pd.device_synchronize()
        eng.event_record(9, app)
        for a in args_list:
            pd.lib().pos_fill_batch(a.ctypes.data, a.shape[0], int(app))
        eng.event_record(2, app)
        app.synchronize()
        app_alone.append(eng.event_elapsed(9, 2))
    # ... and iterated back to back with the app-load pass's own loop (host
    # throttle included): the baseline of its throughput ratio
    app_loop_alone = {}
    if app_alone and direct and not args.no_window and not args.no_app_load:
        for graph in (False, True):
            window, n_it = app_window(args_list, graph), 2000
            window()  # warm
            app.synchronize()
            eng.event_record(9, app)
            window()
            eng.event_record(20, app)
            for it in range(2, n_it + 1):
                window()
                eng.event_record(20 + (it - 1) % 2, app)
                eng.event_elapsed(9, 20 + (it - 2) % 2)
            eng.event_record(2, app)
            app_loop_alone[graph] = eng.event_elapsed(9, 2) / n_it
            window.close()
    link_peak0 = pinned_d2h_peak(pd, eng, flush, copy, pins[0] if pins else None)  # before, and after (max)
    log("timed steps")
    barrier(dist, local)
    res = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            res.append(checkpoint(e, False))
            log(f"step {e}: {res[-1]['ms']:.2f} ms (stw {res[-1]['stw_ms']:.4f} ms, d2h {res[-1]['d2h_ms']:.2f} ms)")
            e += 1
    barrier(dist, local)
    # Application under a continuous load: its window iterated through the
    # whole pre-copy (every write DAG-tracked), untimed for the headline.
    app_load = []
    if direct and app_alone and not args.no_window and not args.no_app_load:
        log("application-load steps")
        for graph in (False, False, True, True):
            app_load.append(checkpoint(e, False, app_load=True, app_graph=graph))
            app_load[-1]["graph"] = graph
            e += 1
    log("e2e steps")
    e2e_res = []
    for _ in range(max(3, min(args.steps, 10))):
        e2e_res.append(checkpoint(e, True))
        e += 1
    # Eager delta capture: the window's buffers gathered behind their writers
    # (pos_delta_pregather), so the stop gathers only what was written since;
    # the last of them is the checkpoint the image-parity check restores
    eager = []
    if direct and not args.no_window:
        log("eager-capture steps")
        for _ in range(3):
            eager.append(checkpoint(e, False, pregather=True))
            e += 1
    # Image parity.  (1) 512 random chunks: host image bytes == device bytes;
    # (2) small states: every buffer byte for byte; large states (c3/c4/c5):
    # the device state is thrown away and restored from the host image, and
    # every chunk digest after the restore equals the checkpoint's (the whole
    # image, at 2^-32 per chunk), then a delta pack is replayed (scatter).
    log("image parity")
    sample_ok = image_sample_check(pd, bufs, host_image, mem, 512, seed=e)
    full = wl.total <= (4 << 30)
    ok = sample_ok and (args.no_host_apply or not full or all(
        np.array_equal(img, mem.download(b.size, offset=b.dev_ptr - mem.ptr)) for b, img in zip(bufs, host_image)))
    restore = (restore_measure(eng, pd, wl, bufs, host_image, mem, e)
               if (wl.name in ("c3", "c4", "c5") and direct) else None)
    writer = image_writer_measure(pd, eng, bufs, host_image) if (direct and wl.total > (4 << 30)) else None
    if restore is not None:
        ok = ok and restore["digests_match_checkpoint"] and restore["delta_replay"]["bit_exact"]

    step_ms = sum(r["ms"] for r in res) / len(res)
    stw_ms = statistics.median(r["stw_ms"] for r in res)
    hash_ms = statistics.mean(r["hash_ms"] for r in res)
    e2e_ms = statistics.median(r["wall_ms"] for r in e2e_res)
    d2h_bytes = statistics.mean(r["precopy_bytes"] + r["delta_bytes"] for r in res)
    delta_bytes = statistics.mean(r["delta_bytes"] for r in res)
    step_ms, stw_ms, e2e_ms, per_rank = rank_summary(dist, local, step_ms, stw_ms, e2e_ms,
                                                     d2h_bytes / (step_ms * 1e-3) / 1e9)

    link_peak = max(link_peak0, pinned_d2h_peak(pd, eng, flush, copy, pins[0] if pins else None))
    d2h_precopy = statistics.mean(r["precopy_bytes"] / (r["d2h_ms"] * 1e-3) / 1e9 for r in res)
    d2h_step = d2h_bytes / (step_ms * 1e-3) / 1e9

    n_chunks = eng.n_chunks
    # per hash launch (one per wave): read B; digest prev read + cur write (8 B) + flag (1 B) per chunk
    n_launch = max(1, min(args.waves, len(wl.sizes))) if direct else max(1, args.waves)
    alg_bytes = (total + 9 * n_chunks) / n_launch
    launch_ms = hash_ms / n_launch
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs", FALLBACK_HBM)
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"hash_traffic_{wl.name}.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = (round(tj["traffic_over_alg"] * alg_bytes) if "traffic_over_alg" in tj
                   else tj.get("dram_bytes_per_launch"))
    stw_gbps = 2 * delta_bytes / (stw_ms * 1e-3) / 1e9 if stw_ms > 0 else 0.0

    out = None
    if rank == 0:
        value = aggregate_value(world, total, step_ms)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            log("CPU baseline (oracle/_ref)")
            try:
                threads = os.cpu_count() or 1
                v, ms, sample, kind = cpu_reference_run(wl, 3, 1, threads, min(total, args.ref_sample_bytes))
                cpu = {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": kind,
                       "cpu_model": cpu_model(),
                       "sample": sample + "; crc32 per 64 KiB chunk + chunk_copied capture of dirty chunks, "
                                          "median of 3 steps after 1 warm-up"}
            except SystemExit as ex:
                cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference", "sample": str(ex)}
        out = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(step_ms, 4),
            "stw_ms": round(stw_ms, 4),
            "stw_window": ("[event, TMA bulk gather of the DAG-dirty buffers into the on-device cache, event] on "
                           "the dump stream, once the application drained and the pre-copy was complete "
                           "(pos_final_stop); the delta's hash and D2H run after the stop"),
            **({"stw_device_clock_ms": round(statistics.median(r["stw_dev_ms"] for r in res), 4)} if args.trace else {}),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic",
            "config": bench_config(wl, world),
            "run": {
                "d2h_bytes_per_step": int(d2h_bytes), "stw_delta_bytes": int(delta_bytes),
                "l2": "flushed between steps (256 MiB memset)", "host_cpus": numa,
                **({"image_huge_pages_gb": huge_gb} if direct else {}),
                "hash_sms": args.hash_sms or "all",
                "mode": ("direct: hash -> O1 -> scan per wave, copy-engine runs from the live buffers into the "
                         "pinned host image" if direct else "pack: POSD packs in the cache, D2H + host apply")},
            "gpu_launches": int(statistics.mean(r["launches"] for r in res)),
            "gpu_launches_counts": "libposdump kernels per step: the dump's (hash, O1, scan, staging, STW gather, "
                                   "delta hash) plus the synthetic application's k_fill window launches",
            "roofline": {"bound": "hbm", "kernel": "k_hash_chunks", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "alg_bytes_per_launch": int(alg_bytes),
                         "launch_ms": round(launch_ms, 5), "launches_per_step": n_launch,
                         "launch_ms_counts": ("mean over the step's hash launches (one per wave; CUDA events on "
                                              "the dump stream around each)"),
                         "traffic_source": ("dram__bytes_read+write of one wave-sized launch under ncu --set full "
                                            "(profiles/r2/ncu_hash_c5wave.json), per algorithmic byte"),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                         "note": ("dominant HBM kernel of the dump; the step itself is bound by the host link "
                                  "(copy-engine runs into the pinned image): see host_link")},
            "host_link": {"bound": "pcie", "achieved": round(d2h_step, 2), "peak": round(link_peak, 2),
                          "unit": "GB/s", "frac": round(d2h_step / link_peak, 4),
                          "achieved_over": "whole step: every byte that crossed PCIe / step time",
                          "precopy_leg_gbps": round(d2h_precopy, 2),
                          "peak_source": "best of 10 pinned cudaMemcpyAsync D2H of 256 MiB, 5 before the timed steps and 5 after"},
            "per_rank": per_rank,
            "host_link_aggregate_gbps": round(sum(r["host_link_gbps"] for r in per_rank), 2),
            **({"stw_eager_capture": {
                "stw_ms": round(statistics.median(r["stw_ms"] for r in eager), 4),
                "ms_per_step": round(statistics.median(r["ms"] for r in eager), 4),
                "how": ("3 extra checkpoints (not in value): pos_delta_pregather gathers the window's DAG-dirty "
                        "buffers into the delta pack behind their last writers, before the stop; the stop "
                        "gathers only buffers written since (none here), the image bytes are the same; the "
                        "last of them is the checkpoint image_parity restores")}}
               if eager else {}),
            "stw_gather": {"bound": "hbm", "bytes": int(delta_bytes), "alg_bytes": int(2 * delta_bytes),
                           "achieved": round(stw_gbps, 1), "peak": peak, "unit": "GB/s",
                           "frac": round(stw_gbps / peak, 4) if peak else None,
                           "note": "read + write of the DAG-dirty buffers over the whole STW window (launch incl.)"},
            **({"app_interference": {
                "window_ms_alone": round(statistics.median(app_alone), 4),
                "window_ms_during_dump": round(statistics.median(r["app_ms"] for r in res), 4),
                "slowdown": round(statistics.median(r["app_ms"] for r in res) / statistics.median(app_alone), 3),
                "window": "the application kernels of the pre-copy window (k_fill of the DAG-dirty buffers), "
                          "event-timed on the application stream",
                **({"under_load": {
                    "app_throughput_vs_alone": round(statistics.median(
                        r["app_iters"] * app_loop_alone[False] / r["app_ms"] for r in app_load if not r["graph"]), 4),
                    "app_throughput_vs_alone_graph": round(statistics.median(
                        r["app_iters"] * app_loop_alone[True] / r["app_ms"] for r in app_load if r["graph"]), 4),
                    "app_iteration_ms_alone": round(app_loop_alone[False], 4),
                    "app_iteration_ms_alone_graph": round(app_loop_alone[True], 4),
                    "app_iterations_per_step": int(statistics.median(r["app_iters"] for r in app_load)),
                    "dump_gbps": round(total / (statistics.median(r["ms"] for r in app_load) * 1e-3) / 1e9, 3),
                    "stw_ms": round(statistics.median(r["stw_ms"] for r in app_load), 4),
                    "why": ("the window is launch-bound (9 kernels of ~25 us): while the host link is saturated "
                            "every stream operation's command fetch waits behind the posted D2H writes; one CUDA "
                            "graph launch per window instead of 9 launches (graph) cuts that cost: "
                            "tools/frontend_micro.cu"),
                    "how": ("4 extra checkpoints (not in value; 2 per variant): the application iterates its window back to back "
                            "until the host leg has submitted its last slice; throughput = iterations x the "
                            "iteration time of the same loop with no dump / event-timed application time")}}
                   if app_load and len(app_loop_alone) == 2
                   and statistics.median(r["app_iters"] for r in app_load) >= 10 else {})}} if app_alone else {}),
            "stages_ms": {k: round(statistics.mean(r[k] for r in res), 4)
                          for k in ("hash_ms", "scan_ms", "compact_ms", "delta_ms", "delta_hash_ms", "d2h_ms")},
            "e2e": {"value": round(world * total / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": int(statistics.mean(r["h2d_bytes"] for r in e2e_res)),
                    "d2h_bytes_per_step": int(statistics.mean(r["precopy_bytes"] + r["delta_bytes"] + 24
                                                              for r in e2e_res)),
                    "how": ("host wall clock around the DumpEngine calls until every byte is in the host image "
                            "(direct: the copy engine writes the pinned image; pack: D2H + host-side pack apply)")},
            "image_parity": bool(ok),
            "image_parity_how": ("512 random chunks byte-compared with the device" +
                                 ("; every buffer byte-compared" if full else
                                  "; whole image: device state lost, restored from the image, every chunk "
                                  "digest == the checkpoint's")),
            **({"restore": restore} if restore else {}),
            **({"image_writer": writer} if writer else {}),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
    eng.close()
    img_pin = None
    return out


def pinned_d2h_peak(pd, eng, flush, stream, pin=None):
    """Best of 5 plain pinned D2H copies of 256 MiB (CUDA events, GB/s)."""
    from paper_2405_12079_b200.posdump import D2H
    pin = pin or pd.PinnedHost(256 << 20)
    n = min(flush.nbytes, pin.nbytes)
    best = 0.0
    for _ in range(5):
        eng.event_record(6, stream)
        pd.check(pd.lib().pos_memcpy(pin.ptr, flush.ptr, n, D2H, int(stream)))
        eng.event_record(7, stream)
        best = max(best, n / (eng.event_elapsed(6, 7) * 1e-3) / 1e9)
    return best


def image_sample_check(pd, bufs, host_image, mem, n, seed):
    """n random 64 KiB-aligned ranges: host image bytes == device bytes."""
    rng = np.random.default_rng(seed)
    for _ in range(n):
        i = int(rng.integers(len(bufs)))
        b = bufs[i]
        off = int(rng.integers((b.size + CHUNK - 1) // CHUNK)) * CHUNK
        ln = min(CHUNK, b.size - off)
        if not np.array_equal(host_image[i][off:off + ln], mem.download(ln, offset=b.dev_ptr - mem.ptr + off)):
            return False
    return True


def restore_measure(eng, pd, wl, bufs, host_image, mem, e):
    """Failover (BASELINE configs 3-5): the device state is lost (zeroed),
    the checkpoint image is loaded back on demand (pos_restore_image_*: loads
    in buffer order, a buffer in the middle gated first as the first replayed
    kernel would), then a delta pack of the next writes (c4: the next decode
    burst; c3/c5: the optimizer tail) is replayed with the scatter kernel
    (delta-restore).  Checks: digests after the restore == the checkpoint's
    digests (every chunk), and the scattered delta == the live writes."""
    eng.hash_chunks()  # the state as of the last checkpoint (nothing written since)
    digests_ckpt = eng.digests()
    total = sum(b.size for b in bufs)
    for b in bufs:
        pd.check(pd.lib().pos_memset(b.dev_ptr, 0, b.size, None))
    pd.device_synchronize()
    h2d, app = pd.Stream(), pd.Stream(priority=1)
    order = [b.handle for b in bufs]
    gate_h = bufs[len(bufs) // 2].handle  # a buffer in the middle of the load order
    eng.event_record(10, h2d)
    t0 = time.perf_counter()
    eng.restore_image_begin(host_image, order=order, h2d_stream=h2d)
    eng.restore_gate(gate_h, stream=app)
    eng.event_record(11, app)
    eng.restore_image_wait()
    eng.event_record(12, h2d)
    t1 = time.perf_counter()
    restore_ms = eng.event_elapsed(10, 12)
    gate_ms = eng.event_elapsed(10, 11)
    eng.hash_chunks()
    restored_ok = bool(np.array_equal(eng.digests(), digests_ckpt))
    # delta-restore replay: the next writes as a POSD pack (pack mode),
    # scattered back onto the restored state
    eng.commit_epoch()
    by_handle = {b.handle: b for b in bufs}
    if wl.name == "c4":
        writes = wl.epoch_writes(e)
    else:  # the optimizer tail's tensors, rewritten
        writes = [(h, 0, by_handle[h].size, mix64(e + 7, h)) for h in sorted(wl.win)]
    pd.fill_batch([(by_handle[h].dev_ptr + o, n, s) for h, o, n, s in writes])
    pd.device_synchronize()
    pack_bytes = eng.plan_precopy()
    cache_ptr, _ = eng.cache()
    probe = writes[:64]
    want = [mem.download(min(n, 1 << 20), offset=by_handle[h].dev_ptr - mem.ptr + o) for h, o, n, _ in probe]
    for h, o, n, _ in writes:
        pd.check(pd.lib().pos_memset(by_handle[h].dev_ptr + o, 0, n, None))
    pd.device_synchronize()
    eng.materialize(cache_ptr, pack_bytes)
    pd.device_synchronize()
    scatter_ms = eng.kernel_ms("scatter")
    got = [mem.download(min(n, 1 << 20), offset=by_handle[h].dev_ptr - mem.ptr + o) for h, o, n, _ in probe]
    eng.hash_chunks()  # every chunk of the replayed state, not only the probes
    replay_dig = eng.digests()
    eng.commit_epoch()
    delta_ok = all(np.array_equal(a, b) for a, b in zip(want, got))
    payload = sum(n for _, _, n, _ in writes)
    peak = measured_peaks().get("hbm_gbs", FALLBACK_HBM)
    sc = 2 * payload / (scatter_ms * 1e-3) / 1e9
    # the host link's H2D peak on this box: best of 5 pinned 256 MiB copies
    from paper_2405_12079_b200.posdump import H2D
    pin, dev = pd.PinnedHost(256 << 20), pd.DeviceMemory(256 << 20)
    h2d_peak = 0.0
    for _ in range(5):
        eng.event_record(6, h2d)
        pd.check(pd.lib().pos_memcpy(dev.ptr, pin.ptr, 256 << 20, H2D, int(h2d)))
        eng.event_record(7, h2d)
        h2d_peak = max(h2d_peak, (256 << 20) / (eng.event_elapsed(6, 7) * 1e-3) / 1e9)
    pin.close()
    dev.close()
    rgbps = total / (restore_ms * 1e-3) / 1e9
    return {"bytes": total, "ms": round(restore_ms, 3), "gbps": round(rgbps, 2),
            "h2d_peak_gbps": round(h2d_peak, 2), "frac": round(rgbps / h2d_peak, 4),
            "wall_ms": round((t1 - t0) * 1e3, 3), "bound": "pcie (H2D, copy engine)",
            "first_gated_buffer_ms": round(gate_ms, 3), "digests_match_checkpoint": restored_ok,
            "delta_replay": {"pack_bytes": pack_bytes, "payload_bytes": payload, "scatter_ms": round(scatter_ms, 4),
                             "scatter_gbps": round(sc, 1), "roofline_frac": round(sc / peak, 4),
                             "alg_bytes": "2 x payload (read pack, write buffers)", "bit_exact": bool(delta_ok),
                             "no_stray_writes": bool(
                                 int(np.count_nonzero(replay_dig != digests_ckpt)) <= pack_entries(writes))}}


def image_writer_measure(pd, eng, bufs, host_image, sample_bytes: int = 8 << 30) -> dict:
    import ctypes as C
    """The streaming POSI writer (write_image, image.hpp:136-207; SURVEY 8(f)
    rank 1) on a prefix of the checkpoint image: Inline records straight from
    the pinned host image into a pre-touched output buffer (the payload
    copies on up to 16 host threads)."""
    recs, allocs, acc = [], [], 0
    for b, img in zip(bufs, host_image):
        if acc >= sample_bytes:
            break
        recs.append(pd.GpuBufferRec(handle=b.handle, kind=0, inline_bytes=img))
        allocs.append((b.handle, 0x7000_0000_0000 + acc, b.size))
        acc += b.size
    ci = pd.CheckpointImage(page_size=4096, gpu_records=recs, allocs=allocs, next_handle=len(recs) + 1)
    out = np.zeros(acc + (1 << 20) + 64 * len(recs), np.uint8)
    out[::4096] = 1  # first touch outside the timed call
    times = []
    for _ in range(2):
        t0 = time.perf_counter()
        n = pd.write_image(ci, out=out)
        times.append(time.perf_counter() - t0)
    ms = min(times) * 1e3
    # read_image's validation of the same bytes (image.hpp:209-361), zero-copy
    off = C.c_uint64(0)
    t0 = time.perf_counter()
    rc = pd.lib().pos_image_check(out.ctypes.data, int(n), C.byref(off))
    check_ms = (time.perf_counter() - t0) * 1e3
    # ... and the image restored from those (pageable) bytes: the buffers get
    # back what they hold (read_image + materialize, pos_image_restore)
    loaded, recomp, coff = C.c_uint32(0), C.c_uint32(0), C.c_uint64(0)
    s = pd.Stream()
    t0 = time.perf_counter()
    rrc = pd.lib().pos_image_restore(eng.ctx, out.ctypes.data, int(n), int(s), C.byref(coff), C.byref(loaded),
                                     C.byref(recomp))
    restore_ms = (time.perf_counter() - t0) * 1e3
    del out
    return {"bytes": int(n), "records": len(recs), "ms": round(ms, 2), "gbps": round(n / (ms * 1e-3) / 1e9, 2),
            "read_check": {"valid": rc == 0, "ms": round(check_ms, 3),
                           "how": "pos_image_check: read_image's structural checks over the bytes in place "
                                  "(zero-copy; the reference's read_image parses and copies every payload)"},
            "threads": min(16, os.cpu_count() or 1),
            "restore_from_image": {"ok": rrc == 0, "records": int(loaded.value), "ms": round(restore_ms, 2),
                                   "gbps": round(n / (restore_ms * 1e-3) / 1e9, 2),
                                   "how": "pos_image_restore of the written image from pageable host memory "
                                          "(checks, then one H2D per record)"},
            "how": "pos_image_write of a POSI image of the first buffers' Inline records (from the pinned host "
                   "image) into a pre-touched buffer; byte-identity with the reference's write_image is "
                   "tests/test_capi.py; the reference's own write_image: cpu_breakdown.write_image"}


def pack_entries(writes) -> int:
    return sum((n + CHUNK - 1) // CHUNK + 1 for _, _, n, _ in writes)


def mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def anon_huge_gb():
    """Transparent huge pages backing this process (the image's IOMMU/TLB reach)."""
    try:
        for line in open("/proc/self/smaps_rollup"):
            if line.startswith("AnonHugePages:"):
                return round(int(line.split()[1]) * 1024 / 1e9, 1)
    except OSError:
        pass
    return None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                name = line.split(":", 1)[1].strip()
                break
        else:
            name = "unknown"
        fam = mod = "?"
        for line in open("/proc/cpuinfo"):
            if line.startswith("cpu family"):
                fam = line.split(":", 1)[1].strip()
            elif line.startswith("model") and not line.startswith("model name"):
                mod = line.split(":", 1)[1].strip()
            if fam != "?" and mod != "?":
                break
        return f"{name} (family {fam} model {mod}), {os.cpu_count()} logical CPUs"
    except OSError:
        return "unknown"


def bench_config(wl: Workload, world: int) -> dict:
    """The config dict both arms print (the driver compares them)."""
    cfg = {"workload": wl.desc, "workload_id": wl.name, "chunk_size": CHUNK, "state_bytes_per_gpu": wl.total,
           "buffers": len(wl.sizes), "parallelism": f"replicas{world}",
           "l2": "flushed between timed steps (256 MiB memset)" +
                 ("; the state is also larger than L2" if wl.total > 126 << 20 else "")}
    return cfg


def run_gpu_stream(args, wl: Workload, world, rank, local, dist):
    """States larger than the O3 cache (configs 3/5): every step is a
    cache-cycled pre-copy (pos_precopy_stream) -- waves hash/compact into two
    cache regions while the previous wave drains into pinned landing slots;
    the sink takes each pack in order (a real target would hand it to storage;
    here it accumulates a byte count and checks every pack's header).  The
    application is idle during the checkpoint (optimizer-step boundary), so
    the STW delta is empty."""
    import paper_2405_12079_b200 as pd
    numa = bind_numa_local(local)
    pd.check(pd.lib().pos_set_device(local))
    total = wl.total
    mem = pd.DeviceMemory(total + 256 * len(wl.sizes))
    bufs, off = [], 0
    for i, n in enumerate(wl.sizes):
        bufs.append(pd.GpuBuffer(handle=i + 1, dev_ptr=mem.ptr + off, size=n))
        off += (n + 255) // 256 * 256
    pd.fill_batch([(b.dev_ptr, b.size, 5000 + b.handle) for b in bufs])
    pd.device_synchronize()
    eng = pd.DumpEngine(pd.SimConfig(chunk_size=CHUNK, cache_capacity=0), device=local)
    eng.register_buffers(bufs)
    peer = None
    if args.peer_cache_gb > 0:  # NVLink peer-GPU cache (config 5): the next GPU, or this one on a 1-GPU box
        peer = (local + 1) % pd.device_count()
        eng.attach_peer_cache(peer, int(args.peer_cache_gb * 1e9))
    ckpt, copy = pd.Stream(priority=1), pd.Stream()
    flush = pd.DeviceMemory(256 << 20)
    by_handle = {b.handle: b for b in bufs}
    seen = {"bytes": 0, "packs": 0, "entries": 0}

    def sink(arr, index):
        assert arr[:4].tobytes() == b"POSD"
        seen["bytes"] += arr.size
        seen["packs"] += 1
        seen["entries"] += int(arr[16:20].view(np.uint32)[0])

    def checkpoint(e):
        pd.fill_batch([(by_handle[h].dev_ptr + o, n, sd) for h, o, n, sd in wl.epoch_writes(e)])
        pd.check(pd.lib().pos_memset(flush.ptr, e & 0xFF, flush.nbytes, None))
        pd.device_synchronize()
        seen.update(bytes=0, packs=0, entries=0)
        t0 = time.perf_counter()
        eng.event_record(0, ckpt)
        nbytes, npk = eng.precopy_stream(sink, stream=ckpt, copy_stream=copy)
        off_, dbytes = eng.at_final_stop(stream=ckpt, stw_begin_slot=3, stw_end_slot=4)
        eng.event_record(5, ckpt)
        ckpt.synchronize()
        copy.synchronize()
        t1 = time.perf_counter()
        r = {"ms": eng.event_elapsed(0, 5), "stw_ms": eng.event_elapsed(3, 4), "wall_ms": (t1 - t0) * 1e3,
             "precopy_bytes": nbytes, "delta_bytes": dbytes, "packs": npk, "entries": seen["entries"],
             "hash_ms": eng.kernel_ms("hash_waves"),
             "capture_ms": eng.peer_cache_stats()[0] if peer is not None else None}
        eng.commit_epoch()
        return r

    checkpoint(0)
    e = 1
    for _ in range(args.warmup):
        checkpoint(e)
        e += 1
    barrier(dist, local)
    res = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            res.append(checkpoint(e))
            e += 1
    barrier(dist, local)
    step_ms = sum(r["ms"] for r in res) / len(res)
    stw_ms = statistics.median(r["stw_ms"] for r in res)
    wall_ms = statistics.median(r["wall_ms"] for r in res)
    link_peak = pinned_d2h_peak(pd, eng, flush, copy)
    d2h = statistics.mean(r["precopy_bytes"] + r["delta_bytes"] for r in res)
    step_ms, stw_ms, wall_ms, per_rank = rank_summary(dist, local, step_ms, stw_ms, wall_ms,
                                                      d2h / (step_ms * 1e-3) / 1e9)
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(aggregate_value(world, total, step_ms), 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "stw_ms": round(stw_ms, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": bench_config(wl, world),
            "run": {"d2h_bytes_per_step": int(d2h), "packs_per_step": res[-1]["packs"], "host_cpus": numa,
                    "mode": "cache-cycled pre-copy (pos_precopy_stream), app idle at the checkpoint"},
            "stages_ms": {"hash_waves_ms": round(statistics.mean(r["hash_ms"] for r in res), 3)},
            "per_rank": per_rank,
            "host_link_aggregate_gbps": round(sum(r["host_link_gbps"] for r in per_rank), 2),
            **({"peer_cache": {"device": peer, "bytes": int(args.peer_cache_gb * 1e9),
                               "capture_ms": round(statistics.mean(r["capture_ms"] for r in res), 3),
                               "note": ("capture = every pack in the peer's HBM (the application may resume); "
                                        "peer == this GPU on a 1-GPU box (D2D slots, not NVLink)"
                                        if peer == local else
                                        "capture = every pack in the peer's HBM over NVLink")}}
               if peer is not None else {}),
            "host_link": {"bound": "pcie", "achieved": round(d2h / (step_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                          "peak": round(link_peak, 2), "frac": round(d2h / (step_ms * 1e-3) / 1e9 / link_peak, 4),
                          "achieved_over": "whole step (D2H-bound)",
                          "peak_source": "best of 5 pinned cudaMemcpyAsync D2H of 256 MiB, measured in this run"},
            "e2e": {"value": round(aggregate_value(world, total, wall_ms), 3), "unit": "GB/s",
                    "h2d_bytes_per_step": len(bufs), "d2h_bytes_per_step": int(d2h),
                    "how": "host wall clock around DumpEngine.precopy_stream incl. the in-order sink"},
            "clocks": clk.summary(),
        }
    eng.close()
    return out


def cpu_breakdown(wl: Workload, threads: int, sample_bytes: int) -> dict:
    """SURVEY §8(d)'s CPU path timed function by function on the same bounded
    sample, on 1 thread and on `threads`: the reference's crc32 per 64 KiB
    chunk (crc32.hpp:26-34), its dump loop (crc32 + chunk_copied capture,
    cr.hpp:481-504), and -- single-threaded, as in the reference --
    write_image / read_image of the sample as Inline records
    (image.hpp:136-361).  GB/s of sample bytes, best of 3."""
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor
    from oracle_ctypes import oracle, reference, Rec, Alloc
    ref, orc = reference(), oracle()
    if ref is None:
        return {}
    idx, acc = [], 0
    for i, n in enumerate(wl.sizes):
        if acc >= sample_bytes:
            break
        idx.append(i)
        acc += n
    bufs = []
    for i in idx:
        a = np.empty(wl.sizes[i], np.uint8)
        orc.or_fill_bytes(9000 + i, a.ctypes.data, a.size)
        bufs.append(a)

    def best(fn, reps=3):
        t = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            t.append(time.perf_counter() - t0)
        return round(acc / min(t) / 1e9, 3)

    # the chunks of the sample, dealt in contiguous ranges over the threads
    # (ctypes drops the GIL inside ref_crc32)
    chunks = [(a.ctypes.data + o, min(CHUNK, a.size - o)) for a in bufs for o in range(0, a.size, CHUNK)]

    def crc_range(t, nt):
        for p, n in chunks[len(chunks) * t // nt:len(chunks) * (t + 1) // nt]:
            ref.ref_crc32(p, n)

    def crc_all(nt):
        if nt == 1:
            crc_range(0, 1)
        else:
            with ThreadPoolExecutor(nt) as ex:
                list(ex.map(lambda t: crc_range(t, nt), range(nt)))

    sizes = np.array([a.size for a in bufs], np.uint64)
    ptrs = (C.c_void_p * len(bufs))(*[a.ctypes.data for a in bufs])
    nch = sum((a.size + CHUNK - 1) // CHUNK for a in bufs)
    prev, cur, fl = np.zeros(nch, np.uint32), np.zeros(nch, np.uint32), np.zeros(nch, np.uint8)
    st = ref.ref_state_create(len(bufs), sizes.ctypes.data, ptrs, CHUNK)
    out = {"sample": f"{len(bufs)} buffers, {acc} B", "threads": threads,
           "crc32_per_chunk": {"1": best(lambda: crc_all(1)), str(threads): best(lambda: crc_all(threads))},
           "dump_loop_all_dirty": {
               "1": best(lambda: ref.ref_state_dump(st, prev.ctypes.data, 0, cur.ctypes.data, fl.ctypes.data, 1)),
               str(threads): best(lambda: ref.ref_state_dump(st, prev.ctypes.data, 0, cur.ctypes.data,
                                                             fl.ctypes.data, threads))}}
    # materialize's write_content of Inline records (cr.hpp:1062-1070, buffer.hpp:80-83): the
    # restore-side byte move, one buffer per thread
    def write_all(nt):
        if nt == 1:
            for k, a in enumerate(bufs):
                ref.ref_state_write(st, k, 0, a.ctypes.data, a.size)
        else:
            with ThreadPoolExecutor(nt) as ex:
                list(ex.map(lambda k: ref.ref_state_write(st, k, 0, bufs[k].ctypes.data, bufs[k].size),
                            range(len(bufs))))
    out["materialize_write_content"] = {"1": best(lambda: write_all(1)), str(threads): best(lambda: write_all(threads))}
    ref.ref_state_destroy(st)
    recs = (Rec * len(bufs))()
    for k, a in enumerate(bufs):
        recs[k].handle, recs[k].kind = k + 1, 0
        recs[k].inline_bytes, recs[k].inline_len = a.ctypes.data, a.nbytes
    allocs = (Alloc * len(bufs))(*[Alloc(k + 1, 0x7000_0000_0000 + (k << 30), a.nbytes) for k, a in enumerate(bufs)])
    args = [4096, None, 0, recs, len(bufs), allocs, len(bufs), None, 0, 0, len(bufs) + 1, 0, None, 0]
    n = ref.ref_write_image(*args, None, 0)
    img = np.empty(n, np.uint8)
    out["write_image"] = best(lambda: ref.ref_write_image(*args, img.ctypes.data, n))
    out["read_image"] = best(lambda: ref.ref_read_image_check(img.ctypes.data, n))
    return out


def run_reference(args, wl: Workload, world, rank):
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    v, ms, sample, kind = cpu_reference_run(wl, args.steps, args.warmup, threads, args.ref_sample_bytes)
    breakdown = cpu_breakdown(wl, threads, min(args.ref_sample_bytes, 64 << 20))
    return {
        "metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": bench_config(wl, world),
        "run": {"executes": "rank 0 only, on the host cores", "cpu_model": cpu_model()},
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_breakdown_gbps": breakdown,
    }


def relaunch_under_torchrun(n: int) -> None:
    """`bench.py --gpus N` without a torchrun environment: re-exec as N ranks
    (one process per GPU) on this node."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c1", "c2", "c3", "c4", "c5"], default="c5",
                    help="c5 (default): BASELINE configs[4], the metric's own configuration (120 GB per GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace", action="store_true", help="per-step device timeline on stderr")
    ap.add_argument("--no-host-apply", action="store_true", help="diagnostic: skip the host image apply")
    ap.add_argument("--waves", type=int, default=0,
                    help="pre-copy pipeline waves (0 = the workload's default: c2 1, c1 4, c3/c4/c5 16)")
    ap.add_argument("--mode", choices=["pack", "direct", "stream"], default="direct",
                    help="direct: runs of shipped chunks copied by the copy engine straight into the pinned host "
                         "image; pack: POSD packs D2H + host apply; stream: cache-cycled packs (c3/c5, with "
                         "--peer-cache-gb through a peer GPU's HBM)")
    ap.add_argument("--ring", type=int, default=3, help="pinned landing buffers (rotated per step)")
    ap.add_argument("--ckpt-priority", type=int, default=1, help="1: dump stream at the highest stream priority")
    ap.add_argument("--app-priority", type=int, default=0, help="1: the application's stream at the highest priority")
    ap.add_argument("--ref-sample-bytes", type=int, default=1 << 30,
                    help="CPU reference: bounded sample (a prefix of the buffer set) of at least this many bytes")
    ap.add_argument("--no-window", action="store_true", help="diagnostic: no application kernels during the dump")
    ap.add_argument("--no-app-load", action="store_true",
                    help="skip the application-load checkpoints (after the timed steps; e.g. under ncu)")
    ap.add_argument("--hash-sms", type=int, default=0,
                    help="SMs the hash may occupy (0 = all); the application's kernels get the rest")
    ap.add_argument("--drain-priority", type=int, default=-1, help="host-leg stream priority (default: as the dump)")
    ap.add_argument("--slice-mib", type=int, default=0, help="host-leg slice size (default: the engine's 16 MiB)")
    ap.add_argument("--image-align", type=int, default=0,
                    help="alignment of each buffer's range in the host image (default 256 B)")
    ap.add_argument("--o2-digest2", action="store_true",
                    help="a second, non-linear chunk digest beside CRC-32 in the O2 compare")
    ap.add_argument("--window", type=int, default=0, help="host-leg slices in flight (default: the engine's 3)")
    ap.add_argument("--peer-cache-gb", type=float, default=0.0,
                    help="--mode stream: NVLink peer-GPU cache of this many GB on the next GPU (config 5)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if os.environ.get("BENCH_WATCHDOG_S"):  # diagnostics: every thread's stack if the run hangs
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["BENCH_WATCHDOG_S"]), exit=True)
    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and env_world is None:
        relaunch_under_torchrun(args.gpus)
    if env_world is not None and int(env_world) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={env_world}: launch one rank per GPU")
    if args.waves <= 0:
        args.waves = {"c1": 4, "c3": 16, "c4": 16, "c5": 16}.get(args.workload, 1)
    world, rank, local, dist = dist_setup()
    wl = Workload(args.workload)
    if args.impl != "reference" and args.mode == "direct" and wl.name in ("c3", "c5"):
        # every rank keeps its own pinned host image of its whole state: when
        # the node's memory cannot hold world x state, the states stream
        # through pinned landing slots instead (same bytes over each link)
        need = world * wl.total * 1.05
        avail = mem_available()
        if avail is not None and avail < need:
            log(f"host memory {avail / 1e9:.0f} GB < {need / 1e9:.0f} GB for {world} host images: --mode stream")
            args.mode = "stream"
    if args.impl == "reference":
        out = run_reference(args, wl, world, rank)
    elif args.mode == "stream":
        if wl.name not in ("c3", "c5"):
            raise SystemExit("--mode stream is for the states larger than the cache (c3, c5)")
        out = run_gpu_stream(args, wl, world, rank, local, dist)
    else:
        out = run_gpu(args, wl, world, rank, local, dist)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
