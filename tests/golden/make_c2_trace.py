"""BASELINE config 2 workload: the reference's own generator (gen_workload,
workload.hpp:162-410) for the resnet-train-desk profile (workload.hpp:485-494:
224 buffers, write_locality 0.5, param_fraction 0.3, 2 streams) rescaled to
~100 MB and to real kernel durations (p50 50 us, p99 200 us),
reduced to what the dump path consumes: buffer sizes, the H2D-loaded
parameter set, and per iteration the ordered kernels (stream, duration, true
write set) between device synchronizes.  Output: tests/golden/c2_resnet_trace.json
(committed; the GPU box replays it without /root/reference).
"""
import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_ctypes import reference  # noqa: E402

ref = reference()
assert ref is not None, "build oracle/_ref first (make -C oracle)"
args = (b"resnet-train-desk", 100_000_000, 50_000, 200_000, 1)
n = ref.ref_gen_workload(*args, None, 0)
buf = C.create_string_buffer(n)
ref.ref_gen_workload(*args, buf, n)
calls = [json.loads(l) for l in buf.raw[:n].decode().splitlines() if l]
sizes, params, phases, cur = [], [], [], []
for c in calls:
    k = c["kind"]
    if k == "Malloc":
        sizes.append(c["bytes"])
    elif k == "MemcpyH2D":
        params.append(c["true_writes"][0])
    elif k in ("LaunchKnown", "LaunchOpaque"):
        cur.append([c["stream"], c["duration_ns"], sorted(set(c["true_writes"]))])
    elif k == "DeviceSynchronize" and cur:
        phases.append(cur)
        cur = []
if cur:
    phases.append(cur)
out = {"profile": "resnet-train-desk", "generator": "gpucrsim::gen_workload", "seed": 1,
       "total_bytes": sum(sizes), "sizes": sizes, "params": params, "phases": phases}
json.dump(out, open(os.path.join(HERE, "c2_resnet_trace.json"), "w"))
print(len(sizes), "buffers", sum(sizes), "bytes;", len(params), "params;",
      len(phases), "phases;", sum(len(p) for p in phases), "kernels")
