#!/usr/bin/env python3
"""Tuning sweep (GPU box): runs bench.py under env/arg variants and prints one
compact line per run: value, ms/step, stw, hash launch ms, stages, e2e.
usage: python tools/sweep.py 'ENV=..;ENV2=.. :: --workload c1 --waves 4' ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for spec in sys.argv[1:]:
    env_s, _, args = spec.partition("::")
    env = dict(os.environ)
    for kv in filter(None, (x.strip() for x in env_s.split(";"))):
        k, _, v = kv.partition("=")
        env[k] = v
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", *args.split()]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    line = next((l for l in p.stdout.splitlines() if l.startswith("{")), None)
    if not line:
        print(f"{spec!r}: FAILED rc={p.returncode} {p.stderr[-800:]}", flush=True)
        continue
    r = json.loads(line)
    out = {"value": r["value"], "ms": r["ms_per_step"], "stw": r.get("stw_ms"), "stw_dev": r.get("stw_device_clock_ms"),
           "e2e": r.get("e2e", {}).get("value"), "frac": r.get("roofline", {}).get("frac"),
           "stages": r.get("stages_ms"), "link": r.get("host_link", {}).get("frac")}
    print(f"{spec!r}: {json.dumps(out)}", flush=True)
    if "--trace" in args:
        print("\n".join(p.stderr.strip().splitlines()[-3:]), flush=True)
