# Bench variants on one B200 box (under gpurun), one summary line each:
#   bash tools/gpu_sweep.sh "--workload c2 --waves 1" "--workload c1 --waves 4" ...
# (round-2 sweeps: host-leg slice/window, waves, pack vs direct, app load --
#  their outputs are under profiles/r2/)
P=gpurun_out/sweep; mkdir -p $P
for v in "$@"; do
  timeout 900 python bench.py --no-cpu-baseline --steps ${STEPS:-5} $v > $P/b.jsonl 2> $P/b.err
  python -c "
import json; d=json.loads(open('$P/b.jsonl').read().splitlines()[-1])
print('$v', d['value'], d['ms_per_step'], d['stw_ms'], d['e2e']['value'], d['host_link']['frac'], d['host_link']['peak'])" || tail -3 $P/b.err
done
