P=gpurun_out/r2k; mkdir -p $P
for v in "--workload c2 --mode pack --steps 10" "--workload c1 --mode pack --steps 10" "--workload c5 --mode stream --steps 3"; do
  timeout 900 python bench.py --no-cpu-baseline $v > $P/b.jsonl 2> $P/b.err
  python -c "
import json; d=json.loads(open('$P/b.jsonl').read().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['stw_ms'], d['host_link']['frac'], d['stages_ms'])" || tail -3 $P/b.err
done
