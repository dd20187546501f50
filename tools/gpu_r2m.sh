P=gpurun_out/r2m; mkdir -p $P
for v in "--workload c2 --waves 1" "--workload c2 --waves 2" "--workload c2 --waves 4" "--workload c2 --waves 8" "--workload c1 --waves 2" "--workload c1 --waves 4" "--workload c1 --waves 8" "--workload c1 --waves 16"; do
  timeout 900 python bench.py --no-cpu-baseline --steps 20 $v > $P/b.jsonl 2> $P/b.err
  python -c "
import json; d=json.loads(open('$P/b.jsonl').read().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['e2e']['value'], d['host_link']['frac'])" || tail -3 $P/b.err
done
