P=gpurun_out/r2j; mkdir -p $P
for w in c2 c5; do
timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 3 > $P/$w.jsonl 2> $P/$w.err
python -c "
import json; d=json.loads(open('$P/$w.jsonl').read().splitlines()[-1]); print('$w', d['value'], d['stw_ms'], json.dumps(d.get('app_interference')))"
tail -3 $P/$w.err
done
