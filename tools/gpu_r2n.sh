P=gpurun_out/r2n; mkdir -p $P
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pregather or delta_copy or direct" 2>&1 | tail -3
for w in c2 c5; do
timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 3 > $P/$w.jsonl 2> $P/$w.err
python -c "
import json; d=json.loads(open('$P/$w.jsonl').read().splitlines()[-1]); print('$w', d['value'], d['stw_ms'], d.get('stw_eager_capture'), d['image_parity'])" || tail -5 $P/$w.err
done
