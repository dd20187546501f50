P=gpurun_out/r2i; mkdir -p $P
for v in "" "--window 8" "--slice-mib 64" "--slice-mib 64 --window 6" "--no-window" "--hash-sms 37"; do
  timeout 600 python bench.py --no-cpu-baseline --steps 3 $v > $P/b.jsonl 2> $P/b.err
  python -c "
import json; d=json.loads(open('$P/b.jsonl').read().splitlines()[-1]); print('$v', d['value'], d['host_link']['precopy_leg_gbps'], d['host_link']['peak'], d['stw_ms'])"
done
