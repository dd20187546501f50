# A/B of the c5 bench on one box: HEAD vs an older build in _ab/ (same box, back to back)
P=gpurun_out/ab; mkdir -p $P
nvidia-smi --query-gpu=name,clocks.sm,pcie.link.gen.current,pcie.link.width.current --format=csv
for i in 1 2; do
  timeout 300 python bench.py --steps 3 --no-cpu-baseline > $P/head_$i.jsonl 2> $P/head_$i.err
  (cd _ab && timeout 300 python bench.py --steps 3 --no-cpu-baseline > ../$P/old_$i.jsonl 2> ../$P/old_$i.err)
done
timeout 300 python bench.py --steps 3 --no-cpu-baseline --no-window > $P/head_nowin.jsonl 2> $P/head_nowin.err
for f in $P/*.jsonl; do python -c "
import json,sys; d=json.loads(open('$f').read().splitlines()[-1]); print('$f', d['value'], d['host_link']['peak'], d['host_link']['precopy_leg_gbps'], d['stw_ms'])"; done
