# c2 profiles (under gpurun): GPU tests, the c2 bench line, ncu --set full of the
# tiled scan and of the STW gather inside the c2 bench.
P=gpurun_out/c2prof; mkdir -p $P
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --workload c2 --steps 20 --no-cpu-baseline > $P/c2.jsonl 2> $P/c2.err
python -c "
import json; d=json.loads(open('$P/c2.jsonl').read().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['stw_ms'], d['host_link'], d['stages_ms'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tiles -s 6 -c 1 -o $P/scan_c2 \
  python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_scan.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_bulk -s 4 -c 1 -o $P/gather_c2 \
  python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_gather.out 2>&1
ls -la $P
