P=gpurun_out/r2l; mkdir -p $P
timeout 600 python bench.py --gpus 2 --workload c2 --steps 5 --warmup 3 > $P/g2.jsonl 2> $P/g2.err; cut -c1-400 $P/g2.jsonl; tail -3 $P/g2.err
timeout 600 python bench.py --gpus 2 --impl reference --workload c2 --steps 2 --warmup 1 > $P/g2ref.jsonl 2> $P/g2ref.err; cut -c1-300 $P/g2ref.jsonl; tail -2 $P/g2ref.err
