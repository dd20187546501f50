P=gpurun_out/r2h; mkdir -p $P
timeout 600 python tools/probe_image_d2h.py > $P/image_d2h.txt 2>&1; tail -1 $P/image_d2h.txt
for k in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 4 > $P/bench_c5_$k.jsonl 2> $P/bench_c5_$k.err; cut -c1-200 $P/bench_c5_$k.jsonl; done
