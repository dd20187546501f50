P=gpurun_out/r2e; mkdir -p $P
for w in c2 c1; do
timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline --trace > $P/${w}_trace.jsonl 2> $P/${w}_trace.err; grep '^{' $P/${w}_trace.err | tail -2
timeout 300 python bench.py --workload $w --steps 20 --no-cpu-baseline > $P/${w}.jsonl 2> $P/${w}.err; cut -c1-300 $P/${w}.jsonl
done
