# k_hash_stream: parity, then size scaling and the default bench against the per-chunk kernel
timeout 600 python -m pytest tests -m gpu -x -q -k "stream or digests or unaligned or direct or pipelined or c1_full" 2>&1 | tail -5
timeout 300 python tools/probe_hash.py > gpurun_out/stream_scale.txt 2>&1
POSDUMP_HASH_STREAM=0 timeout 300 python tools/probe_hash.py >> gpurun_out/stream_scale.txt 2>&1
cat gpurun_out/stream_scale.txt
python tools/sweep.py ":: --steps 30 --warmup 3" "POSDUMP_HASH_STREAM=0 :: --steps 30 --warmup 3" \
  ":: --steps 20 --warmup 3 --workload c1" "POSDUMP_HASH_STREAM=0 :: --steps 20 --warmup 3 --workload c1" > gpurun_out/stream_bench.txt 2>&1
cat gpurun_out/stream_bench.txt
