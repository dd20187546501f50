# 768-thread (24 warps/SM) hash variant with 2-way chunk segments vs the default
for cfg in 512x8 768x4; do POSDUMP_HASH_CFG=$cfg timeout 300 python tools/probe_hash.py; done > gpurun_out/h768.txt 2>&1
POSDUMP_HASH_CFG=768x4 POSDUMP_NSEG=1 timeout 300 python tools/probe_hash.py >> gpurun_out/h768.txt 2>&1
cat gpurun_out/h768.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "stream or digests" 2>&1 | tail -2
POSDUMP_HASH_CFG=768x4 timeout 600 python -m pytest tests -m gpu -x -q -k "stream or digests or direct" 2>&1 | tail -2
