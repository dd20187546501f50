# k_hash_chunks size scaling per variant (tools/probe_hash.py)
for cfg in default 512t6 384x12; do
  if [ $cfg = default ]; then timeout 300 python tools/probe_hash.py; else POSDUMP_HASH_CFG=$cfg timeout 300 python tools/probe_hash.py; fi
done > gpurun_out/hashscale.txt 2>&1
for ns in 2 4; do POSDUMP_NSEG=$ns timeout 300 python tools/probe_hash.py; done >> gpurun_out/hashscale.txt 2>&1
cat gpurun_out/hashscale.txt
