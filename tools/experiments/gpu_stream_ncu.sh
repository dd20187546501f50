# ncu capture of k_hash_stream vs k_hash_chunks on 1526 x 64 KiB chunks (tools/probe_hash.py)
mkdir -p gpurun_out/sncu
PROBE_CHUNKS=1526 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hash -s 3 -c 1 -o gpurun_out/sncu/stream python tools/probe_hash.py > /dev/null 2>&1
PROBE_CHUNKS=1526 POSDUMP_HASH_STREAM=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hash -s 3 -c 1 -o gpurun_out/sncu/chunks python tools/probe_hash.py > /dev/null 2>&1
ls -la gpurun_out/sncu
