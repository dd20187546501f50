P=gpurun_out/r2prof; mkdir -p $P
python tools/profile_c5_wave.py 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_bulk -s 2 -c 1 -o $P/scatter_c5 python tools/profile_c5_wave.py > $P/scatter_c5.out 2>&1; tail -1 $P/scatter_c5.out
