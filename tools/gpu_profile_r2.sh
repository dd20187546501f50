# Round-2 profiles of the default bench (BASELINE config 5): the launch list of
# the bench command itself, and ncu --set full of one wave's hash and of the
# STW gather (standalone: tools/profile_c5_wave.py).
P=gpurun_out/r2prof; mkdir -p $P
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $P/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-app-load > $P/launches_c5.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_chunks -s 2 -c 1 -o $P/hash_c5wave \
  python tools/profile_c5_wave.py > $P/hash_c5wave.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_bulk -s 1 -c 1 -o $P/gather_c5 \
  python tools/profile_c5_wave.py > $P/gather_c5.out 2>&1
python tools/profile_c5_wave.py > $P/c5wave_timing.txt 2>&1
ls -la $P
