timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
S="--steps 20 --warmup 3"
python tools/sweep.py ":: $S --mode pack" ":: $S" ":: --steps 5 --warmup 3 --trace" 2>&1 | tee gpurun_out/scan2.txt
ncu --set full --clock-control none --import-source on -k regex:k_pack_scan -s 6 -c 1 -o gpurun_out/scan_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/scan_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/scan_c2_source.csv 2>/dev/null; ls -la gpurun_out/scan_c2*
