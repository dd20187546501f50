P=gpurun_out/r2d; mkdir -p $P
timeout 120 python tools/probe_ship.py 2>&1 | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/ship_launches.csv python tools/probe_ship.py > /dev/null 2>&1; cut -d, -f5 $P/ship_launches.csv | sort | uniq -c
