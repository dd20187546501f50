timeout 300 ./tools/runs_micro > gpurun_out/runs_micro.txt 2>&1; cat gpurun_out/runs_micro.txt
bash tools/gpu_check.sh
