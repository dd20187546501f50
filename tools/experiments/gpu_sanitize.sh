# compute-sanitizer memcheck / racecheck over a subset of the GPU parity tests, then the full GPU suite twice (flakiness)
export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 99 python -m pytest tests -m gpu -x -q -k "digest_layouts or delta_copy or direct_precopy_into_image or scatter or final_stop or provenance" > gpurun_out/memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/memcheck.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 99 python -m pytest tests -m gpu -x -q -k "chunk_digests_and_epoch or tiled_scan or o1_verdicts" > gpurun_out/racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/racecheck.txt
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
