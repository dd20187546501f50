# compute-sanitizer memcheck over the whole GPU suite (child processes included)
export PYTHONUNBUFFERED=1
timeout 2400 compute-sanitizer --tool memcheck --target-processes all --print-limit 30 --error-exitcode 99 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/memcheck_all.txt 2>&1; echo "memcheck rc=$?"
grep -E "passed|failed|ERROR SUMMARY" gpurun_out/memcheck_all.txt | tail -5
