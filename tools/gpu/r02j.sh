# round 2j: find the test that stalls the -m gpu suite (per-test timeout, verbose, durations)
set -x
timeout 2400 python -m pytest tests -m gpu -x -v -p no:cacheprovider --timeout=300 --timeout-method=thread --durations=40 > gpurun_out/r02j_pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "PASSED|FAILED|Timeout|ERROR" gpurun_out/r02j_pytest_gpu.log | tail -5
