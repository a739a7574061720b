set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ap_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02ap_smoke.log
timeout 1800 python -m pytest tests -x -q -m gpu -p no:cacheprovider --durations=5 > gpurun_out/r02ap_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02ap_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02ap_bench_default.json 2> gpurun_out/r02ap_bench_default.err; echo "bench default rc=$?"
