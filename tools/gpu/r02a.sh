set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02a_pytest_gpu.log
./tools/fp_peak > gpurun_out/r02a_fp_peak.json 2>&1; cat gpurun_out/r02a_fp_peak.json
for c in C2 C4 C5 C3; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_$c.json 2> gpurun_out/r02a_bench_$c.err; echo "bench $c rc=$?"; done
