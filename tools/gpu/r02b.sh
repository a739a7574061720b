# round 2b: bench contract tests with the new keys, the default bench line, full ncu
# captures (with source) of the C3 and C4 escape kernels
set -x
timeout 900 python -m pytest tests/test_bench_gpu.py -x -q -p no:cacheprovider > gpurun_out/r02b_pytest_bench.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02b_pytest_bench.log
timeout 600 python bench.py > gpurun_out/r02b_bench_default.json 2> gpurun_out/r02b_bench_default.err; echo "bench rc=$?"
for c in C3 C4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:escape_ -s 3 -c 1 \
    -o gpurun_out/r02b_${c}_full python bench.py --profile --config $c --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r02b_${c}_ncu.log 2>&1; echo "ncu $c rc=$?"
done
