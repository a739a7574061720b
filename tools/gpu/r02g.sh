# round 2g: eviction-based store staging -- whole -m gpu suite, stage A/B sweep
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02g_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02g_pytest_gpu.log
for rep in 1 2; do
timeout 900 python tools/sweep.py --configs C2,C5,C3,C4 --kernels refill --schemes block --stage 1,0 --steps 10 >> gpurun_out/r02g_sweep_stage.jsonl 2>> gpurun_out/r02g_sweep.err
done
