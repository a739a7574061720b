# round 2h: templated staging (default: staged only for a remote map) -- stage A/B sweep first,
# then the whole -m gpu suite
set -x
for rep in 1 2; do
timeout 900 python tools/sweep.py --configs C2,C5,C3,C4 --kernels refill --schemes block --stage 1,0 --steps 10 >> gpurun_out/r02h_sweep_stage.jsonl 2>> gpurun_out/r02h_sweep.err
done
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02h_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02h_pytest_gpu.log
