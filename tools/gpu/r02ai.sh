set -x
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_abi.py -x -q -m gpu -p no:cacheprovider -k "fused or c1_all or random_small or edge or batched or full_size or small_view" > gpurun_out/r02ai_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02ai_pytest.log
for fy in 0 -1; do
timeout 900 python tools/sweep.py --configs C1,C2,C3,C4,C5 --kernels refill --schemes block --steps 10 --warmup 2 --fused-y=$fy > gpurun_out/r02ai_sweep_fy$fy.jsonl 2>&1; echo "rc=$?"
done
