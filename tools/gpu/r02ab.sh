set -x
timeout 300 python tools/host_overhead.py > gpurun_out/r02ab_host_overhead.json 2>&1; echo "rc=$?"
for rep in 1 2; do
timeout 900 python tools/sweep.py --configs C2,C3,C5 --kernels refill --schemes block --steps 10 --warmup 2 > gpurun_out/r02ab_sweep_new_$rep.jsonl 2>&1; echo "rc=$?"
MANDEL_LIB=paper_2007_00745_b200/libmandel_ab.so timeout 900 python tools/sweep.py --configs C2,C3,C5 --kernels refill --schemes block --steps 10 --warmup 2 > gpurun_out/r02ab_sweep_old_$rep.jsonl 2>&1; echo "rc=$?"
done
timeout 1500 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -p no:cacheprovider -k "c1_all or random_small or edge or batched or full_size_whole_map or fp32_packed" > gpurun_out/r02ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02ab_pytest.log
