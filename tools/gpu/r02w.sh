set -x
timeout 600 python tools/small_view.py --kernels lazy1,lazy2,batch8x1,batch8x2,refill --order 1,-1 --tiles 0,32 > gpurun_out/r02w_small_view.jsonl 2> gpurun_out/r02w_small_view.err; echo "rc=$?"
timeout 900 python tools/sweep.py --configs C2,C3,C4,C5 --kernels refill --schemes block --order -1,1 --steps 5 --warmup 2 > gpurun_out/r02w_sweep.jsonl 2> gpurun_out/r02w_sweep.err; echo "rc=$?"
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -p no:cacheprovider -k "cost_ordered or c1_all or max_logical or edge or random_small" > gpurun_out/r02w_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02w_pytest.log
