set -x
timeout 600 python tools/small_view.py --kernels static,lazy1,refill > gpurun_out/r02ad_small_view_new.jsonl 2>&1; echo "rc=$?"
MANDEL_LIB=paper_2007_00745_b200/libmandel_ab.so timeout 600 python tools/small_view.py --kernels static > gpurun_out/r02ad_small_view_old.jsonl 2>&1; echo "rc=$?"
timeout 600 python tools/sweep.py --configs C1,C2 --kernels static --schemes block,cyclic --steps 10 --warmup 2 > gpurun_out/r02ad_sweep_static.jsonl 2>&1; echo "rc=$?"
timeout 900 python tools/sweep.py --configs C3 --kernels batch8x1,batch8x2,refill --pack 1,0 --schemes block --steps 10 --warmup 2 > gpurun_out/r02ad_sweep_c3.jsonl 2>&1; echo "rc=$?"
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -p no:cacheprovider -k "static or c1_all" > gpurun_out/r02ad_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02ad_pytest.log
