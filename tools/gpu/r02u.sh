set -x
timeout 600 python tools/small_view.py --kernels lazy,lazy1,batch8x1,static --tiles 0,32 > gpurun_out/r02u_small_view.jsonl 2> gpurun_out/r02u_small_view.err; echo "rc=$?"
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_abi.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r02u_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02u_pytest.log
