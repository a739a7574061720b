set -x
timeout 900 python tools/small_view.py --kernels static,lazy1,lazy2,batch4x1,batch4x2,batch8x1,batch8x2,refill1,adaptive1 --tiles 0,128 > gpurun_out/r02v_small_view.jsonl 2> gpurun_out/r02v_small_view.err; echo "rc=$?"
timeout 300 python tools/small_view.py --kernels lazy1,lazy2 --lanes 4,8,16,24,32 > gpurun_out/r02v_small_view_lanes.jsonl 2>&1; echo "rc=$?"
timeout 300 python tools/small_view.py --kernels static,lazy1,batch8x1 --scheme cyclic > gpurun_out/r02v_small_view_cyclic.jsonl 2>&1; echo "rc=$?"
