set -x
timeout 600 python tools/small_view.py --kernels lazy,lazy1,batch8x1,batch8x2,static --tiles 0,32,64 --ctas 0,2,4 --iters 20 > gpurun_out/r02s_small_view.jsonl 2> gpurun_out/r02s_small_view.err; echo "rc=$?"
timeout 300 python tools/small_view.py --kernels lazy,batch8x2 --lanes 8,16,24 --tiles 0,32 > gpurun_out/r02s_small_view_lanes.jsonl 2>&1; echo "rc=$?"
