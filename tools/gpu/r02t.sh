set -x
timeout 600 python tools/small_view.py --kernels lazy,lazy1,batch8x1,batch8x2,refill1,static --tiles 0,32 --iters 20 > gpurun_out/r02t_small_view.jsonl 2> gpurun_out/r02t_small_view.err; echo "rc=$?"
timeout 100 python tools/host_overhead.py > gpurun_out/r02t_host_overhead.txt 2>&1
