set -x
timeout 1200 python tools/sweep.py --configs C2,C3,C5 --kernels refill --schemes block --order=-1,1 --tiles 128,256,512 --steps 5 --warmup 2 > gpurun_out/r02z_sweep.jsonl 2> gpurun_out/r02z_sweep.err; echo "rc=$?"
timeout 600 python tools/sweep.py --configs C4 --kernels refill --schemes block --order=-1,1 --tiles 128,256,512 --steps 5 --warmup 2 >> gpurun_out/r02z_sweep.jsonl 2>> gpurun_out/r02z_sweep.err; echo "rc=$?"
