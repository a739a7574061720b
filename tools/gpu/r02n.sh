set -x
python tools/host_overhead.py > gpurun_out/r02n_host_overhead.txt 2>&1; cat gpurun_out/r02n_host_overhead.txt
timeout 900 python tools/sweep.py --configs C1 --kernels refill,batch8x1,refill1,refill2,lazy2,batch4x2 --schemes block --tiles 0,32,64,128 --steps 50 > gpurun_out/r02n_sweep_c1.jsonl 2> gpurun_out/r02n_sweep.err; echo "sweep rc=$?"
timeout 900 python tools/sweep.py --configs C1 --kernels refill --schemes block --ctas 0,1,2 --tile-rows 0,4,2 --steps 50 >> gpurun_out/r02n_sweep_c1.jsonl 2>> gpurun_out/r02n_sweep.err
timeout 900 python tools/sweep.py --configs C3 --kernels refill --schemes block,fcfs --steps 10 >> gpurun_out/r02n_sweep_c1.jsonl 2>> gpurun_out/r02n_sweep.err
