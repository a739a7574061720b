set -x
export MANDEL_LIB=paper_2007_00745_b200/libmandel_trace.so
timeout 300 python tools/trace_view.py --config C1 --kernels lazy1,lazy2,batch8x1,static --orders -1,1 > gpurun_out/r02x_trace_c1.jsonl 2> gpurun_out/r02x_trace.err; echo "rc=$?"
timeout 300 python tools/trace_view.py --config C2 --kernels refill --orders -1 >> gpurun_out/r02x_trace_c2.jsonl 2>> gpurun_out/r02x_trace.err; echo "rc=$?"
timeout 300 python tools/trace_view.py --config C4 --kernels refill --orders -1 >> gpurun_out/r02x_trace_c4.jsonl 2>> gpurun_out/r02x_trace.err; echo "rc=$?"
unset MANDEL_LIB
timeout 900 python tools/sweep.py --configs C2,C3,C4,C5 --kernels refill --schemes block --order=-1,1 --steps 5 --warmup 2 > gpurun_out/r02x_sweep.jsonl 2> gpurun_out/r02x_sweep.err; echo "rc=$?"
