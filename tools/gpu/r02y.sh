set -x
export MANDEL_LIB=paper_2007_00745_b200/libmandel_trace.so
timeout 300 python tools/trace_view.py --config C1 --kernels lazy1,lazy2,batch8x1,static --orders=-1,1 > gpurun_out/r02y_trace_c1.jsonl 2> gpurun_out/r02y_trace.err; echo "rc=$?"
timeout 300 python tools/trace_view.py --config C2 --kernels refill --orders=1 > gpurun_out/r02y_trace_c2.jsonl 2>> gpurun_out/r02y_trace.err; echo "rc=$?"
timeout 300 python tools/trace_view.py --config C2 --kernels refill --orders=-1 --tile 64 >> gpurun_out/r02y_trace_c2.jsonl 2>> gpurun_out/r02y_trace.err; echo "rc=$?"
