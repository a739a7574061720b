set -x
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline --no-schemes > gpurun_out/r02m_bench_c1.json 2>&1; echo "bench rc=$?"
grep -o '"render_ms": {[^}]*}' gpurun_out/r02m_bench_c1.json
timeout 900 python tools/sweep.py --configs C2,C5,C3,C4 --kernels refill --schemes block,fcfs --steps 10 > gpurun_out/r02m_sweep.jsonl 2> gpurun_out/r02m_sweep.err; echo "sweep rc=$?"
timeout 900 python tools/sweep.py --configs C3 --kernels refill --schemes block --ctas 0,4,3 --steps 10 >> gpurun_out/r02m_sweep.jsonl 2>> gpurun_out/r02m_sweep.err; echo "sweep rc=$?"
