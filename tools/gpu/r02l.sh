set -x
timeout 900 python tools/hang_probe.py --schemes fcfs,block --ns 1,3 --kernels refill,lazy2 --stage 1,0 --sizes 512x97,800x800 --it 2000 --reps 2 --extra '{"tile_rows": 1}' > gpurun_out/r02l_hang.jsonl 2>&1
grep -c HANG gpurun_out/r02l_hang.jsonl; grep -v '"bad\\": 0' gpurun_out/r02l_hang.jsonl | cut -c1-400
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline --no-schemes > gpurun_out/r02l_bench_c1.json 2>&1; echo "bench rc=$?"
grep -o '"value": [0-9.]*' gpurun_out/r02l_bench_c1.json | head -2; grep -o '"render_ms": {[^}]*}' gpurun_out/r02l_bench_c1.json
timeout 900 python tools/sweep.py --configs C2,C5,C3,C4 --kernels refill --schemes block,fcfs --stage 0 --steps 10 > gpurun_out/r02l_sweep.jsonl 2> gpurun_out/r02l_sweep.err; echo "sweep rc=$?"
