set -x
V1="-2.5,1.5,-2.0,2.0,800,800,200"
V4="-0.743693887,-0.743593887,0.131775904,0.131875904,800,800,2000"
for v in $V1 $V4; do
timeout 300 python tools/small_view.py --view=$v --kernels refill,batch8x1 >> gpurun_out/r02ah_small_views.jsonl 2>&1; echo "rc=$?"
done
timeout 300 python bench.py --config C1 --steps 200 --warmup 5 > gpurun_out/r02ah_bench_C1.json 2> gpurun_out/r02ah_bench_C1.err; echo "bench rc=$?"
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 --timeout-method=thread > gpurun_out/r02ah_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02ah_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ah_smoke.log 2>&1; echo "smoke rc=$?"
