set -x
V1="-2.5,1.5,-2.0,2.0,800,800,200"
V2="-2.5,1.5,-2.0,2.0,1024,1024,500"
V3="-2.5,1.5,-2.0,2.0,640,480,1000"
V4="-0.743693887,-0.743593887,0.131775904,0.131875904,800,800,2000"
V5="-2.0,0.5,-1.25,1.25,1200,1200,100"
V6="-0.75,-0.74,0.1,0.11,512,512,5000"
for v in $V1 $V2 $V3 $V4 $V5 $V6; do
timeout 300 python tools/small_view.py --view=$v --kernels refill >> gpurun_out/r02ag_small_views.jsonl 2>&1; echo "rc=$?"
done
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_abi.py tests/test_output_stage.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r02ag_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02ag_pytest.log
timeout 300 python bench.py --config C1 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/r02ag_bench_C1.json 2>&1; echo "bench rc=$?"
