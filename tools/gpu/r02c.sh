# round 2c: store staging -- parity suite, A/B sweep stage on/off, FCFS delay stress
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02c_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c_pytest_gpu.log
for rep in 1 2; do
timeout 900 python tools/sweep.py --configs C2,C5,C3,C4 --kernels refill --schemes block --stage 1,0 --steps 10 >> gpurun_out/r02c_sweep_stage.jsonl 2>> gpurun_out/r02c_sweep.err
done
timeout 600 python tools/sweep.py --configs C4 --kernels lazy2,batch8x2 --schemes block --stage 1,0 --steps 5 >> gpurun_out/r02c_sweep_stage.jsonl 2>> gpurun_out/r02c_sweep.err
echo sweep done
