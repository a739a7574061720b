# round 2d: parity suite with store staging (two-rank bench tests deselected), repro of the
# two-rank share-device bench hang with stack dumps, clean stage A/B sweep
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not two_ranks_shared_device" > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02d_pytest_gpu.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 2 --config C1 --steps 4 --warmup 3 --e2e-steps 2 --share-device --gather fused --scheme fcfs --no-schemes > gpurun_out/r02d_twor.out 2> gpurun_out/r02d_twor.err &
TR=$!
for t in 1 2 3 4 5 6 7 8 9 10 11 12; do sleep 10; if ! kill -0 $TR 2>/dev/null; then break; fi; done
if kill -0 $TR 2>/dev/null; then
  echo "STILL RUNNING after 120 s"; nvidia-smi >> gpurun_out/r02d_twor.err 2>&1
  for c in $(pgrep -P $TR); do echo "child $c"; kill -USR1 $c; done
  sleep 5
  for c in $(pgrep -P $TR); do kill -9 $c; done; kill -9 $TR
fi
wait $TR; echo "twor rc=$?"
tail -50 gpurun_out/r02d_twor.err
for rep in 1 2; do
timeout 900 python tools/sweep.py --configs C2,C5,C3,C4 --kernels refill --schemes block --stage 1,0 --steps 10 >> gpurun_out/r02d_sweep_stage.jsonl 2>> gpurun_out/r02d_sweep.err
done
