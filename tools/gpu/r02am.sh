set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
# occupancy: the fp64 batched loop at 3 vs 4 resident CTAs per SM (64-register budget)
for rep in 1 2; do
  timeout 900 python tools/sweep.py --configs C2,C5 --kernels batch8x2,batch8x1 --minb 3,4 --schemes block \
    --steps 10 --warmup 2 > gpurun_out/r02am_minb_$rep.jsonl 2>&1; echo "minb $rep rc=$?"
done
timeout 600 python tools/sweep.py --configs C3 --kernels refill --schemes block --steps 20 --warmup 3 \
  > gpurun_out/r02am_c3.jsonl 2>&1; echo "c3 rc=$?"
