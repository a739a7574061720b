set -x
for lu in 0 4 8; do
MANDEL_DEV_LAZY_LU=$lu timeout 600 python tools/small_view.py --kernels lazy1,lazy2 --lanes 0,24,32 > gpurun_out/r02ae_small_view_lu$lu.jsonl 2>&1; echo "rc=$?"
done
MANDEL_DEV_LAZY_LU=4 timeout 600 python tools/sweep.py --configs C1 --kernels lazy1,lazy2 --schemes block --steps 10 > gpurun_out/r02ae_check.jsonl 2>&1
