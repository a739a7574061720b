set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
# A/B on one box: the fused-y batch start kept as a copy of x (default) vs as x + x
# (libmandel_f64t0.so, MANDEL_F64Y_SAVEX=false); the two libraries alternate
for rep in 1 2; do
  for lib in libmandel libmandel_f64t0; do
    MANDEL_LIB=paper_2007_00745_b200/$lib.so timeout 600 python tools/sweep.py --configs C2,C5 --kernels refill \
      --schemes block --steps 10 --warmup 2 > gpurun_out/r02al_ab_${lib}_$rep.jsonl 2>&1; echo "ab $lib $rep rc=$?"
  done
done
# fp32 (C3): ILP1 with x + x (default) or a copy (libmandel_f32sx.so); ILP2 scalar and packed
for lib in libmandel libmandel_f32sx; do
  MANDEL_LIB=paper_2007_00745_b200/$lib.so timeout 600 python tools/sweep.py --configs C3 --kernels refill,refill2 \
    --pack 1,0 --schemes block --steps 20 --warmup 3 > gpurun_out/r02al_c3_${lib}.jsonl 2>&1; echo "c3 $lib rc=$?"
done
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_abi.py -x -q -m gpu -p no:cacheprovider \
  -k "fused or c1_all or random_small or edge or batched or full_size or small_view" > gpurun_out/r02al_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02al_pytest.log
