set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
# first block (options.first_block): thresholds against off and against the previous commit's library
S=gpurun_out/r02as_sweep_first_block.jsonl; : > $S
run() { # lib first_block configs
  echo "{\"lib\": \"$1\", \"first_block\": $2}" >> $S
  MANDEL_LIB=$PWD/paper_2007_00745_b200/$1 timeout 600 python tools/sweep.py --configs $3 --kernels refill --schemes block --first-block $2 --steps 6 --warmup 2 >> $S 2>> gpurun_out/r02as.err
}
for rep in 1 2; do
  MANDEL_LIB=$PWD/paper_2007_00745_b200/libmandel_old.so timeout 600 python tools/sweep.py --configs C2,C3,C5 --kernels refill --schemes block --steps 6 --warmup 2 2>> gpurun_out/r02as.err | sed 's/^{/{"lib": "old", /' >> $S
  for fb in -1 1 4 8 12 16; do run libmandel.so $fb C2,C3,C5; done
done
run libmandel.so -1 C1,C4; run libmandel.so 0 C1,C4
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "first_block" -p no:cacheprovider > gpurun_out/r02as_pytest_first_block.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/r02as_pytest_first_block.log
for c in C1 C2 C3 C4 C5; do
  st=20; [ $c = C1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline > gpurun_out/r02as_bench_$c.json 2> gpurun_out/r02as_bench_$c.err; echo "bench $c rc=$?"
done
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider --durations=5 > gpurun_out/r02as_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02as_pytest_gpu.log
