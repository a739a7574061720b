set -x
# NOTE: ran against the first prototype (threshold from the MANDEL_FIRST_BLOCK_MIN environment variable, since replaced by
# options.first_block) and A/B builds libmandel_fb4/fb6.so = -DMANDEL_FIRST_BLOCK=4/6 (build.build_debug)
# first-block A/B: MANDEL_FIRST_BLOCK_MIN (lanes' worth of fresh slots; 0 = off) x block length 8 / 6 / 4
S=gpurun_out/r02ar_sweep_first_block.jsonl; : > $S
run() { # lib fb configs
  echo "{\"lib\": \"$1\", \"first_block_min\": $2}" >> $S
  MANDEL_LIB=$PWD/paper_2007_00745_b200/$1 MANDEL_FIRST_BLOCK_MIN=$2 timeout 600 python tools/sweep.py --configs $3 --kernels refill --schemes block --steps 6 --warmup 2 >> $S 2>> gpurun_out/r02ar.err
}
for rep in 1 2; do
  for fb in 0 16 32 8 24; do run libmandel.so $fb C2,C3,C5; done
  for fb in 16 32; do run libmandel_fb4.so $fb C2,C3,C5; run libmandel_fb6.so $fb C2,C3,C5; done
done
run libmandel.so 0 C1,C4; run libmandel.so 16 C1,C4
# parity with the default threshold
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "full_size_whole_map or random_small or edge_cases or batched_check or fused_y or c1_all_schemes or store_staging" > gpurun_out/r02ar_pytest_subset.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/r02ar_pytest_subset.log
