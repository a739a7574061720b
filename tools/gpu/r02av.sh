set -x
# NOTE: libmandel_vA_B.so = A/B builds of a first block with early-exit votes after updates A and B (not adopted,
# DESIGN.md "Tried: early-exit votes inside the first block"); the code is not in the tree
# first block with early-exit votes (all of the warp's pixels escaped) after updates A and B: A/B builds
S=gpurun_out/r02av_sweep_first_block_vote.jsonl; : > $S
run() { # lib configs
  echo "{\"lib\": \"$1\"}" >> $S
  MANDEL_LIB=$PWD/paper_2007_00745_b200/$1 timeout 600 python tools/sweep.py --configs $2 --kernels refill --schemes block --steps 6 --warmup 2 >> $S 2>> gpurun_out/r02av.err
}
for rep in 1 2 3; do
  for v in libmandel.so libmandel_v2_4.so libmandel_v1_3.so libmandel_v2_99.so; do run $v C2,C3,C5; done
done
MANDEL_LIB=$PWD/paper_2007_00745_b200/libmandel_v2_4.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "first_block or full_size_whole_map or random_small or edge_cases" -p no:cacheprovider > gpurun_out/r02av_pytest_v2_4.log 2>&1; echo "rc=$?"
tail -2 gpurun_out/r02av_pytest_v2_4.log
MANDEL_LIB=$PWD/paper_2007_00745_b200/libmandel_v1_3.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "first_block or full_size_whole_map or random_small or edge_cases" -p no:cacheprovider > gpurun_out/r02av_pytest_v1_3.log 2>&1; echo "rc=$?"
tail -2 gpurun_out/r02av_pytest_v1_3.log
