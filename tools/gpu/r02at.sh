set -x
# NOTE: libmandel_fbP.so = -DMANDEL_FIRST_BLOCK=P -DMANDEL_FB_ENV=1 A/B builds; MANDEL_FB_ENV (threshold in slots from the
# MANDEL_FB_SLOTS environment variable) existed only for this sweep and is not in the library
# first block: block length (4..16, -DMANDEL_FIRST_BLOCK) x threshold in slots (MANDEL_FB_SLOTS; A/B builds only)
S=gpurun_out/r02at_sweep_first_block_len.jsonl; : > $S
run() { # lib slots configs
  echo "{\"lib\": \"$1\", \"slots\": $2}" >> $S
  MANDEL_FB_SLOTS=$2 MANDEL_LIB=$PWD/paper_2007_00745_b200/$1 timeout 600 python tools/sweep.py --configs $3 --kernels refill --schemes block --steps 6 --warmup 2 >> $S 2>> gpurun_out/r02at.err
}
for rep in 1 2; do
  echo "{\"lib\": \"off\", \"slots\": 0}" >> $S
  timeout 600 python tools/sweep.py --configs C2,C3,C5 --kernels refill --schemes block --first-block -1 --steps 6 --warmup 2 >> $S 2>> gpurun_out/r02at.err
  for P in 8 4 6 12 16; do for sl in 1 2; do run libmandel_fb$P.so $sl C2,C3,C5; done; done
  run libmandel_fb8.so 4 C2,C3,C5
done
