#!/bin/bash
# ncu --set full captures of kernel variants on one config each (1 GPU).
# usage: tools/profile_variants.sh TAG "CONFIG:KERNEL:TILE:LANES" ...
set -u
mkdir -p gpurun_out
tag=$1; shift
for spec in "$@"; do
  IFS=: read cfg kern tile lanes scheme <<< "$spec"
  scheme=${scheme:-block}
  CMD="python tools/sweep.py --configs $cfg --kernels $kern --schemes $scheme --tiles $tile --lanes $lanes --steps 1 --warmup 1"
  out="gpurun_out/${tag}_${cfg}_${kern}_t${tile}_l${lanes}_${scheme}"
  $CMD > ${out}.plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:escape_ -s 1 -c 1 -o $out $CMD > ${out}.ncu.log 2>&1
  echo "$spec rc=$?"
done
