#!/bin/bash
# Round-1 profiling on one B200 (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
./tools/fp_peak > gpurun_out/fp_peak.json 2> gpurun_out/fp_peak.err
CMD="python bench.py --profile --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r01_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape_refill -s 3 -c 1 \
    -o gpurun_out/r01_refill_c2 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
CMD2="python bench.py --profile --steps 3 --warmup 3 --no-cpu-baseline --kernel static --scheme block"
$CMD2 > gpurun_out/prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape_static -s 3 -c 1 \
    -o gpurun_out/r01_static_c2 $CMD2 > gpurun_out/ncu_full_static.log 2>&1
echo "static rc=$?"
