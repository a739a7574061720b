#!/bin/bash
# Round profiling of the bench command on one B200: launch list + one full capture of
# the escape kernel (run from the repo root under gpurun).  usage: profile_bench.sh TAG [bench args]
# Back in the container:  python tools/ncu_summary.py --traffic gpurun_out/TAG_full.ncu-rep \
#     CONFIG 1 profiles/TAG_traffic.json profiles/TAG_ncu_summary.json
set -u
mkdir -p gpurun_out
tag=$1; shift
CMD="python bench.py --profile --steps 3 --warmup 3 --no-cpu-baseline $*"
$CMD > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv $CMD > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/${tag}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape_ -s 3 -c 1 \
    -o gpurun_out/${tag}_full $CMD > gpurun_out/${tag}_ncu_full.log 2>&1
echo "full rc=$?"
