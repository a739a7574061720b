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
# the instruction mix the roofline argument rests on (SURVEY §8(d) metric list)
$CMD > gpurun_out/${tag}_plain3.log 2>&1 && \
ncu --clock-control none -k regex:escape_ -s 3 -c 1 --csv --log-file gpurun_out/${tag}_mix.csv \
    --metrics sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    $CMD > gpurun_out/${tag}_ncu_mix.log 2>&1
echo "mix rc=$?"
