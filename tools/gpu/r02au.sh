set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
T=r02au
M=gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__thread_inst_executed_pred_on_per_inst_executed.ratio,smsp__sass_average_branch_targets_threads_uniform.pct,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
python __graft_entry__.py smoke > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
for c in C1 C2 C3 C4 C5; do
  st=20; [ $c = C1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "bench default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_reference.json 2>&1; echo "ref rc=$?"
for c in C1 C2 C3 C4 C5; do
  for k in static refill; do
    timeout 900 ncu --metrics $M --clock-control none -k regex:escape_ -s 5 -c 1 --csv \
      --log-file gpurun_out/${T}_weff_${c}_${k}.csv python tools/warp_eff.py --config $c --kernel $k --renders 6 \
      > gpurun_out/${T}_weff_${c}_${k}.json 2> gpurun_out/${T}_weff_${c}_${k}.err; echo "weff $c $k rc=$?"
  done
done
for c in c2 c3 c5; do
  C=$(echo $c | tr a-z A-Z)
  timeout 1200 bash tools/profile_bench.sh ${T}_$c --config $C
  python tools/ncu_summary.py --traffic gpurun_out/${T}_${c}_full.ncu-rep $C 1 gpurun_out/${T}_${c}_traffic.json gpurun_out/${T}_${c}_ncu_summary.json > gpurun_out/${T}_${c}_summary.log 2>&1; echo "summary $c rc=$?"
  python tools/ncu_regions.py gpurun_out/${T}_${c}_full.ncu-rep > gpurun_out/${T}_${c}_regions.json 2> gpurun_out/${T}_${c}_regions.err; echo "regions $c rc=$?"
  rm -f gpurun_out/${T}_${c}_full.ncu-rep
done
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider --durations=5 > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 700 python tools/fuzz.py --seconds 600 --seed 71 > gpurun_out/${T}_fuzz.jsonl 2> gpurun_out/${T}_fuzz.err
echo "fuzz rc=$?"; tail -1 gpurun_out/${T}_fuzz.jsonl
