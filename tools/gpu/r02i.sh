# round 2i: C1 small-view latency -- bench line, launch list, full capture of the C1 kernel
set -x
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline --no-schemes > gpurun_out/r02i_bench_c1.json 2> gpurun_out/r02i_bench_c1.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_c1_launches.csv \
  python bench.py --profile --config C1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_c1_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:escape_ -s 5 -c 1 \
  -o gpurun_out/r02i_c1_full python bench.py --profile --config C1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_c1_ncu.log 2>&1; echo "full rc=$?"
