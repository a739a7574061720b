set -x
# current-state benches of all five configs, the default line, the reference arm
timeout 600 python bench.py > gpurun_out/r02q_bench_default.json 2> gpurun_out/r02q_bench_default.err; echo "bench default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02q_bench_reference.json 2> gpurun_out/r02q_bench_reference.err; echo "bench ref rc=$?"
for c in C1 C2 C3 C4 C5; do
  st=20; [ $c = C1 ] && st=100
  timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline > gpurun_out/r02q_bench_$c.json 2> gpurun_out/r02q_bench_$c.err; echo "bench $c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/r02q_bench_$c.json'))
print('$c', d['value'], d['roofline']['frac'], d['roofline']['frac_unit_count'], d['config']['kernel_variant'], d['e2e']['value'], d['e2e']['latency_ms'], {k: v['value'] for k, v in d['per_scheme'].items()})"
done
# launch list + full capture + instruction mix of the bench kernel (C2)
bash tools/profile_bench.sh r02q_c2
# store sectors per request: staged vs direct stores, C2 kernel
for s in 1 -1; do
  ncu --clock-control none -k regex:escape_ -s 2 -c 1 --csv --log-file gpurun_out/r02q_c2_store_sectors_stage$s.csv \
    --metrics l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,smsp__sass_inst_executed_op_global_st.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    python tools/sweep.py --configs C2 --kernels refill --schemes block --stage $s --steps 1 --warmup 2 > gpurun_out/r02q_ncu_stage$s.log 2>&1; echo "ncu stage $s rc=$?"
done
