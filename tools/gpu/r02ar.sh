set -x
# final round-2 measurement on the library at HEAD: bench lines of C1-C5, the default line
# with cpu_baseline, the reference arm, and the launch list + ncu --set full capture + FP
# instruction mix of C2-C5 (kernels unchanged since r02an; host code changed in eb76655)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for c in C1 C2 C3 C4 C5; do
  st=20; [ $c = C1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline > gpurun_out/r02ar_bench_$c.json 2> gpurun_out/r02ar_bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py > gpurun_out/r02ar_bench_default.json 2> gpurun_out/r02ar_bench_default.err; echo "bench default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02ar_bench_reference.json 2>&1; echo "ref rc=$?"
for c in c2 c3 c4 c5; do
  C=$(echo $c | tr a-z A-Z)
  timeout 1200 bash tools/profile_bench.sh r02ar_$c --config $C
  python tools/ncu_summary.py --traffic gpurun_out/r02ar_${c}_full.ncu-rep $C 1 gpurun_out/r02ar_${c}_traffic.json gpurun_out/r02ar_${c}_ncu_summary.json > gpurun_out/r02ar_${c}_summary.log 2>&1; echo "summary $c rc=$?"
  python tools/ncu_regions.py gpurun_out/r02ar_${c}_full.ncu-rep > gpurun_out/r02ar_${c}_regions.json 2> gpurun_out/r02ar_${c}_regions.err; echo "regions $c rc=$?"
  rm -f gpurun_out/r02ar_${c}_full.ncu-rep
done
ls -la gpurun_out | head -80
