set -x
for c in C1 C2 C3 C4 C5; do
  st=20; [ $c = C1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline > gpurun_out/r02ak_bench_$c.json 2> gpurun_out/r02ak_bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py > gpurun_out/r02ak_bench_default.json 2> gpurun_out/r02ak_bench_default.err; echo "bench default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02ak_bench_reference.json 2>&1; echo "ref rc=$?"
for c in c2 c3 c4; do
  C=$(echo $c | tr a-z A-Z)
  bash tools/profile_bench.sh r02ak_$c --config $C
  python tools/ncu_summary.py --traffic gpurun_out/r02ak_${c}_full.ncu-rep $C 1 gpurun_out/r02ak_${c}_traffic.json gpurun_out/r02ak_${c}_ncu_summary.json > gpurun_out/r02ak_${c}_summary.log 2>&1; echo "summary $c rc=$?"
  python tools/ncu_regions.py gpurun_out/r02ak_${c}_full.ncu-rep > gpurun_out/r02ak_${c}_regions.json 2> gpurun_out/r02ak_${c}_regions.err; echo "regions $c rc=$?"
  rm -f gpurun_out/r02ak_${c}_full.ncu-rep
done
ls -la gpurun_out | head -50
