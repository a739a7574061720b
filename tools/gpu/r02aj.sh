set -x
for c in C1 C2 C3 C4 C5; do
  st=20; [ $c = C1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline > gpurun_out/r02aj_bench_$c.json 2> gpurun_out/r02aj_bench_$c.err; echo "bench $c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/r02aj_bench_$c.json'))
print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['frac_of_fma_flop_peak'], d['config']['kernel_variant'], d['e2e']['value'], d['e2e']['latency_ms'], {k: v['value'] for k, v in d['per_scheme'].items()})"
done
timeout 600 python bench.py > gpurun_out/r02aj_bench_default.json 2> gpurun_out/r02aj_bench_default.err; echo "bench default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02aj_bench_reference.json 2>&1; echo "ref rc=$?"
bash tools/profile_bench.sh r02aj_c2
bash tools/profile_bench.sh r02aj_c4 --config C4
bash tools/profile_bench.sh r02aj_c3 --config C3
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 --timeout-method=thread > gpurun_out/r02aj_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02aj_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02aj_smoke.log 2>&1; echo "smoke rc=$?"
