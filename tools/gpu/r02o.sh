set -x
timeout 300 python bench.py --config C1 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r02o_bench_c1.json 2> gpurun_out/r02o_bench_c1.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02o_bench_c1.json'))
print(d['value'], d['render_ms'], d['config']['kernel_variant'], d['e2e']['value'], d['e2e']['latency_ms'], d.get('per_scheme'))"
for c in C2 C3 C4 C5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_bench_$c.json 2> gpurun_out/r02o_bench_$c.err; echo "bench $c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/r02o_bench_$c.json'))
print('$c', d['value'], d['roofline']['frac'], d['roofline']['frac_unit_count'], d['config']['kernel_variant'], d['e2e']['value'], d['e2e']['latency_ms'], {k: v['value'] for k, v in d['per_scheme'].items()})"; done
