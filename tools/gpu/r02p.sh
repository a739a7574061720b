set -x
timeout 300 python bench.py --config C1 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r02p_bench_c1.json 2> gpurun_out/r02p_bench_c1.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02p_bench_c1.json'))
print(d['value'], d['render_ms'], d['config']['kernel_variant'], d['e2e']['value'], d['e2e']['latency_ms'], {k: (v['value'], v['chunks_claimed']) for k, v in d['per_scheme'].items()})"
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 --timeout-method=thread --durations=25 > gpurun_out/r02p_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -32 gpurun_out/r02p_pytest_gpu.log
