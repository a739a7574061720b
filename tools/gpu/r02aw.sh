set -x
T=r02aw
python __graft_entry__.py smoke > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "bench default rc=$?"
timeout 1200 bash tools/profile_bench.sh ${T}_c4 --config C4
python tools/ncu_summary.py --traffic gpurun_out/${T}_c4_full.ncu-rep C4 1 gpurun_out/${T}_c4_traffic.json gpurun_out/${T}_c4_ncu_summary.json > gpurun_out/${T}_c4_summary.log 2>&1; echo "summary c4 rc=$?"
python tools/ncu_regions.py gpurun_out/${T}_c4_full.ncu-rep > gpurun_out/${T}_c4_regions.json 2> gpurun_out/${T}_c4_regions.err; echo "regions c4 rc=$?"
rm -f gpurun_out/${T}_c4_full.ncu-rep
timeout 1000 python tools/fuzz.py --seconds 900 --seed 83 > gpurun_out/${T}_fuzz.jsonl 2> gpurun_out/${T}_fuzz.err
echo "fuzz rc=$?"; tail -1 gpurun_out/${T}_fuzz.jsonl
