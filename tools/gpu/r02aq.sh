set -x
# randomised parity campaign on the final round-2 library, incl. the per-device host hand-off
timeout 1700 python tools/fuzz.py --seconds 1500 --seed 71 > gpurun_out/r02aq_fuzz.jsonl 2> gpurun_out/r02aq_fuzz.err
echo "fuzz rc=$?"; tail -1 gpurun_out/r02aq_fuzz.jsonl; grep -c '"bad"' gpurun_out/r02aq_fuzz.jsonl
