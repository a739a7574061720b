set -x
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_abi.py tests/test_multiproc_gpu.py -x -q -m gpu -p no:cacheprovider \
  -k "host_handoff or c1_all_schemes or multiproc or rank or abi or async or band or full_size_whole_map" > gpurun_out/r02ao_pytest.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r02ao_pytest.log
# randomised parity campaign on the round-2 kernels (fused y, copy backup)
timeout 1000 python tools/fuzz.py --seconds 900 --seed 61 > gpurun_out/r02ao_fuzz.jsonl 2> gpurun_out/r02ao_fuzz.err
echo "fuzz rc=$?"; tail -1 gpurun_out/r02ao_fuzz.jsonl
