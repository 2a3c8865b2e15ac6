mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r02z4_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02z4_tests.log
timeout 300 python tools/rcg_phases.py > gpurun_out/r02z4_phases.json 2>&1; echo "phases rc=$?"
cat gpurun_out/r02z4_phases.json | tr -d '\n '; echo
