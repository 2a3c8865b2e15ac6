# round 1 (aj): c4 full-size sampled parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_c4_fullsize.py -q > gpurun_out/pytest_c4_r01aj.log 2>&1; tail -3 gpurun_out/pytest_c4_r01aj.log
