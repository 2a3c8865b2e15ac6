# round 1 (ab): the plain Ax at N = 8..11 on the tensor cores (opt-in) -- parity + c4 sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dmma and (ax_parity or relabel)" > gpurun_out/pytest_dg_r01ab.log 2>&1; tail -3 gpurun_out/pytest_dg_r01ab.log
SEM_DMMAG=1 timeout 900 python tools/order_sweep.py --orders 8 9 10 11 --out gpurun_out/order_sweep_dg.json > gpurun_out/order_sweep_dg.log 2>&1; cut -c1-140 gpurun_out/order_sweep_dg.log
