# round 1 (ak): single-stage tensor-core Ax with split next-element copies (N=13, 15): parity + c4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_c4_fullsize.py tests/test_gpu_parity.py -q -k "fullsize or (ax_parity and (13 or 15))" > gpurun_out/pytest_r01ak.log 2>&1; tail -2 gpurun_out/pytest_r01ak.log
timeout 600 python tools/order_sweep.py --orders 12 13 14 15 --out gpurun_out/order_sweep_r01ak.json > gpurun_out/order_sweep_r01ak.log 2>&1; cut -c1-140 gpurun_out/order_sweep_r01ak.log
