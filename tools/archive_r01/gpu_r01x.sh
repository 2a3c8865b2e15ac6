# round 1 (x): high-order kernel with a register floor (fewer groups, no spills): c4 N=10..15
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/order_sweep.py --orders 8 9 10 11 12 13 14 15 --out gpurun_out/order_sweep_r01x.json > gpurun_out/order_sweep_r01x.log 2>&1; cut -c1-150 gpurun_out/order_sweep_r01x.log
SEM_AX_KERNEL=hi timeout 900 python tools/order_sweep.py --orders 8 9 10 --out gpurun_out/order_sweep_r01x_hi.json > gpurun_out/order_sweep_r01x_hi.log 2>&1; cut -c1-150 gpurun_out/order_sweep_r01x_hi.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hi" > gpurun_out/pytest_hi_r01x.log 2>&1; tail -2 gpurun_out/pytest_hi_r01x.log
