# round 1 (af): dmmag at N = 15 (single stage, 229 KB) opt-in: parity + c4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SEM_DMMAG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ax_parity and 15" > gpurun_out/pytest_dg15.log 2>&1; tail -2 gpurun_out/pytest_dg15.log
SEM_DMMAG=1 timeout 600 python tools/order_sweep.py --orders 15 --out gpurun_out/order_sweep_dg15.json > gpurun_out/order_sweep_dg15.log 2>&1; cut -c1-140 gpurun_out/order_sweep_dg15.log
