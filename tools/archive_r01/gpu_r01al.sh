# round 1 (al): single-stage + split copies with 2 groups at N=10, 11 (element-major and slice-major G^)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_c4_fullsize.py tests/test_gpu_parity.py -q -k "fullsize or ax_parity or relabel" > gpurun_out/pytest_r01al.log 2>&1; tail -2 gpurun_out/pytest_r01al.log
timeout 600 python tools/order_sweep.py --orders 10 11 12 13 14 15 --out gpurun_out/order_sweep_r01al.json > gpurun_out/order_sweep_r01al.log 2>&1; cut -c1-140 gpurun_out/order_sweep_r01al.log
