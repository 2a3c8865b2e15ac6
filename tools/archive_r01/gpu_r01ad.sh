# round 1 (ad): dmmag single-stage for N = 12..14 (opt-in SEM_DMMAG=1): parity + c4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SEM_DMMAG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ax_parity" > gpurun_out/pytest_dg_r01ad.log 2>&1; tail -3 gpurun_out/pytest_dg_r01ad.log
SEM_DMMAG=1 timeout 900 python tools/order_sweep.py --orders 8 9 12 13 14 --out gpurun_out/order_sweep_dg2.json > gpurun_out/order_sweep_dg2.log 2>&1; cut -c1-140 gpurun_out/order_sweep_dg2.log
