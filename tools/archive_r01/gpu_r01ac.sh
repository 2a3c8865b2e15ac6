# round 1 (ac): dmmag default for N = 10, 11 -- full GPU suite + c4 sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01ac.log 2>&1; tail -1 gpurun_out/smoke_r01ac.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01ac.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01ac.log
timeout 900 python tools/order_sweep.py --out gpurun_out/order_sweep_r01ac.json > gpurun_out/order_sweep_r01ac.log 2>&1; cut -c1-120 gpurun_out/order_sweep_r01ac.log
