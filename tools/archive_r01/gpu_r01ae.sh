# round 1 (ae): dmmag default for N = 10..14 -- full GPU suite + c4 sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01ae.log 2>&1; tail -1 gpurun_out/smoke_r01ae.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01ae.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01ae.log
timeout 900 python tools/order_sweep.py --out gpurun_out/order_sweep_r01ae.json > gpurun_out/order_sweep_r01ae.log 2>&1; cut -c1-120 gpurun_out/order_sweep_r01ae.log
