# round 1 (ao): single-stage split-copy CUDA-core Ax at N=8, 9 (3-4 groups per SM)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_c4_fullsize.py tests/test_gpu_parity.py -q -k "fullsize or ax_parity or relabel" > gpurun_out/pytest_r01ao.log 2>&1; tail -2 gpurun_out/pytest_r01ao.log
timeout 600 python tools/order_sweep.py --orders 8 9 --out gpurun_out/os_t1.json > gpurun_out/os_t1.log 2>&1; cut -c1-140 gpurun_out/os_t1.log
SEM_TMA1=0 timeout 600 python tools/order_sweep.py --orders 8 9 --out gpurun_out/os_t0.json > gpurun_out/os_t0.log 2>&1; cut -c1-140 gpurun_out/os_t0.log
