# round 1 (at): high-order tensor-core Ax with G^ read into registers (u double-buffered, f in smem)
mkdir -p gpurun_out
SEM_DMMAG_R=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ax_parity or annihilates" > gpurun_out/pytest_gpu_r01at.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01at.log
SEM_DMMAG_R=1 timeout 900 python tools/order_sweep.py --orders 10 11 12 13 14 15 --out gpurun_out/order_sweep_r01at_r.json 2>&1 | cut -c1-150
SEM_DMMAG=1 SEM_DMMAG_R=1 timeout 900 python tools/order_sweep.py --orders 8 9 --out gpurun_out/order_sweep_r01at_r89.json 2>&1 | cut -c1-150
timeout 900 python tools/order_sweep.py --orders 10 11 12 13 14 15 --out gpurun_out/order_sweep_r01at_base.json 2>&1 | cut -c1-150
