# round 1 (au): high-order tensor-core Ax, k-slice loops unrolled by 2 (both staging variants)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ax_parity or annihilates" > gpurun_out/pytest_gpu_r01au.log 2>&1; tail -1 gpurun_out/pytest_gpu_r01au.log
SEM_DMMAG_R=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ax_parity_all" > gpurun_out/pytest_gpu_r01au_r.log 2>&1; tail -1 gpurun_out/pytest_gpu_r01au_r.log
timeout 900 python tools/order_sweep.py --orders 10 11 12 13 14 15 --out gpurun_out/order_sweep_r01au_base.json 2>&1 | cut -c1-150
SEM_DMMAG_R=1 timeout 900 python tools/order_sweep.py --orders 10 11 12 13 14 15 --out gpurun_out/order_sweep_r01au_r.json 2>&1 | cut -c1-150
