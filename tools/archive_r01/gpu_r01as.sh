# round 1 (as): Ax on the tensor cores at N = 12..15 with 16 warps per element (one group per SM)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ax_parity or annihilates" > gpurun_out/pytest_gpu_r01as.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01as.log
timeout 900 python tools/order_sweep.py --orders 10 11 12 13 14 15 --out gpurun_out/order_sweep_r01as.json > gpurun_out/order_sweep_r01as.log 2>&1; cut -c1-160 gpurun_out/order_sweep_r01as.log
