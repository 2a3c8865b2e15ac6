# round 1 (ax): high-order tensor-core Ax, 128-bit node-pair shared accesses at even n (bank conflicts, ncu r01aw)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ax_parity or annihilates" > gpurun_out/pytest_gpu_r01ax.log 2>&1; tail -1 gpurun_out/pytest_gpu_r01ax.log
SEM_DMMAG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ax_parity" > gpurun_out/pytest_gpu_r01ax_dg.log 2>&1; tail -1 gpurun_out/pytest_gpu_r01ax_dg.log
timeout 900 python tools/order_sweep.py --orders 10 11 12 13 14 15 --out gpurun_out/order_sweep_r01ax.json 2>&1 | cut -c1-150
SEM_DMMAG=1 timeout 900 python tools/order_sweep.py --orders 8 9 --out gpurun_out/order_sweep_r01ax_89.json 2>&1 | cut -c1-150
ncu --set full --clock-control none --import-source on -k regex:ax_dmmag_kernel -s 2 -c 1 -o gpurun_out/prof_dmmag13_r01ax python tools/order_sweep.py --orders 13 --reps 1 --out gpurun_out/os13.json > /dev/null 2>&1
