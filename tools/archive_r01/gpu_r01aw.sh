# round 1 (aw): ncu --set full of the high-order tensor-core Ax (N = 13, the weakest c4 order) for round 2
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:ax_dmmag_kernel -s 2 -c 1 -o gpurun_out/prof_dmmag13_r01aw python tools/order_sweep.py --orders 13 --reps 1 --out gpurun_out/os13.json > gpurun_out/ncu_dmmag13_r01aw.log 2>&1
ls -la gpurun_out/prof_dmmag13_r01aw.ncu-rep
