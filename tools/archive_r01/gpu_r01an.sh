# round 1 (an): TMA elements per unit at N=6: 2 (current) vs 4 (prebuilt libraries)
mkdir -p gpurun_out
for E in 2 4; do
  cp k2libs/libsem_e$E.so paper_1403_0968_b200/libsem.so
  timeout 300 python tools/order_sweep.py --orders 6 --out gpurun_out/os_e$E.json > gpurun_out/os_e$E.log 2>&1; echo "EPG=$E"; cut -c1-160 gpurun_out/os_e$E.log
done
