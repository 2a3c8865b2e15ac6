# round 1 (p): k-split K1/Ax (two threads per column) A/B + parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in ks default; do
  if [ $v = ks ]; then export SEM_AX_KERNEL=ks; else unset SEM_AX_KERNEL; fi
  timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01p_$v.json 2> gpurun_out/bench_r01p_$v.err; tail -1 gpurun_out/bench_r01p_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01p_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v', d['value'], d['config']['cg_iters'], r['avg_launch_us'], r['iteration']['us'], d['ax']['kernel_ms'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in r['kernels_replayed'].items()})"
done
unset SEM_AX_KERNEL
SEM_AX_KERNEL=ks timeout 600 python tools/order_sweep.py --orders 7 8 9 10 --out gpurun_out/order_sweep_ks.json > gpurun_out/order_sweep_ks.log 2>&1; cat gpurun_out/order_sweep_ks.log | cut -c1-200
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "ks" > gpurun_out/pytest_ks_r01p.log 2>&1; tail -3 gpurun_out/pytest_ks_r01p.log
