# round 1 (s): DMMA K1/Ax (N=7) parity + A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dmma" > gpurun_out/pytest_dmma_r01s.log 2>&1; tail -3 gpurun_out/pytest_dmma_r01s.log
for v in dmma default; do
  if [ $v = dmma ]; then export SEM_AX_KERNEL=dmma; else unset SEM_AX_KERNEL; fi
  timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01s_$v.json 2> gpurun_out/bench_r01s_$v.err; tail -1 gpurun_out/bench_r01s_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01s_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v', d['value'], d['config']['cg_iters'], r['avg_launch_us'], r['iteration']['us'], d['ax']['kernel_ms'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in r['kernels_replayed'].items()})"
done
unset SEM_AX_KERNEL
SEM_AX_KERNEL=dmma timeout 300 python tools/order_sweep.py --orders 7 --out gpurun_out/order_sweep_dmma.json > gpurun_out/order_sweep_dmma.log 2>&1; cut -c1-220 gpurun_out/order_sweep_dmma.log
SEM_AX_KERNEL=dmma ncu --set full --clock-control none --import-source on -k regex:ax_dmma_kernel -s 10 -c 1 -o gpurun_out/prof_dmma_r01s python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_dmma.log 2>&1
ls gpurun_out/prof_dmma_r01s.ncu-rep
