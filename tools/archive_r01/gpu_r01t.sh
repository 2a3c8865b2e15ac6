# round 1 (t): DMMA default for N=7 + prologue loads issued before bulk copies (K1, K2); full suite; A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01t.log 2>&1; tail -1 gpurun_out/smoke_r01t.log
for v in default tma; do
  if [ $v = tma ]; then export SEM_AX_KERNEL=tma; else unset SEM_AX_KERNEL; fi
  timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01t_$v.json 2> gpurun_out/bench_r01t_$v.err; tail -1 gpurun_out/bench_r01t_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01t_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v', d['value'], d['config']['cg_iters'], r['avg_launch_us'], r['iteration']['us'], d['ax']['kernel_ms'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in r['kernels_in_solve'].items()})"
done
unset SEM_AX_KERNEL
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01t.log 2>&1; tail -3 gpurun_out/pytest_gpu_r01t.log
