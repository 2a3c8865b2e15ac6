# round 1 (az): N=7 DMMA kernel with the f_r slice stored column-swizzled (conflict-free phase-B fragment loads; Poisson variants only)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x -k "dmma or 7-" > gpurun_out/pytest_gpu_r01az.log 2>&1; tail -1 gpurun_out/pytest_gpu_r01az.log
for i in 1 2 3; do
for opt in "" "--operator screened"; do
  timeout 300 python bench.py --steps 10 --no-cpu-baseline $opt > gpurun_out/bench_r01az_x.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01az_x.json').read().strip().splitlines()[-1]); r=d['roofline']
print('[$opt]', round(d['value'],2), d['config']['cg_iters'], round(r['iteration']['us'],2), round(r['frac'],3), round(r['kernels_replayed']['ax']['avg_launch_us'],2))"
done; done
