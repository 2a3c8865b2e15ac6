# round 1 (ar): DMMA K1 with split per-operand copies (6 groups/SM) vs whole-element copies
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01ar.log 2>&1; tail -1 gpurun_out/smoke_r01ar.log
timeout 900 python -m pytest tests -m gpu -q -k "dmma or 7-" -x > gpurun_out/pytest_gpu_r01ar.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01ar.log
for sp in 1 0 1 0; do
for opt in "" "--precond jacobi" "--operator screened"; do
  SEM_DMMA_SPLIT=$sp timeout 300 python bench.py --steps 10 --no-cpu-baseline $opt > gpurun_out/bench_r01ar_x.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01ar_x.json').read().strip().splitlines()[-1]); r=d['roofline']
print('split=$sp [$opt]', round(d['value'],2), d['config']['cg_iters'], round(r['iteration']['us'],2), r.get('k1_frac', r.get('frac')))"
done; done
