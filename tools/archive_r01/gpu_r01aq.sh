# round 1 (aq): full GPU suite after the K2<PC> / KB register changes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01aq.log 2>&1; tail -1 gpurun_out/smoke_r01aq.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01aq.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01aq.log
for opt in "" "--precond jacobi" "--cg-variant single_reduction" "--operator screened"; do
  timeout 300 python bench.py --steps 10 --no-cpu-baseline $opt > gpurun_out/bench_r01aq_x.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01aq_x.json').read().strip().splitlines()[-1]); r=d['roofline']
print('[$opt]', round(d['value'],2), d['config']['cg_iters'], round(r['iteration']['us'],2))"
done
