# round 1 (ap): K2<PC> and KB without spills -- Jacobi / single-reduction parity + bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_cg_sr.py -q > gpurun_out/pytest_r01ap.log 2>&1; tail -2 gpurun_out/pytest_r01ap.log
for opt in "--precond jacobi" "--cg-variant single_reduction"; do
  timeout 300 python bench.py --steps 10 --no-cpu-baseline $opt > gpurun_out/bench_r01ap_x.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01ap_x.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$opt', d['value'], d['config']['cg_iters'], r['iteration']['us'])"
done
