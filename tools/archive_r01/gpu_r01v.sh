# round 1 (v): K2/KB as one 768-thread block per SM (148 partials instead of 444); + PDL A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01v.log 2>&1; tail -1 gpurun_out/smoke_r01v.log
for v in base pdl; do
  if [ $v = pdl ]; then export SEM_PDL=1; else unset SEM_PDL; fi
  timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01v_$v.json 2> gpurun_out/bench_r01v_$v.err; tail -1 gpurun_out/bench_r01v_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01v_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v', d['value'], d['config']['cg_iters'], r['avg_launch_us'], r['iteration']['us'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in r['kernels_in_solve'].items()})"
done
unset SEM_PDL
for opt in "--precond jacobi" "--cg-variant single_reduction"; do
  timeout 300 python bench.py --steps 10 --no-cpu-baseline $opt > gpurun_out/bench_r01v_x.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01v_x.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$opt', d['value'], d['config']['cg_iters'], r['iteration']['us'])"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg.py tests/test_gpu_cg_sr.py -q -x > gpurun_out/pytest_r01v.log 2>&1; tail -2 gpurun_out/pytest_r01v.log
