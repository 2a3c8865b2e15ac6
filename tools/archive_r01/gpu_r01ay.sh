# round 1 (ay): full GPU suite + smoke + default bench on the final code (after the high-order double2 change)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01ay.log 2>&1; tail -1 gpurun_out/smoke_r01ay.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01ay.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01ay.log
timeout 600 python bench.py > gpurun_out/bench_r01ay.json 2> gpurun_out/bench_r01ay.err; tail -1 gpurun_out/bench_r01ay.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r01ay.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['value'],2), d['config']['cg_iters'], round(r['iteration']['us'],2), round(r['frac'],3), round(d['e2e']['value'],2), d['clocks'])"
