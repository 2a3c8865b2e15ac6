# round 1 (ag): final validation after the N=15 default
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01ag.log 2>&1; tail -1 gpurun_out/smoke_r01ag.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01ag.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01ag.log
timeout 900 python tools/order_sweep.py --out gpurun_out/order_sweep_r01ag.json > gpurun_out/order_sweep_r01ag.log 2>&1; cut -c1-100 gpurun_out/order_sweep_r01ag.log | tail -6
timeout 600 python bench.py > gpurun_out/bench_r01ag.json 2> gpurun_out/bench_r01ag.err; tail -1 gpurun_out/bench_r01ag.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r01ag.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['cg_iters_per_s'], r['iteration']['us'], r['frac'], d['e2e']['value'])"
