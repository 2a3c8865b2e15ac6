mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -2 gpurun_out/bench_quick.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_quick.json'))
r=d['roofline']
print('value', round(d['value'],3), 'it/s', round(d['cg_iters_per_s']), 'ms/step', round(d['ms_per_step'],2), 'its', d['config']['cg_iters'])
print('K1 GB/s', round(r['achieved']), 'frac', round(r['frac'],3), 'avg us', round(r['avg_launch_us'],2), 'shares', {k: round(v,3) for k,v in r['step_share'].items()})
print('ax', {k: (round(v,3) if isinstance(v,float) else v) for k,v in d['ax'].items()})
print('e2e', d['e2e'], 'clocks', d['clocks'])
PY
