# round 1 (ba): final full GPU suite + smoke + default bench (all keys) + ncu K1 on the final code
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01ba.log 2>&1; tail -1 gpurun_out/smoke_r01ba.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01ba.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01ba.log
timeout 600 python bench.py > gpurun_out/bench_r01ba.json 2> gpurun_out/bench_r01ba.err; tail -1 gpurun_out/bench_r01ba.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r01ba.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['value'],2), d['config']['cg_iters'], round(r['iteration']['us'],2), round(r['frac'],3), round(d['e2e']['value'],2), d['clocks'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01ba.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ax_dmma_kernel -s 10 -c 1 -o gpurun_out/prof_k1_r01ba python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ls gpurun_out/prof_k1_r01ba.ncu-rep
