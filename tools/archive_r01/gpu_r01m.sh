# round 1 (m): single-reduction CG (NEXT-3) parity + bench; c2 measurement
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01m.log 2>&1; tail -1 gpurun_out/smoke_r01m.log
timeout 900 python -m pytest tests/test_gpu_cg_sr.py -q > gpurun_out/pytest_sr_r01m.log 2>&1; tail -3 gpurun_out/pytest_sr_r01m.log
timeout 300 python bench.py --steps 10 --no-cpu-baseline --cg-variant single_reduction > gpurun_out/bench_r01m_sr.json 2> gpurun_out/bench_r01m_sr.err; tail -1 gpurun_out/bench_r01m_sr.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r01m_sr.json').read().strip().splitlines()[-1]); r=d['roofline']
print('sr', d['value'], d['config']['cg_iters'], r['avg_launch_us'], r['iteration']['us'], r['step_share'])"
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01m.json 2> gpurun_out/bench_r01m.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r01m.json').read().strip().splitlines()[-1]); r=d['roofline']
print('cg', d['value'], d['config']['cg_iters'], r['avg_launch_us'], r['iteration']['us'], r['step_share'])"
timeout 120 python tools/c2_bench.py > gpurun_out/c2_r01m.json 2> gpurun_out/c2_r01m.err; cat gpurun_out/c2_r01m.json; tail -2 gpurun_out/c2_r01m.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01m.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01m.log
