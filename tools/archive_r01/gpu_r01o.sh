# round 1 (o): FD launch bounds (no spills), SR alternate test, c4 order sweep (current kernels), bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_cg_sr.py tests/test_gpu_fd.py -q > gpurun_out/pytest_srfd_r01o.log 2>&1; tail -2 gpurun_out/pytest_srfd_r01o.log
timeout 600 python bench.py --workload fd --steps 20 > gpurun_out/bench_fd_r01o.json 2> gpurun_out/bench_fd_r01o.err; tail -2 gpurun_out/bench_fd_r01o.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_fd_r01o.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], {k:(round(v['mnodes_s']),round(v['achieved_gbs'])) for k,v in d['sweep'].items()})"
timeout 900 python tools/order_sweep.py --out gpurun_out/order_sweep_r01o.json > gpurun_out/order_sweep_r01o.log 2>&1; tail -3 gpurun_out/order_sweep_r01o.log
timeout 600 python bench.py > gpurun_out/bench_r01o.json 2> gpurun_out/bench_r01o.err; tail -1 gpurun_out/bench_r01o.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r01o.json').read().strip().splitlines()[-1]); r=d['roofline']
print('cg', d['value'], d['config']['cg_iters'], r['avg_launch_us'], r['iteration']['us'], r['kernels_in_solve'])"
