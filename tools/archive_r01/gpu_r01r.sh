# round 1 (r): relabelled-mesh parity, full GPU suite, FD bench with R-dependent strips
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01r.log 2>&1; tail -1 gpurun_out/smoke_r01r.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01r.log 2>&1; tail -3 gpurun_out/pytest_gpu_r01r.log
timeout 600 python bench.py --workload fd --steps 20 > gpurun_out/bench_fd_r01r.json 2> gpurun_out/bench_fd_r01r.err; tail -1 gpurun_out/bench_fd_r01r.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_fd_r01r.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], {k:round(v['mnodes_s']/1e3) for k,v in d['sweep'].items()}, d['cpu_baseline']['value'])"
