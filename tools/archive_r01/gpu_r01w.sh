# round 1 (w): FD two rows per barrier; smoke with the N=7 tensor-core check
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01w.log 2>&1; tail -1 gpurun_out/smoke_r01w.log
timeout 900 python -m pytest tests/test_gpu_fd.py -q -x > gpurun_out/pytest_fd_r01w.log 2>&1; tail -2 gpurun_out/pytest_fd_r01w.log
timeout 600 python bench.py --workload fd --steps 20 > gpurun_out/bench_fd_r01w.json 2> gpurun_out/bench_fd_r01w.err; tail -1 gpurun_out/bench_fd_r01w.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_fd_r01w.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], {k:round(v['mnodes_s']/1e3) for k,v in d['sweep'].items()})"
