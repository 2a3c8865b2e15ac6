# round 1 (n): SR tests again; FD rotating register queue; full GPU suite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01n.log 2>&1; tail -1 gpurun_out/smoke_r01n.log
timeout 900 python -m pytest tests/test_gpu_cg_sr.py tests/test_gpu_fd.py -q > gpurun_out/pytest_srfd_r01n.log 2>&1; tail -3 gpurun_out/pytest_srfd_r01n.log
timeout 600 python bench.py --workload fd --steps 20 > gpurun_out/bench_fd_r01n.json 2> gpurun_out/bench_fd_r01n.err; tail -2 gpurun_out/bench_fd_r01n.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_fd_r01n.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], {k:(round(v['mnodes_s']),round(v['achieved_gbs'])) for k,v in d['sweep'].items()})"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01n.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01n.log
