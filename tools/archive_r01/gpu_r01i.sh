# round 1 (i): FD stencil (NEXT-4) parity + bench sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fd.py -x -q > gpurun_out/pytest_fd_r01i.log 2>&1; tail -3 gpurun_out/pytest_fd_r01i.log
timeout 600 python bench.py --workload fd --steps 20 > gpurun_out/bench_fd_r01i.json 2> gpurun_out/bench_fd_r01i.err; tail -2 gpurun_out/bench_fd_r01i.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_fd_r01i.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], {k:(round(v['mnodes_s']),round(v['achieved_gbs'])) for k,v in d['sweep'].items()}, d['cpu_baseline'])"
ncu --set full --clock-control none --import-source on -k regex:fd2d_kernel -s 3 -c 1 -o gpurun_out/prof_fd_r01i python bench.py --workload fd --steps 3 --warmup 3 --fd-radii 7 --no-cpu-baseline > gpurun_out/ncu_fd.log 2>&1
ls -la gpurun_out/prof_fd_r01i.ncu-rep
