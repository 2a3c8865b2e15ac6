# round 1 (k): FD symmetric kernel parity + sweep; CG bench after the prologue change
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01k.log 2>&1; tail -1 gpurun_out/smoke_r01k.log
timeout 900 python -m pytest tests/test_gpu_fd.py -x -q > gpurun_out/pytest_fd_r01k.log 2>&1; tail -3 gpurun_out/pytest_fd_r01k.log
timeout 600 python bench.py --workload fd --steps 20 > gpurun_out/bench_fd_r01k.json 2> gpurun_out/bench_fd_r01k.err; tail -2 gpurun_out/bench_fd_r01k.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_fd_r01k.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], {k:(round(v['mnodes_s']),round(v['achieved_gbs'])) for k,v in d['sweep'].items()})"
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01k.json 2> gpurun_out/bench_r01k.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r01k.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], r['avg_launch_us'], r['iteration']['us'], r['step_share'])"
ncu --set full --clock-control none --import-source on -k regex:fd2d_kernel -s 3 -c 1 -o gpurun_out/prof_fd_r01k python bench.py --workload fd --steps 3 --warmup 3 --fd-radii 7 --no-cpu-baseline > gpurun_out/ncu_fd.log 2>&1
ls gpurun_out/prof_fd_r01k.ncu-rep
