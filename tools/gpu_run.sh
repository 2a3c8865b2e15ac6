mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02y_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02y_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02y_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02y_gputests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r02y_bench.json').read().strip().splitlines()[-1])
print('value %.2f'%d['value'], 'ms %.3f'%d['ms_per_step'], d['roofline']['frac'], {k:round(x['avg_launch_us'],2) for k,x in d['roofline']['kernels_in_solve'].items()}, d['e2e']['value'], d['gpu_launches'], d['clocks'])"
timeout 600 python bench.py --precond jacobi --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02y_bench_pcg.json 2>/dev/null; echo "pcg rc=$?"
timeout 900 python tools/order_sweep.py --orders 9 --out gpurun_out/order_sweep_r02y_n9.json > /dev/null 2>&1; echo "sweep rc=$?"
