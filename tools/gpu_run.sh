mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_topology.py tests/test_gpu_multirank.py tests/test_gpu_c3_parity.py -x -q -p no:cacheprovider > gpurun_out/pcgz_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/pcgz_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precond jacobi > gpurun_out/pcgz_bench.json 2>/dev/null; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/pcgz_bench.json').read().strip().splitlines()[-1])
print('value %.2f'%d['value'], 'ms %.3f'%d['ms_per_step'], d['config']['cg_iters'], {k:round(v['avg_launch_us'],2) for k,v in d['roofline']['kernels_in_solve'].items()})"
