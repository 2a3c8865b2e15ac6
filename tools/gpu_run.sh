mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg.py tests/test_gpu_screened.py tests/test_gpu_multirank.py -x -q -p no:cacheprovider -k "dmma or 7 or pcg or screened or multirank" > gpurun_out/xd_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/xd_tests.log
b() { timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline $2 > gpurun_out/xd.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/xd.json').read().strip().splitlines()[-1])
print('$1 $2', 'value %.2f'%d['value'], 'ms %.3f'%d['ms_per_step'], {k:round(x['avg_launch_us'],2) for k,x in d['roofline']['kernels_in_solve'].items()})"; }
b xdirect ""; b xdirect "--precond jacobi"; b xdirect "--operator screened"
SEM_NVCC_EXTRA="-DSEM_K1_XDIRECT=0" python -c "from paper_1403_0968_b200 import _build; _build.build(force=True, verbose=False)" > /dev/null 2>&1
b staged ""; b staged "--precond jacobi"; b staged "--operator screened"
b staged ""
SEM_NVCC_EXTRA="" python -c "from paper_1403_0968_b200 import _build; _build.build(force=True, verbose=False)" > /dev/null 2>&1
b xdirect ""
