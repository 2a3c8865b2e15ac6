mkdir -p gpurun_out
SEM_PDL=1 timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pdl_tests.log
for i in 1 2; do for v in 0 1; do
SEM_PDL=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pdl_b$v.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/pdl_b$v.json').read().strip().splitlines()[-1])
print('PDL=$v', 'value %.2f'%d['value'], 'ms %.3f'%d['ms_per_step'], {k:round(x['avg_launch_us'],2) for k,x in d['roofline']['kernels_in_solve'].items()})"
done; done
