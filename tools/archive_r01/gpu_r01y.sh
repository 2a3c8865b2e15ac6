# round 1 (y): K2 interior nodes per thread per chunk U = 4 / 5 / 6 (prebuilt libraries)
mkdir -p gpurun_out
for U in 4 5 6; do
  cp k2libs/libsem_u$U.so paper_1403_0968_b200/libsem.so
  timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01y_u$U.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_r01y_u$U.json').read().strip().splitlines()[-1]); r=d['roofline']
print('U=$U', d['value'], d['config']['cg_iters'], r['avg_launch_us'], r['iteration']['us'], {k:round(v['avg_launch_us'],1) for k,v in r['kernels_in_solve'].items()})"
done
