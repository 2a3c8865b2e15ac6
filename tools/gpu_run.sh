mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02f_smi.txt
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02f_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02f_gputests.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/r02f_bench$i.json 2> gpurun_out/r02f_bench$i.err; echo "bench rc=$?"; done
SEM_L2_PERSIST=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_nol2.json 2> gpurun_out/r02f_bench_nol2.err; echo "bench nol2 rc=$?"
for f in gpurun_out/r02f_bench1.json gpurun_out/r02f_bench2.json gpurun_out/r02f_bench_nol2.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('kernels_in_solve',{}).get('k2',{}).get('avg_launch_us'), d['e2e']['value'], d.get('clocks'))"; done
