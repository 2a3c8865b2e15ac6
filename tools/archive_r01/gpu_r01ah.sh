# round 1 (ah): K1 element assignment group-major (tail spread over SMs) A/B vs r01ag
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01ah_$i.json 2> /dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_r01ah_$i.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], r['avg_launch_us'], r['iteration']['us'], d['ax']['kernel_ms'])"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cg" > gpurun_out/pytest_r01ah.log 2>&1; tail -2 gpurun_out/pytest_r01ah.log
