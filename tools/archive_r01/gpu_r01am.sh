# round 1 (am): full GPU suite + final c4 sweep after the split-copy groups
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01am.log 2>&1; tail -1 gpurun_out/smoke_r01am.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01am.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01am.log
timeout 900 python tools/order_sweep.py --out gpurun_out/order_sweep_r01am.json > gpurun_out/order_sweep_r01am.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/order_sweep_r01am.json')); print([(r['N'], round(r['ax_frac'],3)) for r in d['rows']])"
