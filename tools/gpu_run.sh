mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_k1ax.py tests/test_gpu_parity.py tests/test_gpu_c4_fullsize.py -x -q -p no:cacheprovider > gpurun_out/k1dot9_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/k1dot9_tests.log
timeout 900 python tools/order_sweep.py --orders 9 --out gpurun_out/order_sweep_k1dot9.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/order_sweep_k1dot9.json'))
print([(r['N'], r['kernel'], round(r['ax_frac'],3), round(r.get('cg_gdof_s',0),2)) for r in d['rows']])"
