# round 1 (z): final state -- smoke, full GPU suite, default bench (cpu baseline), reference arm, c4 sweep, c2, FD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01z.log 2>&1; tail -1 gpurun_out/smoke_r01z.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01z.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01z.log
timeout 600 python bench.py > gpurun_out/bench_r01z.json 2> gpurun_out/bench_r01z.err; tail -1 gpurun_out/bench_r01z.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01z.json 2> gpurun_out/bench_ref_r01z.err
timeout 900 python tools/order_sweep.py --out gpurun_out/order_sweep_r01z.json > gpurun_out/order_sweep_r01z.log 2>&1; cut -c1-120 gpurun_out/order_sweep_r01z.log
timeout 120 python tools/c2_bench.py > gpurun_out/c2_r01z.json 2> /dev/null; cat gpurun_out/c2_r01z.json
timeout 600 python bench.py --workload fd --steps 20 > gpurun_out/bench_fd_r01z.json 2> /dev/null
python - <<'PY'
import json
for f in ["gpurun_out/bench_r01z.json", "gpurun_out/bench_ref_r01z.json", "gpurun_out/bench_fd_r01z.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d.get("unit"), (d.get("roofline") or {}).get("frac"), d.get("e2e", {}).get("value"), (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
