# round 1 (f): Jacobi PCG (NEXT-2) parity + bench; K1 register change check
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01f.log 2>&1; tail -1 gpurun_out/smoke_r01f.log
timeout 900 python -m pytest tests/test_gpu_pcg.py -x -q > gpurun_out/pytest_pcg_r01f.log 2>&1; tail -3 gpurun_out/pytest_pcg_r01f.log
timeout 600 python bench.py > gpurun_out/bench_r01f.json 2> gpurun_out/bench_r01f.err; tail -2 gpurun_out/bench_r01f.err
timeout 600 python bench.py --precond jacobi > gpurun_out/bench_r01f_jacobi.json 2> gpurun_out/bench_r01f_jacobi.err; tail -2 gpurun_out/bench_r01f_jacobi.err
python - <<'PY'
import json
for f in ["gpurun_out/bench_r01f.json", "gpurun_out/bench_r01f_jacobi.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f, d["value"], d["config"]["cg_iters"], d["cg_iters_per_s"], r["frac"], r["iteration"], {k: (v["avg_launch_us"], v["frac"]) for k, v in r["kernels_replayed"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01f.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01f.log
