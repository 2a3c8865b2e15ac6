# round 1 (h): one-round-trip CG prologues; bench + GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01h.log 2>&1; tail -1 gpurun_out/smoke_r01h.log
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01h.json 2> gpurun_out/bench_r01h.err; tail -1 gpurun_out/bench_r01h.err
python - <<'PY'
import json
f = "gpurun_out/bench_r01h.json"
d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
print(d["value"], d["config"]["cg_iters"], r["avg_launch_us"], r["iteration"]["us"], r["step_share"], {k: (v["avg_launch_us"], v["frac"]) for k, v in r["kernels_replayed"].items()})
PY
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01h.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01h.log
