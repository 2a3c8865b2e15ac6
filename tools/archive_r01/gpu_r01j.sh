# round 1 (j): pipelined K2 (cp.async gathers) A/B vs direct, then GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01j.log 2>&1; tail -1 gpurun_out/smoke_r01j.log
for v in pipe direct; do
  SEM_K2=$v timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01j_$v.json 2> gpurun_out/bench_r01j_$v.err; tail -1 gpurun_out/bench_r01j_$v.err
done
python - <<'PY'
import json
for v in ("pipe", "direct"):
    try:
        d = json.loads(open(f"gpurun_out/bench_r01j_{v}.json").read().strip().splitlines()[-1]); r = d["roofline"]
        print(v, d["value"], d["config"]["cg_iters"], r["avg_launch_us"], r["iteration"]["us"], r["step_share"], {k: (v2["avg_launch_us"], v2["frac"]) for k, v2 in r["kernels_replayed"].items()})
    except Exception as e:
        print(v, "ERR", e)
PY
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01j.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01j.log
ncu --set full --clock-control none --import-source on -k regex:k2p_kernel -s 10 -c 1 -o gpurun_out/prof_k2p_r01j python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_k2p.log 2>&1
ls gpurun_out/prof_k2p_r01j.ncu-rep
