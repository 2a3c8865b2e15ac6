mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_poisson.json 2> gpurun_out/bench_poisson.err
timeout 600 python bench.py --steps 10 --warmup 3 --operator screened > gpurun_out/bench_screened.json 2> gpurun_out/bench_screened.err
tail -c 300 gpurun_out/bench_poisson.err; tail -c 300 gpurun_out/bench_screened.err
python - <<'P'
import json
for f in ("poisson", "screened"):
    d = json.load(open(f"gpurun_out/bench_{f}.json"))
    r = d["roofline"]
    print(f, d["config"]["cg_iters"], round(d["ms_per_step"], 2), "its/s", round(d["cg_iters_per_s"]),
          "K1 frac", round(r["frac"], 3), "iter frac", round(r["iteration"]["frac"], 3),
          "ax frac", round(d["ax"]["frac"], 3), {k: round(v["avg_launch_us"], 1) for k, v in r["kernels_replayed"].items()})
P
