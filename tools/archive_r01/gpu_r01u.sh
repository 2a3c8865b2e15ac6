# round 1 (u): DMMA for every N=7 variant (screened, Jacobi, single reduction); suite; benches; ncu for profiles
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01u.log 2>&1; tail -1 gpurun_out/smoke_r01u.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01u.log 2>&1; tail -3 gpurun_out/pytest_gpu_r01u.log
timeout 600 python bench.py > gpurun_out/bench_r01u.json 2> gpurun_out/bench_r01u.err; tail -1 gpurun_out/bench_r01u.err
for opt in "--operator screened" "--precond jacobi" "--cg-variant single_reduction"; do
  tag=$(echo $opt | tr -d ' -' | cut -c1-14)
  timeout 300 python bench.py --steps 10 --no-cpu-baseline $opt > gpurun_out/bench_r01u_$tag.json 2> /dev/null
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_r01u*.json")):
    d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f, round(d["value"], 2), d["config"]["cg_iters"], round(d["cg_iters_per_s"]), round(r["iteration"]["us"], 2), round(r["frac"] or 0, 3), d.get("e2e", {}).get("value"), (d.get("cpu_baseline") or {}).get("value"))
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01u.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ax_dmma_kernel -s 10 -c 1 -o gpurun_out/prof_k1_r01u python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_kernel -s 10 -c 1 -o gpurun_out/prof_k2_r01u python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ls gpurun_out/*r01u*.ncu-rep
