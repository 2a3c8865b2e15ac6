# round 1 (av): final state of the session -- smoke, full GPU suite, default bench (all keys), variants, FD, ncu K1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01av.log 2>&1; tail -1 gpurun_out/smoke_r01av.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01av.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01av.log
timeout 600 python bench.py > gpurun_out/bench_r01av.json 2> gpurun_out/bench_r01av.err; tail -1 gpurun_out/bench_r01av.err
for opt in "--operator screened" "--precond jacobi" "--cg-variant single_reduction"; do
  tag=$(echo $opt | tr -d ' -' | cut -c1-14)
  timeout 300 python bench.py --steps 10 --no-cpu-baseline $opt > gpurun_out/bench_r01av_$tag.json 2> /dev/null
done
timeout 600 python bench.py --workload fd --steps 20 > gpurun_out/bench_fd_r01av.json 2> /dev/null
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench*r01av*.json")):
    d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f, round(d["value"], 2), d["config"].get("cg_iters"), round(d.get("cg_iters_per_s") or 0), round((r.get("iteration") or {}).get("us", 0), 2), round(r["frac"] or 0, 3), (d.get("e2e") or {}).get("value"))
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01av.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ax_dmma_kernel -s 10 -c 1 -o gpurun_out/prof_k1_r01av python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ls gpurun_out/prof_k1_r01av.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:k2_kernel -s 10 -c 1 -o gpurun_out/prof_k2_r01av python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01av.json 2> gpurun_out/bench_ref_r01av.err
timeout 900 python tools/order_sweep.py --out gpurun_out/order_sweep_r01av.json > gpurun_out/order_sweep_r01av.log 2>&1; cut -c1-120 gpurun_out/order_sweep_r01av.log
timeout 120 python tools/c2_bench.py > gpurun_out/c2_r01av.json 2> /dev/null; cat gpurun_out/c2_r01av.json
