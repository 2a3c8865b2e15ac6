# round 1 (g): K2 experiments (4 blocks/SM) + ncu launch list and full captures (K1, K2 with source)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for bps in 3 4; do
  SEM_K2_BPS=$bps timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_r01g_bps$bps.json 2> gpurun_out/bench_r01g_bps$bps.err
done
python - <<'PY'
import json
for b in (3, 4):
    f = f"gpurun_out/bench_r01g_bps{b}.json"
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(b, d["value"], r["iteration"]["us"], r["step_share"], {k: (v["avg_launch_us"], v["frac"]) for k, v in r["kernels_replayed"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01g.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ax_tma_kernel -s 10 -c 1 -o gpurun_out/prof_k1_r01g python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_k1g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_kernel -s 10 -c 1 -o gpurun_out/prof_k2_r01g python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_k2g.log 2>&1
tail -1 gpurun_out/ncu_k1g.log gpurun_out/ncu_k2g.log; ls -la gpurun_out/*.ncu-rep
