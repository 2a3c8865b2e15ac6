mkdir -p gpurun_out
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err
tail -3 gpurun_out/bench_r01a.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01a.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ax_kernel -s 6 -c 2 -o gpurun_out/prof_k1_r01a python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
