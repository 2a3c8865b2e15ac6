mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err
tail -2 gpurun_out/bench_r01c.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ax_tma_kernel -s 10 -c 1 -o gpurun_out/prof_k1_r01c python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_k1c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_kernel -s 10 -c 1 -o gpurun_out/prof_k2_r01c python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_k2c.log 2>&1
tail -1 gpurun_out/ncu_k1c.log gpurun_out/ncu_k2c.log
