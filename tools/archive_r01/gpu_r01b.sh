mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
tail -3 gpurun_out/bench_r01b.err
SEM_AX_KERNEL=simple python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r01b_simple.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ax_tma_kernel -s 10 -c 1 -o gpurun_out/prof_k1_r01b python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_full_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gs_kernel|rr_kernel" -s 20 -c 2 -o gpurun_out/prof_gsrr_r01b python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ax-reps 5 > gpurun_out/ncu_full_c.log 2>&1
tail -3 gpurun_out/ncu_full_b.log
