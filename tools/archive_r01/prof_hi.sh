python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SEM_AX_KERNEL=hi ncu --set full --import-source on --clock-control none -k regex:ax_hi_kernel -c 1 -o gpurun_out/prof_hi11 python tools/dbg_n4.py 11 21 21 21 > gpurun_out/ncu_hi.log 2>&1
tail -2 gpurun_out/ncu_hi.log
