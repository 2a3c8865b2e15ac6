python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"gs_kernel|rr_kernel" -s 40 -c 2 -o gpurun_out/prof_gsrr_warm python tools/cg_variants.py > gpurun_out/ncu_gsrr.log 2>&1
tail -2 gpurun_out/ncu_gsrr.log
