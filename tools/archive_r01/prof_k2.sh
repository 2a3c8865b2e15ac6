python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k2_kernel" -s 20 -c 1 -o gpurun_out/prof_k2 python tools/cg_variants.py > gpurun_out/ncu_k2.log 2>&1
tail -2 gpurun_out/ncu_k2.log
