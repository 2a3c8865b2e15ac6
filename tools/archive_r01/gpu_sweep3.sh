mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SEM_AX_KERNEL=hi timeout 300 compute-sanitizer --tool memcheck python tools/dbg_n4.py 11 4 3 3 2>&1 | tail -2
SEM_AX_KERNEL=hi timeout 300 compute-sanitizer --tool racecheck python tools/dbg_n4.py 8 3 3 2 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q -k "ax_parity or cg_iteration" 2>&1 | tail -3
SEM_AX_KERNEL=hi timeout 1200 python tools/order_sweep.py --orders 6 7 8 9 10 11 12 13 14 15 --out gpurun_out/order_sweep_hi.json 2>&1 | tail -12
