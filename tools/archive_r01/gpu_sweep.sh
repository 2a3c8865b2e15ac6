mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 120 compute-sanitizer --tool memcheck python tools/dbg_n4.py 4 21 21 21 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python tools/order_sweep.py 2>&1 | tail -15
