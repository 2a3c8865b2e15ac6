mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
SEM_K1_SPLIT=0.3 timeout 300 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-400
timeout 300 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-400
