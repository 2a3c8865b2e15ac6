python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/cg_variants.py 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_warm.csv -s 3000 -c 300 python tools/cg_variants.py > /dev/null 2>&1
python tools/ncu_summary.py --tag tmpwarm --launches gpurun_out/launches_warm.csv > /dev/null; grep '^| `' profiles/ncu_summary_tmpwarm.md | head -5; rm -f profiles/ncu_summary_tmpwarm.*
