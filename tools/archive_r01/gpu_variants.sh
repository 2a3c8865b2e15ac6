python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
python tools/micro.py 2>&1 | tail -1
python tools/micro.py 7 32 32 32 2>&1 | tail -1
for v in "SEM_PDL=0 SEM_CG_GRAPH=1" "SEM_PDL=1 SEM_CG_GRAPH=1"; do
  env $v python tools/cg_variants.py 2>&1 | tail -1
done
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_warm.csv -s 3000 -c 300 python tools/cg_variants.py > /dev/null 2>&1
python tools/ncu_summary.py --tag tmpwarm --launches gpurun_out/launches_warm.csv > /dev/null; cat profiles/ncu_summary_tmpwarm.md | head -12; rm -f profiles/ncu_summary_tmpwarm.*
