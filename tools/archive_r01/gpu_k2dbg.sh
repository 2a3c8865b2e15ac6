python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for d in 0 1 2 3 4 7; do
  echo "dbg=$d"; SEM_K2_DEBUG=$d python tools/cg_variants.py 2>&1 | tail -1 | cut -c1-220
  SEM_K2_DEBUG=$d ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv -k regex:k2_kernel -s 200 -c 20 python tools/cg_variants.py 2>/dev/null | grep k2_kernel | tail -3 | awk -F'","' '{print $NF}'
done
