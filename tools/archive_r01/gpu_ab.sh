# A/B: the library in ab/old (an older build) vs the current tree, same box
mkdir -p gpurun_out
for rep in 1 2; do
  (cd ab/old && timeout 300 python ../../tools/cg_variants.py 2>&1 | tail -1 | sed 's/^/old /')
  timeout 300 python tools/cg_variants.py 2>&1 | tail -1 | sed 's/^/new /'
done
