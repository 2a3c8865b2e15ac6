# round 1 (q): FD strip height sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ty in 32 64 128 256; do
  SEM_FD_STRIP=$ty timeout 300 python bench.py --workload fd --steps 20 --no-cpu-baseline > gpurun_out/bench_fd_r01q_$ty.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_fd_r01q_$ty.json').read().strip().splitlines()[-1])
print($ty, {k:round(v['mnodes_s']/1e3) for k,v in d['sweep'].items()})"
done
