# round 1 (e): re-validate after container restore: smoke, GPU tests, bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r01e.log 2>&1; tail -1 gpurun_out/smoke_r01e.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01e.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01e.log
timeout 600 python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err; tail -2 gpurun_out/bench_r01e.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01e.json 2> gpurun_out/bench_ref_r01e.err
cat gpurun_out/bench_r01e.json | cut -c1-400
