# round 1 (aa): relabelled-mesh PCG / single-reduction GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_cg_sr.py -q -k "relabel" > gpurun_out/pytest_relabel_r01aa.log 2>&1; tail -2 gpurun_out/pytest_relabel_r01aa.log
