# Quick GPU check (gpurun -- bash tools/gpu_check.sh): the full GPU test suite and
# one headline bench line into gpurun_out/.  tools/gpu_final_r02.sh is the full evidence run.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02q_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02q_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02q_gputests.log
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err; echo "bench rc=$?"
cat gpurun_out/r02q_bench.json | head -c 3000
