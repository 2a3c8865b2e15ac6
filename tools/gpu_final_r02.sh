# Final round-2 evidence run on one B200 (tools/gpu_final_r02.sh):
# full GPU suite, headline bench (+ variants, reference arm, FD), ncu launch
# list + full captures of K1 and K2, c4 order sweep.  Outputs in gpurun_out/.
mkdir -p gpurun_out
T=r02z
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_smi.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gputests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/${T}_gputests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?"
for v in "--precond jacobi" "--cg-variant single_reduction" "--operator screened"; do
  tag=$(echo $v | tr -d ' -' | cut -c1-14)
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $v > gpurun_out/${T}_bench_$tag.json 2>/dev/null; echo "variant $tag rc=$?"
done
timeout 600 python bench.py --workload fd --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_fd.json 2>/dev/null; echo "fd rc=$?"
timeout 900 python tools/order_sweep.py --out gpurun_out/order_sweep_${T}.json > gpurun_out/${T}_sweep.log 2>&1; echo "sweep rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'ax_dmma_kernel<1' -s 30 -c 1 -o gpurun_out/${T}_k1 python tools/cg_time.py --reps 1 > gpurun_out/${T}_ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k2_kernel<7, 0' -s 30 -c 1 -o gpurun_out/${T}_k2 python tools/cg_time.py --reps 1 > gpurun_out/${T}_ncu_k2.log 2>&1; echo "ncu k2 rc=$?"
echo done
