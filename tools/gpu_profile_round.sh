set -x
mkdir -p gpurun_out
timeout 600 python tools/sweep.py --configs c1,c2,c3,c4 --out gpurun_out/sweep.json 2>&1 | tail -6
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_dmma|mpo_order|multidot|multiaxpy|reduce_partial|scale_kernel|lanczos_alpha|relayout" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_dmma_tma|mpo_orderA" -s 3 -c 3 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
