# bench + launch list + one ncu --set full capture of the hot kernels (run under gpurun)
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json | cut -c1-300
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_dmma|mpo_order|multidot|multiaxpy|reduce_partial|scale_kernel|lanczos_alpha|relayout|streamk|cgs2" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_dmma_tma|mpo_orderA|streamk" -s 4 -c 4 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
