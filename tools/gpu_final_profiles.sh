# Refresh the per-config measurement files under gpurun_out/ (copied to profiles/ afterwards)
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --configs c1,c2,c3,c4,c5 --reps 5 --out gpurun_out/r01_sweep_final.json > /dev/null 2>&1; echo "sweep rc=$?"
timeout 900 python tools/bench_split.py --configs c1,c2,c3,c4 --kinds random,graded --reps 3 --out gpurun_out/r01_split_sweep_final.json > /dev/null 2>&1; echo "split rc=$?"
timeout 600 python tools/sweep_qn.py --out gpurun_out/r01_qn_sweep_final.json > /dev/null 2>&1; echo "qn rc=$?"
timeout 600 python tools/sweep_complex.py --out gpurun_out/r01_complex_sweep_final.json > /dev/null 2>&1; echo "complex rc=$?"
timeout 600 python tools/sweep_env.py > gpurun_out/r01_env_sweep_final.txt 2>&1; echo "env rc=$?"
timeout 900 python tools/shard_model.py --out gpurun_out/r01_shard_model_c4_final.json > /dev/null 2>&1; echo "shard rc=$?"
