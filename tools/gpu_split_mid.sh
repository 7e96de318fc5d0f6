# Mid-size split timing: phase breakdown (HEFF_SVD_TIMING) for 128..1024-bond two-site matrices.
mkdir -p gpurun_out
for m in 64 128 256 512; do
  HEFF_SVD_TIMING=1 timeout 120 python tools/split_once.py $m random 2>&1 | tail -3
done
timeout 300 python tools/bench_split.py --configs c2,c3 --kinds random --reps 5 2>/dev/null | cut -c1-400
