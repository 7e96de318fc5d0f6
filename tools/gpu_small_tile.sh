# Small-tile GEMM check: kernel tests, then C1-C3 timings with the tile forced / automatic.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -3
for t in 128 64 auto; do
  if [ $t = auto ]; then unset HEFF_GEMM_TILE; else export HEFF_GEMM_TILE=$t; fi
  timeout 300 python tools/sweep.py --configs c1,c2,c3 --reps 50 > gpurun_out/sweep_tile$t.json 2> gpurun_out/sweep_tile$t.err
  echo "tile $t rc=$?"; tail -2 gpurun_out/sweep_tile$t.err
done
