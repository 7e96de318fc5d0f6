# In-kernel stream-K fixup check: GEMM kernel tests, then C1-C3 timings (in-kernel vs fixup kernel).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -3
for m in inkernel fixupkernel; do
  if [ $m = fixupkernel ]; then export HEFF_SK_FIXUP_KERNEL=1; else unset HEFF_SK_FIXUP_KERNEL; fi
  timeout 300 python tools/sweep.py --configs c1,c2,c3 --reps 50 > gpurun_out/sweep_$m.json 2> gpurun_out/sweep_$m.err
  echo "$m rc=$?"; tail -2 gpurun_out/sweep_$m.err
done
