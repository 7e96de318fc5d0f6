# PDL check: split tests, then split timings with and without programmatic dependent launch
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_split_qn.py -q -x 2>&1 | tail -2
for v in pdl nopdl; do
  if [ $v = nopdl ]; then export HEFF_NO_PDL=1; else unset HEFF_NO_PDL; fi
  timeout 600 python tools/bench_split.py --configs c2,c3,c4 --kinds random --reps 3 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  r=json.loads(l); print('$v', r['config'], r['dir'], round(r['ms'],2), r['sweeps'])
"
done
