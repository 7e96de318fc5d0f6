# GEMM raster (GROUP_M) vs C4 GEMM time and DRAM traffic
mkdir -p gpurun_out
for gm in 16 8 4 32; do
  export HEFF_GEMM_GROUP_M=$gm
  t=$(timeout 300 python tools/sweep.py --configs c4 --reps 2 2>/dev/null | python -c "
import sys,json
r=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(r['gemm_first_ms'],2), round(r['gemm_last_ms'],2))")
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_dmma -c 2 --csv --log-file gpurun_out/gm$gm.csv python tools/matvec_once.py c4 1 > /dev/null 2>&1
  echo "GROUP_M=$gm: $t"
  grep -h "dram__bytes" gpurun_out/gm$gm.csv | awk -F'","' '{print "   ", $5, $(NF-2), $(NF-1), $NF}' | cut -c1-160
done
