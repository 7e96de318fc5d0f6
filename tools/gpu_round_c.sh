mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x 2>&1 | tail -4
timeout 600 python tools/sweep.py --configs c1,c2,c3,c4 --out gpurun_out/sweep4.json 2>&1 | cut -c1-400
HEFF_NO_FUSED_STEP=1 timeout 600 python tools/sweep.py --configs c1,c2 --out gpurun_out/sweep4_nofuse.json 2>&1 | cut -c1-400
