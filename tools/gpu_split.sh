mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py -q -x --timeout 600 2>&1 | tail -25
