set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x 2>&1 | tail -4
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --config c3 --sharded --no-cpu-baseline 2>&1 | tail -2
timeout 600 python bench.py --steps 2 --warmup 3 --sharded --no-cpu-baseline --e2e-steps 1 2>&1 | tail -2
timeout 900 python tools/sweep.py --configs c5 --reps 3 --out gpurun_out/sweep_c5.json 2>&1 | tail -3
