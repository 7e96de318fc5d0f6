# pair-eigen rewrite check: split tests + mid/large split timings + the eig microbenchmark
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DEIG_NO_INSTR -I paper_2007_14822_b200/csrc tools/eigbench/eig_bench.cu -o /tmp/eig_bench && /tmp/eig_bench 16 | grep "inner=\|index-table"
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_split_qn.py tests/test_gpu_dmrg.py -q -x 2>&1 | tail -2
timeout 600 python tools/bench_split.py --configs c2,c3,c4 --kinds random --reps 3 2>/dev/null | cut -c1-300
