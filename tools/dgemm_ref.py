"""cuBLAS DGEMM context numbers (torch.matmul float64) at the hot-path GEMM shapes.
Context only -- not the product path; see DESIGN.md."""
import torch, time, json, sys
torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
res = {}
for (M, N, K, tag) in [(8192, 8192, 8192, "8192^3"), (5120, 4096, 1024, "C3 GEMM1"), (4096, 1024, 5120, "C3 GEMM4"),
                       (81920, 16384, 4096, "C4 GEMM1"), (16384, 4096, 81920, "C4 GEMM4")]:
    a = torch.randn(M, K, dtype=torch.float64, device=dev)
    b = torch.randn(K, N, dtype=torch.float64, device=dev)
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3 if M * N * K > 1e12 else 10
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2 * M * N * K / ms / 1e9
    res[tag] = {"M": M, "N": N, "K": K, "ms": ms, "tflops": tf}
    print(f"cuBLAS DGEMM {tag} {M}x{N}x{K}: {ms:.3f} ms  {tf:.2f} TFLOP/s", flush=True)
    del a, b, c
    torch.cuda.empty_cache()
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else "dgemm.json", "w"), indent=1)
