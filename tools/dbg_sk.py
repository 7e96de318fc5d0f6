import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2007_14822_b200.heff import gemm, lib
dev = torch.device('cuda:0')
torch.manual_seed(0)
M, N, K = 1280, 1024, 256
A = torch.randn(M, K, dtype=torch.float64, device=dev)
B = torch.randn(K, N, dtype=torch.float64, device=dev)
ref = A @ B
outs = []
for rep in range(3):
    C = gemm(A, B, False)
    torch.cuda.synchronize()
    outs.append(C.clone())
print('run-to-run identical:', torch.equal(outs[0], outs[1]), torch.equal(outs[1], outs[2]))
ws = torch.empty(2 * 148 * 128 * 128, dtype=torch.float64, device=dev)
lib().heff_debug_gemm_ws.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
print('copy rc', lib().heff_debug_gemm_ws(ws.data_ptr(), ws.numel() * 8))
torch.cuda.synchronize()
ws = ws.reshape(296, 128, 128)
total, grid, kt = 80 * 16, 148, 16
def coords(tile):  # group_m 16, num_m 10, num_n 8
    return tile % 10, tile // 10
nbad = 0
for b in range(grid):
    it, end = total * b // grid, total * (b + 1) // grid
    first = True
    while it < end:
        local = it // kt; kb0 = it - local * kt; kb1 = min(kt, kb0 + end - it); it += kb1 - kb0
        mb, nb = coords(local)
        exp = A[mb*128:(mb+1)*128, kb0*16:kb1*16] @ B[kb0*16:kb1*16, nb*128:(nb+1)*128]
        slot = 2 * b + (0 if first else 1)
        err = (ws[slot] - exp).abs().max().item()
        if err > 1e-10:
            nbad += 1
            if nbad < 12: print('slot', slot, 'cta', b, 'tile', local, (mb, nb), 'kb', kb0, kb1, 'err', err)
        first = False
print('bad slots', nbad)
D = outs[-1] - ref
print('bad tiles', (D.abs() > 1e-9).reshape(10, 128, 8, 128).any(dim=3).any(dim=1).nonzero().tolist())
# identify what the bad slots contain
for b in range(grid):
    it, end = total * b // grid, total * (b + 1) // grid
    local = it // kt; kb0 = it - local * kt; kb1 = min(kt, kb0 + end - it)
    mb, nb = coords(local)
    exp = A[mb*128:(mb+1)*128, kb0*16:kb1*16] @ B[kb0*16:kb1*16, nb*128:(nb+1)*128]
    if (ws[2*b] - exp).abs().max().item() < 1e-10:
        continue
    found = []
    for t2 in range(80):
        m2, n2 = coords(t2)
        for a0 in range(16):
            for a1 in range(a0 + 1, 17):
                e2 = A[m2*128:(m2+1)*128, a0*16:a1*16] @ B[a0*16:a1*16, n2*128:(n2+1)*128]
                if (ws[2*b] - e2).abs().max().item() < 1e-9:
                    found.append((t2, a0, a1))
    # also: maybe sum of expected + something
    diff = ws[2*b] - exp
    rows_bad = (diff.abs() > 1e-9).any(dim=1).nonzero().flatten().tolist()
    cols_bad = (diff.abs() > 1e-9).any(dim=0).nonzero().flatten().tolist()
    print('cta', b, 'tile', local, 'kb', kb0, kb1, 'matches', found[:4], 'bad rows', rows_bad[:8], len(rows_bad), 'bad cols', cols_bad[:8], len(cols_bad))
