import time, torch, sys
sys.path.insert(0, '/root/repo')
from heffgen import configs as C
from paper_2007_14822_b200 import Heff
dev = torch.device('cuda:0')
for m in (10, 50, 100, 200):
    x = C.make('c1', m=m, device=dev)
    for _ in range(3):
        with Heff(x.L, x.W1, x.W2, x.R) as h: pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        with Heff(x.L, x.W1, x.W2, x.R) as h: pass
    torch.cuda.synchronize()
    tc = (time.perf_counter() - t0) / 50
    with Heff(x.L, x.W1, x.W2, x.R) as h:
        psi = x.psi.clone()
        h.lanczos_ground(psi.clone(), max_iter=40, tol=1e-12, converge=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = 0
        for _ in range(20):
            r = h.lanczos_ground(psi.clone(), max_iter=40, tol=1e-12, converge=True)
            n += r.iters
        torch.cuda.synchronize()
        tl = (time.perf_counter() - t0) / 20
    print(f"m={m}: create+destroy {tc*1e3:.3f} ms; lanczos converge {tl*1e3:.3f} ms ({n/20:.1f} iters, {tl/(n/20)*1e6:.0f} us/iter)")
