import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2109_04131_b200 import binding as B
from oracle import fe as ofe, lattice as olat
ctx = B.Context(0)
for d in (10, 32, 40, 48, 56, 64):
    cfg = dict(n=16, d=d, amp=[0.3 / (j * j) for j in range(1, d + 1)], theta="sin", form="affine", f="x2")
    p = B.usfft_plan_round(ctx, 3, 2, 2, 1, d, 4, 10, "A", 30)
    nb = 3
    Y = olat.nodes(p.M, p.z, p.shift, 2)[:, :nb]
    ref = ofe.sample_pde(cfg, Y)
    out = {}
    for pc in ("mg", "jacobi"):
        u = torch.empty((225, nb), dtype=torch.float64, device="cuda")
        B.usfft_sample_pde(ctx, B.pde_desc(cfg, precond=pc), p, 0, nb, u, nb)
        out[pc] = u.cpu().numpy()
    # explicit nodes path
    u = torch.empty((225, nb), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 0, nb, u, nb, torch.as_tensor(np.ascontiguousarray(Y), device="cuda"))
    out["nodes"] = u.cpu().numpy()
    print(d, {k: float(np.abs(v - ref).max() / np.abs(ref).max()) for k, v in out.items()})
