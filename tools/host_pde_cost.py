import sys, time, ctypes as C, torch
sys.path.insert(0, '/root/repo')
from paper_2109_04131_b200 import binding as B
from usfft_inputs import config
cfg = config(2); ctx = B.Context(0)
p = B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 1, cfg["d"], cfg["N"], cfg["s"], "A", 1000)
pde = B.pde_desc(cfg)
u = torch.empty((961, 4), dtype=torch.float64, device="cuda")
dsc, keep = p.desc(); pdsc, amp = pde
args = (ctx.h, C.byref(pdsc), C.byref(dsc), 0, 4, None, u.data_ptr(), 4, None, None, None)
f = ctx.lib.usfft_sample_pde
for _ in range(50): f(*args)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500): f(*args)
t1 = time.perf_counter(); torch.cuda.synchronize()
print("raw ctypes sample_pde: %.1f us" % (1e6 * (t1 - t0) / 500))
t0 = time.perf_counter()
for _ in range(500): B.usfft_sample_pde(ctx, pde, p, 0, 4, u, 4)
t1 = time.perf_counter(); torch.cuda.synchronize()
print("binding sample_pde: %.1f us" % (1e6 * (t1 - t0) / 500))
t0 = time.perf_counter()
for i in range(500): B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 1 + i % 5, cfg["d"], cfg["N"], cfg["s"], "A", 1000)
t1 = time.perf_counter()
print("binding plan_round: %.1f us" % (1e6 * (t1 - t0) / 500))
