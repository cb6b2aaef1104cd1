"""Diagnostics for the smoke round: GPU vs oracle per-node sets, lstar and coefficients."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import detect as odet, dft as odft, fe as ofe, lattice as olat
from paper_2109_04131_b200.driver import Detector
from usfft_inputs import config

cfg = config(1, mode="A")
det = Detector(cfg, device=0)
rng = np.random.default_rng(0)
t = 3
I_prev = np.unique(rng.integers(-8, 9, size=(12, t - 1)), axis=0)
kt = np.arange(-4, 5)
Id = torch.as_tensor(I_prev, dtype=torch.int16, device="cuda").contiguous()
ktd = torch.as_tensor(kt, dtype=torch.int16, device="cuda")
J = olat.candidates(I_prev, kt)
flags = torch.zeros(J.shape[0], dtype=torch.uint8, device="cuda")
res = det.round(2, t, 1, Id, I_prev.shape[0], ktd, cfg["s"], flags, want_coef=True)
p = res.plan
bins = olat.bins(J, p.z, p.M)
Y = olat.nodes(p.M, p.z, p.shift, t)
U_ref = ofe.sample_pde(cfg, Y)
U = res.u.cpu().numpy()
print("u err", np.abs(U - U_ref).max() / np.abs(U_ref).max())
V = odft.round_values(U_ref, p.M, p.L, bins)
ref = odet.detect_round(V, bins, cfg["s"], cfg["theta_rel"])
frag = odet.fragile(ref["kappa_min"], cfg["s"], ref["theta2"])
print("fragile", frag.sum(), "n_det gpu", res.n_det, "oracle", len(ref["det"]))
km = res.kappa_min.cpu().numpy()
print("kappa rel err", np.abs(np.sqrt(km) - np.sqrt(ref["kappa_min"])).max() / np.sqrt(ref["kappa_min"].max()))
print("theta2 gpu", res.theta2.item(), "oracle", ref["theta2"])
dg = res.det_g.cpu().numpy(); nd = res.n_det_g.cpu().numpy()
bad = [g for g in range(dg.shape[0]) if dg[g, :nd[g]].tolist() != ref["D"][g].tolist()]
print("nodes with different D_g:", len(bad), bad[:5])
if bad:
    g = bad[0]; print(dg[g, :nd[g]].tolist()); print(ref["D"][g].tolist())
ls = res.lstar.cpu().numpy()
print("lstar equal", np.array_equal(ls, ref["lstar"]), "fallbacks gpu", (ls < 0).sum(), "oracle", (ref["lstar"] < 0).sum())
c = res.coef.cpu().numpy(); cg = c[..., 0] + 1j * c[..., 1]
d = np.abs(cg - ref["coef"]); g, q = np.unravel_index(d.argmax(), d.shape)
print("coef max diff", d.max(), "at", g, q, "rel", d.max() / np.abs(ref["coef"]).max(), "lstar", ls[g, q], ref["lstar"][g, q], cg[g, q], ref["coef"][g, q])
Vg = np.abs(V).max(); print("max|V|", Vg)

km_ref = ref["kappa_min"]
dd = np.abs(np.sqrt(km) - np.sqrt(km_ref)); g, k = np.unravel_index(dd.argmax(), dd.shape)
print("worst kappa at g,k", g, k, "gpu", km[g, k], "oracle", km_ref[g, k])
Vg = odft.round_values(U, p.M, p.L, bins)          # oracle DFT of the GPU samples (diagnostic only)
kg = odet.kappa_min(Vg)
print("oracle-DFT-of-GPU-u vs GPU kappa:", np.abs(np.sqrt(kg) - np.sqrt(km)).max() / np.sqrt(km_ref.max()))
print("oracle-DFT-of-GPU-u vs oracle kappa:", np.abs(np.sqrt(kg) - np.sqrt(km_ref)).max() / np.sqrt(km_ref.max()))
sp = res.spectra.cpu().numpy(); Mh = p.M // 2 + 1
full = np.stack([odft.lattice_dft(U[:, l * p.M:(l + 1) * p.M], p.M, np.arange(Mh)) for l in range(p.L)], 1)
print("spectra err", np.abs((sp[..., 0] + 1j * sp[..., 1]) / p.M - full).max() / np.abs(full).max())
kk = odet.kappa(V)
print("per-lattice kappa at worst:", kk[:, g, k], "bins", bins[:, k])
