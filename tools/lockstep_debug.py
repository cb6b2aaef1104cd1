"""Config-2 lockstep debugging: run the GPU detection round by round with the oracle beside it and
dump the first round whose D_g differ without a fragile decision."""
import multiprocessing as mp
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import detect as odet, dft as odft, fe as ofe, lattice as olat, plan as oplan  # noqa
from usfft_inputs import config  # noqa


def _solve(job):
    cfg, Y = job
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        return ofe.sample_pde(cfg, Y)


def main():
    from paper_2109_04131_b200.driver import Detector
    cfg = config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
    pool = mp.get_context("fork").Pool(os.cpu_count())
    done = [False]

    class D(Detector):
        def round(self, step, t, i, I_prev, n_prev, kt, s_tilde, flags, want_coef=False, keep_iters=False,
                  counts=True):
            res = super().round(step, t, i, I_prev, n_prev, kt, s_tilde, flags, want_coef, keep_iters)
            if done[0] or step == 1:
                return res
            p = res.plan
            shift = oplan.shift(cfg["seed"], step, t, i, cfg["d"])
            J = olat.candidates(I_prev.cpu().numpy().astype(np.int64).reshape(n_prev, t - 1),
                                kt.cpu().numpy().astype(np.int64))
            Y = olat.nodes(p.M, p.z, shift, t)
            bins = olat.bins(J, p.z, p.M)
            parts = np.array_split(np.arange(Y.shape[1]), os.cpu_count())
            U = np.concatenate(pool.map(_solve, [(cfg, Y[:, q]) for q in parts]), axis=1)
            V = odft.round_values(U, p.M, p.L, bins)
            ref = odet.detect_round(V, bins, s_tilde, cfg["theta_rel"], want_coef=False)
            frag = odet.fragile(ref["kappa_min"], s_tilde, ref["theta2"])
            dg, nd = res.det_g.cpu().numpy(), res.n_det_g.cpu().numpy()
            kg = res.kappa_min.cpu().numpy()
            Ug = res.u.cpu().numpy()
            for g in range(dg.shape[0]):
                mine, theirs = dg[g, :nd[g]].tolist(), ref["D"][g].tolist()
                if mine != theirs and not frag[g].any():
                    done[0] = True
                    mo, mg = np.sqrt(ref["kappa_min"][g]), np.sqrt(kg[g])
                    print(f"round t={t} i={i} |J|={J.shape[0]} M={p.M} L={p.L} node {g}: s~={s_tilde}")
                    print("  samples max|dU| =", np.abs(Ug - U).max(), " max|U| =", np.abs(U).max())
                    print("  theta (oracle) =", np.sqrt(ref["theta2"]), " GPU theta2 =", float(res.theta2.item()) ** 0.5,
                          " max m oracle =", np.sqrt(ref["kappa_min"].max()), " GPU kmax =", res.kappa_max.item() ** 0.5)
                    print("  |D| gpu", len(mine), "oracle", len(theirs))
                    for k in sorted(set(mine) ^ set(theirs)):
                        print(f"   k={k} J={J[k].tolist()} in_gpu={k in mine} m_oracle={mo[k]:.6e} m_gpu={mg[k]:.6e}")
                    order = np.lexsort((np.arange(J.shape[0]), -mo))
                    print("  oracle rank of cut region:", [(int(j), f"{mo[j]:.4e}") for j in order[max(0, len(theirs) - 3):len(theirs) + 3]])
                    break
            return res

    det = D(cfg)
    det.run()
    print("done, mismatch found" if done[0] else "no mismatch")


if __name__ == "__main__":
    main()
