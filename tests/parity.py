"""Fragility-aware comparison of one detection round, GPU vs oracle (reading Z25).

Decisions (k in D_g) may differ only where the oracle marks them fragile.  The resolved index
l*(k,g) depends only on D_g and the bins, so wherever the two D_g agree, l* must agree exactly
and the resolved values must agree to the value tolerance.
"""
import numpy as np


def compare_round(det_g, n_det_g, det_idx, lstar, coef, ref, frag, val_tol):
    """det_g/n_det_g/det_idx/lstar/coef: GPU arrays (numpy); ref: oracle detect_round dict;
    frag: oracle fragile mask [G][|J|].  Returns a dict of counts; raises AssertionError."""
    G = det_g.shape[0]
    same = np.zeros(G, dtype=bool)
    for g in range(G):
        mine = det_g[g, :n_det_g[g]].tolist()
        theirs = ref["D"][g].tolist()
        if not frag[g].any():                      # no fragile decision at g: D_g identical
            assert mine == theirs, f"D_g differs at node {g} with no fragile decision"
        diff = set(mine) ^ set(theirs)
        assert all(frag[g, k] for k in diff), f"non-fragile decision differs at node {g}: {sorted(diff)}"
        same[g] = not diff
    out = {"nodes": G, "nodes_same_D": int(same.sum()), "fragile": int(frag.sum()),
           "strict_set_check": not frag.any()}
    if not frag.any():
        assert det_idx.tolist() == ref["det"].tolist(), "round set differs with no fragile decision"
    if lstar is None:
        return out
    if det_idx.tolist() != ref["det"].tolist():
        # union differs (only possible through fragile decisions): compare the common columns
        common, ia, ib = np.intersect1d(det_idx, ref["det"], return_indices=True)
    else:
        ia = ib = np.arange(det_idx.shape[0])
    c = coef[..., 0] + 1j * coef[..., 1]
    for g in np.nonzero(same)[0]:
        assert np.array_equal(lstar[g, ia], ref["lstar"][g, ib]), f"l* differs at node {g}"
        err = np.abs(c[g, ia] - ref["coef"][g, ib]).max() if ia.size else 0.0
        assert err <= val_tol, f"resolved value differs at node {g}: {err:.3e} > {val_tol:.3e}"
    return out
