"""Oracle: the black-box sampler — one P1 finite-element solve per parameter node
(test infrastructure only, see oracle/__init__.py).

Problem (eq. pde; weak form P:155-158): find u(., y) in H^1_0(D), D = (0,1)^2, with
    int_D a(x,y) grad u . grad v dx = int_D f v dx   for all v in H^1_0(D).
"we just evaluate the finite element solution u(., y) at the given point x_g": the
G values u(x_g, y) of one solve are the G samples of one node y (Alg. 1 Step 2c P:313).

Random coefficient (eq. random_coefficient_1; lognormal P:94-98), in the form the
BASELINE configs and the paper's three examples instantiate (Z14/Z15/Z28):
    affine form:     a(x,y) = 1 + sum_j amp_j * theta(y_j) * psi_j(x)
    lognormal form:  a(x,y) = exp( sum_j amp_j * theta(y_j) * psi_j(x) )
    psi_j = sin(j pi x1) sin(j pi x2)                  (BASELINE configs, periodic example P:1006)
          | cos(2 pi m1(j) x1) cos(2 pi m2(j) x2)      (affine example P:1207, Table 3)
          | sin(2 pi j x1) cos(2 pi (d+1-j) x2)        (lognormal example P:1418)
    theta = sin(2 pi y)              (periodic model Theta_j)
          | 1 - |2(1 - 2y)|          (tent, eq. tent P:473-479 with alpha=-1, beta=1)
          | clip(Phi^-1(y), -6, 6)   (lognormal config literal reading, Z15)
          | clip(tau1(tau2_Delta(y)), -6, 6)  (lognormal periodization phi_Delta, Z27)
    f = x2 | 1 | sin(1.3 pi x1 + 3.4 pi x2) cos(4.3 pi x1 - 3.1 pi x2)

Discretisation (Z11, Z12): uniform n x n cells of width h = 1/n, each split
by its SW->NE diagonal into T_lo = {(i,j),(i+1,j),(i+1,j+1)} and T_up = {(i,j),(i+1,j+1),(i,j+1)};
P1 elements; a and f taken at the triangle centroid (one-point rule); zero Dirichlet data;
interior node (i,j), 1 <= i,j <= n-1, has index (j-1)(n-1) + (i-1) (x1 fastest).

Assembly is element by element with the textbook P1 formulas; the solve is a banded Cholesky
factorisation (LAPACK via scipy: a library primitive used as one step).  Nothing here uses
the 5-point stencil the GPU path derives from it (that derivation is *checked* against this).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.special


# ---------------------------------------------------------------------------------------------
# coefficient field
# ---------------------------------------------------------------------------------------------
def tau2(y: np.ndarray, delta: float) -> np.ndarray:
    """Shifted tent tau_{2,Delta}: T -> [-1/2, 1/2] (three branches)."""
    y = np.asarray(y, dtype=np.float64)
    return np.where(y < delta, -0.5 - 2.0 * (y - delta),
                    np.where(y < 0.5 + delta, -0.5 + 2.0 * (y - delta), 1.5 - 2.0 * (y - delta)))


def tau1(yb: np.ndarray) -> np.ndarray:
    """tau_1(y) = sqrt(2) erf^-1(2 y) on (-1/2, 1/2), written as Phi^-1(y + 1/2) with
    Phi(y) = (1 + erf(y / sqrt 2)) / 2."""
    return scipy.special.ndtri(np.asarray(yb, dtype=np.float64) + 0.5)


def global_delta(M0: int) -> float:
    """The one global pole shift of a run (reading Z27): Delta_opt = 1/(4 M0) of the Lemma
     for M0 = the Step-2 lattice size of the configuration (Z2)."""
    return 1.0 / (4.0 * M0)


def theta_map(kind: str, y: np.ndarray, delta: float | None = None) -> np.ndarray:
    """Theta_j(y_j) of the coefficient families (Z14, Z15, Z27)."""
    y = np.asarray(y, dtype=np.float64)
    if kind == "sin":
        return np.sin(2.0 * np.pi * y)                               # P:91 (without 1/sqrt6)
    if kind == "tent":
        return 1.0 - np.abs(2.0 * (1.0 - 2.0 * y))                   # eq. tent, alpha=-1, beta=1
    if kind == "probit":
        return np.clip(scipy.special.ndtri(y), -6.0, 6.0)            # Phi^-1 clipped (Z15)
    if kind == "phi_delta":                                          # phi_Delta = tau1 o tau2 (Z27)
        return np.clip(tau1(tau2(y, delta)), -6.0, 6.0)              # eq. lognormal_transfo
    raise ValueError(f"unknown theta kind {kind!r}")


def diag_index(j: int):
    """(m_1(j), m_2(j), k(j)) of the affine example (Table 3):
    k(j) = floor(-1/2 + sqrt(1/4 + 2j)), m_1(j) = j - k(j)(k(j)+1)/2, m_2(j) = k(j) - m_1(j)."""
    k = int(np.floor(-0.5 + np.sqrt(0.25 + 2.0 * j)))
    m1 = j - k * (k + 1) // 2
    return m1, k - m1, k


def psi(model: dict, j: int, x1: np.ndarray, x2: np.ndarray) -> np.ndarray:
    """psi_j(x) / amp_j, the spatial factor of term j (1-based) of the coefficient:
    "sinsin"      sin(j pi x1) sin(j pi x2)                          (periodic example)
    "cos_diag"    cos(2 pi m_1(j) x1) cos(2 pi m_2(j) x2)            (affine example)
    "sin_cos_rev" sin(2 pi j x1) cos(2 pi (d + 1 - j) x2)            (lognormal example)
    (the factor c j^-mu of the first two and 1/j of the third is amp_j)."""
    kind = model.get("psi", "sinsin")
    x1 = np.asarray(x1, dtype=np.float64)
    x2 = np.asarray(x2, dtype=np.float64)
    if kind == "sinsin":
        return np.sin(j * np.pi * x1) * np.sin(j * np.pi * x2)
    if kind == "cos_diag":
        m1, m2, _ = diag_index(j)
        return np.cos(2.0 * np.pi * m1 * x1) * np.cos(2.0 * np.pi * m2 * x2)
    if kind == "sin_cos_rev":
        return np.sin(2.0 * np.pi * j * x1) * np.cos(2.0 * np.pi * (model["d"] + 1 - j) * x2)
    raise ValueError(f"unknown psi family {kind!r}")


def coefficient(model: dict, y: np.ndarray, x1: np.ndarray, x2: np.ndarray) -> np.ndarray:
    """a(x, y) at the points (x1, x2) for one parameter vector y (length d):
    1 + sum_j amp_j theta(y_j) psi_j(x) (affine form) or exp(sum_j ...) (lognormal form)."""
    d = model["d"]
    th = theta_map(model["theta"], np.asarray(y, dtype=np.float64)[:d], model.get("delta"))
    s = np.zeros_like(np.asarray(x1, dtype=np.float64))
    for j in range(1, d + 1):
        s = s + model["amp"][j - 1] * th[j - 1] * psi(model, j, x1, x2)
    if model["form"] == "affine":
        return 1.0 + s
    if model["form"] == "exp":
        return np.exp(s)
    raise ValueError(f"unknown coefficient form {model['form']!r}")


# ---------------------------------------------------------------------------------------------
# mesh
# ---------------------------------------------------------------------------------------------
def triangles(n: int):
    """The 2n^2 triangles as integer vertex coordinates [2n^2][3][2] (Z11)."""
    tris = []
    for cj in range(n):
        for ci in range(n):
            tris.append([(ci, cj), (ci + 1, cj), (ci + 1, cj + 1)])      # T_lo
            tris.append([(ci, cj), (ci + 1, cj + 1), (ci, cj + 1)])      # T_up
    return np.asarray(tris, dtype=np.int64)


def node_index(n: int, i: np.ndarray, j: np.ndarray) -> np.ndarray:
    """Interior node number (x1 fastest); -1 on the Dirichlet boundary."""
    inside = (i >= 1) & (i <= n - 1) & (j >= 1) & (j <= n - 1)
    return np.where(inside, (j - 1) * (n - 1) + (i - 1), -1)


def node_coords(n: int):
    """x_g of the G = (n-1)^2 interior nodes, in node order."""
    jj, ii = np.meshgrid(np.arange(1, n), np.arange(1, n), indexing="ij")
    return ii.reshape(-1) / n, jj.reshape(-1) / n


# ---------------------------------------------------------------------------------------------
# assembly
# ---------------------------------------------------------------------------------------------
def element_matrices(n: int, a_T: np.ndarray):
    """Local P1 stiffness K_T[p][q] = a_T |T| grad(phi_p) . grad(phi_q) for every triangle.

    grad(phi_p) = (y_{p+1} - y_{p+2}, x_{p+2} - x_{p+1}) / (2 |T|_signed) (textbook P1).
    """
    tri = triangles(n).astype(np.float64) / n                    # physical coordinates
    x = tri[:, :, 0]
    yv = tri[:, :, 1]
    area2 = (x[:, 1] - x[:, 0]) * (yv[:, 2] - yv[:, 0]) - (x[:, 2] - x[:, 0]) * (yv[:, 1] - yv[:, 0])
    grads = np.empty((tri.shape[0], 3, 2))
    for p in range(3):
        p1, p2 = (p + 1) % 3, (p + 2) % 3
        grads[:, p, 0] = (yv[:, p1] - yv[:, p2]) / area2
        grads[:, p, 1] = (x[:, p2] - x[:, p1]) / area2
    area = 0.5 * np.abs(area2)
    K = np.einsum("tpc,tqc->tpq", grads, grads) * (a_T * area)[:, None, None]
    return K, area


def centroids(n: int):
    tri = triangles(n).astype(np.float64) / n
    c = tri.mean(axis=1)
    return c[:, 0], c[:, 1]


def assemble(n: int, a_T: np.ndarray, f_T: np.ndarray):
    """Banded (upper, LAPACK 'ab' layout) stiffness matrix and load vector.

    Load: b_p += f(c_T) |T| / 3 for the three vertices of T (centroid rule).
    Boundary rows/columns are dropped (zero Dirichlet data).
    Returns (ab, b) with ab[u + r - c, c] = A[r, c] for r <= c, bandwidth u = n.
    """
    G = (n - 1) ** 2
    u = n                                                # largest |index difference| = n
    K, area = element_matrices(n, a_T)
    tri = triangles(n)
    idx = node_index(n, tri[:, :, 0], tri[:, :, 1])      # [T][3]
    ab = np.zeros((u + 1, G))
    b = np.zeros(G)
    for p in range(3):
        rows = idx[:, p]
        ok = rows >= 0
        np.add.at(b, rows[ok], (f_T * area / 3.0)[ok])
        for q in range(3):
            cols = idx[:, q]
            sel = ok & (cols >= 0) & (rows <= cols)
            np.add.at(ab, (u + rows[sel] - cols[sel], cols[sel]), K[sel, p, q])
    return ab, b


def banded_to_dense(ab: np.ndarray) -> np.ndarray:
    u = ab.shape[0] - 1
    G = ab.shape[1]
    A = np.zeros((G, G))
    for c in range(G):
        for r in range(max(0, c - u), c + 1):
            A[r, c] = ab[u + r - c, c]
            A[c, r] = ab[u + r - c, c]
    return A


def banded_matvec(ab: np.ndarray, x: np.ndarray) -> np.ndarray:
    u = ab.shape[0] - 1
    G = ab.shape[1]
    out = ab[u] * x
    for k in range(1, u + 1):                      # superdiagonal k: A[c-k, c] = ab[u-k, c]
        v = ab[u - k, k:]
        out[:G - k] += v * x[k:]
        out[k:] += v * x[:G - k]
    return out


def f_values(model: dict, x1: np.ndarray, x2: np.ndarray) -> np.ndarray:
    kind = model.get("f", "x2")
    if kind == "x2":
        return np.asarray(x2, dtype=np.float64).copy()               # BASELINE configs: f = x2
    if kind == "one":
        return np.ones_like(np.asarray(x1, dtype=np.float64))        # affine example
    if kind == "trig":                                               # lognormal example
        x1 = np.asarray(x1, dtype=np.float64)
        x2 = np.asarray(x2, dtype=np.float64)
        return np.sin(1.3 * np.pi * x1 + 3.4 * np.pi * x2) * np.cos(4.3 * np.pi * x1 - 3.1 * np.pi * x2)
    if callable(kind):
        return np.asarray(kind(x1, x2), dtype=np.float64)
    raise ValueError(f"unknown right-hand side {kind!r}")


def solve(model: dict, y: np.ndarray, return_residual: bool = False):
    """u(x_g, y) at every interior node for one parameter node y (Alg. 1 Step 2c)."""
    n = model["n"]
    cx, cy = centroids(n)
    if "a_func" in model:                                            # manufactured pins
        a_T = np.asarray(model["a_func"](cx, cy), dtype=np.float64)
    else:
        a_T = coefficient(model, y, cx, cy)
    f_T = f_values(model, cx, cy)
    ab, b = assemble(n, a_T, f_T)
    cb = scipy.linalg.cholesky_banded(ab, lower=False)
    u = scipy.linalg.cho_solve_banded((cb, False), b)
    if return_residual:
        r = b - banded_matvec(ab, u)
        return u, float(np.linalg.norm(r) / np.linalg.norm(b))
    return u


def sample_pde(model: dict, Y: np.ndarray) -> np.ndarray:
    """Samples u(x_g, y_b) for all nodes y_b (columns of Y, [d][B]) -> [G][B] (sample fastest)."""
    Y = np.asarray(Y, dtype=np.float64)
    G = (model["n"] - 1) ** 2
    U = np.empty((G, Y.shape[1]))
    for bcol in range(Y.shape[1]):
        U[:, bcol] = solve(model, Y[:, bcol])
    return U
