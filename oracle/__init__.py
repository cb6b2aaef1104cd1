"""CPU oracle for the usFFT detection step of arXiv 2109.04131 — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA path is checked
against.  It is NOT part of the product:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
  ``--impl reference`` legs may import it;
* it shares no code with ``paper_2109_04131_b200/`` (no kernels, headers, helpers, tables or
  constant generators) and neither side imports the other; the only module both sides may
  consume is ``usfft_inputs`` (seeded synthetic inputs, none of the method's arithmetic);
* every floating-point step is fp64 numpy/scipy, written as the paper's definition or
  algorithm step by step.  Library primitives (a banded Cholesky solve, ``np.sort``,
  ``np.fft.fftn`` for the brute-force pin) serve as single steps only.

Citation convention: ``P:n`` = line n of the paper's PAPER.md (LaTeX source), with the
section / equation / algorithm it falls in; ``S:n`` = line n of SPEC.md.  Readings of
places where the paper is silent are labelled Z1..Z31 as in DESIGN.md §3.

Pin status (what fixes each function besides itself; see tests/test_oracle_*.py):

=====================  ==========================================================
function               pin
=====================  ==========================================================
plan.sm64              published SplitMix64 output for state 0
plan.* (M, L rules)    primality/smoothness by trial division; closed-form sizes
lattice.nodes/bins     SPEC worked examples; exact rational identity k.y_i = i.b(k)/M
lattice.injective      SPEC examples; brute-force pair check
fe.assemble/solve      5-point Laplacian stencil for a=1; manufactured solutions O(h^2);
                       SPD + M-matrix (u >= 0); y=0 -> a=1; ellipticity bounds
fe.psi / diag_index    Table 3 m1/m2/k (golden); affine a_min/a_max 0.1/1.9
/ f_values (examples)  and c ~ 0.547; lognormal P(|b| <= 3) > 99%;
                       zero sets of psi_j; f = 1 load h^2; product-to-sum identity of f
fe.tau1/tau2/phi_delta SPEC examples, poles, symmetry, inversion-method distribution
dft.lattice_dft        orthogonality; exact recovery of trig polynomials on a
                       reconstructing lattice; brute-force tensor-grid FFT for t <= 3
detect.*               brute force on tiny inputs; Thm 1.1 exact recovery of sparse
                       trig polynomials (SPEC acceptance 1); invariants
usfft.run              exact support/coefficient recovery on sparse trig polynomials
evaluate.evaluate      SPEC special cases; direct trig identities
cover.build_cover      brute-force alias-freeness against the full set; Remark 4 lattice
                       count / size bound; singleton
cover.cover_coeffs     exact recovery of polynomials supported on I; zero samples
cover.errors           closed forms (constant offset, single spike, complex modulus)
moments.expectation    E[u(Y)] of known functions of uniform / normal Y through the tent /
                       phi_Delta periodizations + FFT; half-period Gauss-Legendre integral
moments.variance/gsi   Parseval; Sobol components by brute-force conditional means (d = 3)
index_sets.brute_force the set definitions of P:1630-1638 as a filter of the box (itself
                       the pin of the package's budgeted enumeration)
mode-A detected sets   parity unpinned on PDE data (only trig-polynomial exactness pins
on PDE samples         the algorithm; PDE-data sets are oracle-vs-GPU only, Z25)
=====================  ==========================================================
"""
