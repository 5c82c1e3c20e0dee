"""Float64 CPU oracle for the tensor-based sketch hot path (arXiv 2209.14637).

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
directory; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may call it.  It shares no code
with the CUDA path (``paper_2209_14637_b200/``): no kernels, headers, helpers,
constants or pre/post-processing.

What it computes, each function citing the passage it follows (PAPER.md line
numbers, "P:NNN"):

* ``tucker1.mode1_gram``      G = A_(1) A_(1)^T = sum_d A_d A_d^T
* ``tucker1.tucker1_sketch``  S* = (U^(1))_k^T, the top-k left singular vectors of
                              A_(1), i.e. the top-k eigenvectors of G
* ``scw.scw``                 Algorithm 1: V from the SVD of SA, [AV]_r,
                              A_hat = [AV]_r V^T
* ``scw.scw_error``           ||A - SCW(A, S, r)||_F, dense residual
* ``scw.best_rank_r_error``   ||A - [A]_r||_F  (Eckart-Young)
* ``scw.test_error``          the paper's test-error metric
* ``tucker2``                 the two-sided variant (Algorithm 5): mode-2 Gram, HOOI,
                              two-sided SCW
* ``matrix_free``             the Tucker1 sketch by randomized block Krylov without forming G
                              (readings mf1-mf4 in DESIGN.md)
* ``validators``              Theorem 1 and Theorem 2 checks

Everything is numpy float64 with LAPACK/BLAS library primitives (matmul, eigh,
svd) as single steps; no blocking or reordering beyond the definitions.
Inputs are the fp32 arrays the GPU consumes, cast exactly to float64.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function to something
other than itself: brute force on the explicit mode-1 unfolding, the identical-
slices special case, closed forms on exactly-low-rank data, Eckart-Young,
k = m, Theorems 1 and 2, SPEC worked examples (tests/golden/).  No function here is
"parity unpinned" except the paper's dataset-bound Table 2 numbers, which this
oracle does not reproduce (datasets missing).
"""
from . import tucker1, scw, validators, tucker2, matrix_free  # noqa: F401
