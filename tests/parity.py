"""Parity helpers (SURVEY §8c procedure): subspace gaps between factor
spans, core comparison after factor alignment, reconstruction-error deltas."""
import numpy as np

import srtt_oracle as O


def projector_gap(a, b):
    """||A A^T - B B^T||_F for orthonormal A, B (test_htucker.cpp:216-217).
    Tall bases (the n x n projectors would not fit) use the equivalent
    sqrt(||(I - B B^T) A||_F^2 + ||(I - A A^T) B||_F^2), exact for orthonormal
    columns and free of cancellation."""
    if a.shape[0] > 25000:
        ra = a - b @ (b.T @ a)
        rb = b - a @ (a.T @ b)
        return float(np.sqrt(np.linalg.norm(ra) ** 2 + np.linalg.norm(rb) ** 2))
    return float(np.linalg.norm(a @ a.T - b @ b.T))


def aligned_core_error(core_g, factors_g, core_c, factors_c):
    """S_gpu x_k (U_gpu,k^T U_cpu,k)^T vs S_cpu, relative."""
    s = core_g
    for k, (ug, uc) in enumerate(zip(factors_g, factors_c)):
        s = O.ttm(s, (ug.T @ uc).T, k)
    return float(np.linalg.norm(s - core_c) / max(np.linalg.norm(core_c), 1e-300))


def tucker_rel_error(x, core, factors):
    return O.rel_error(x, O.reconstruct(O.TuckerDecomposition(core, factors)))
