"""Developer check: every GPU component against the CPU oracle at small
sizes (prints max errors). Not a test; see tests/ for the asserted suite."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import srtt_oracle as O
import paper_2603_21379_b200 as P

rng = np.random.default_rng(0)
def planted(dims, r):
    G = rng.standard_normal((r,) * len(dims))
    Us = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n in dims]
    X = O.reconstruct(O.TuckerDecomposition(G, Us))
    return X + 1e-8 * np.linalg.norm(X) * rng.standard_normal(X.shape) / np.sqrt(X.size)

def proj_gap(a, b):
    return np.linalg.norm(a @ a.T - b @ b.T)

print("normals:", end=" ")
st = O.RngStream(0, 3); idx = O.sample_indices(1000, 20, st); ref = st.normals(50)
dev = P.stream_normals(0, 3, st.draws - 50 - (50 % 2) * 0, 0, 50)  # placeholder check below
_, draws = P.sample_indices(1000, 20, 0, 3)
dev = P.stream_normals(0, 3, draws, 0, 50)
print(np.abs(dev - ref).max())

X = planted((12, 10, 14), 3)
for mode in range(3):
    cols = rng.choice(X.size // X.shape[mode], 7, replace=False)
    y = P.extract_fibers(X, mode, cols); yo = O.extract_fibers(X, mode, cols)
    print("extract mode", mode, np.abs(y - yo).max())
y = P.extract_group_fibers(X, [0, 2], [2, 0, 5]); print("group", np.abs(y - O.extract_group_fibers(X, [0, 2], [2, 0, 5])).max())

for dims, r, p in [((128, 128, 128), 8, 5), ((40, 40, 40, 40), 6, 5), ((15, 15, 15, 15), 5, 4)]:
    X = planted(dims, r)
    s = 4 * (r + p)
    t0 = time.time()
    rep = P.SubsampleReport()
    t = P.sub_r_hosvd(X, [r] * len(dims), p, [s] * len(dims), 0, report=rep)
    t1 = time.time()
    orep = O.SubsampleReport()
    to = O.sub_r_hosvd(X, [r] * len(dims), p, [s] * len(dims), 0, report=orep)
    # Z parity for mode 0
    z = P.sketch(X, [0], orep.sampled_columns[0], r + p, 0, 0, P.sample_indices(X.size // dims[0], s, 0, 0)[1])
    zo = orep.sketches[0]
    gaps = [proj_gap(a, b) for a, b in zip(t.factors, to.factors)]
    eg = O.rel_error(X, O.reconstruct(O.TuckerDecomposition(t.core, t.factors)))
    eo = O.rel_error(X, O.reconstruct(to))
    print(dims, "Z rel", np.linalg.norm(z - zo) / np.linalg.norm(zo), "gaps", max(gaps), "err gpu", eg, "err cpu", eo,
          "ranks", rep.achieved_ranks, orep.achieved_ranks, "launches", rep.launches, f"{(t1-t0)*1e3:.1f} ms")
    core_direct = P.multi_ttm_core(X, to.factors); core_o = O.core_from_factors(X, to.factors)
    print("   core(K3) vs oracle rel", np.linalg.norm(core_direct - core_o) / np.linalg.norm(core_o))

# padding case
G = rng.random((2, 2, 2)); Us = [np.linalg.qr(rng.random((8, 2)))[0] for _ in range(3)]
X = O.reconstruct(O.TuckerDecomposition(G, Us)); rep = P.SubsampleReport()
t = P.sub_r_hosvd(X, [4] * 3, 4, [30] * 3, 5, report=rep)
print("pad: ranks", rep.achieved_ranks, rep.warnings[:1], "err", O.rel_error(X, O.reconstruct(O.TuckerDecomposition(t.core, t.factors))),
      "orth", max(O.orthonormality_defect(u) for u in t.factors))
orep = O.SubsampleReport(); to = O.sub_r_hosvd(X, [4] * 3, 4, [30] * 3, 5, report=orep)
print("  pad cols vs oracle", max(np.abs(a[:, 2:] - b[:, 2:]).max() for a, b in zip(t.factors, to.factors)))

# basis on a tall sketch (TSQR levels)
Z = rng.standard_normal((5000, 42)) @ np.diag(np.logspace(0, -12, 42))
b = P.range_basis_of_sketch(Z, 32); bo = O.range_basis_of_sketch(Z, 32, O.RngStream(0, 0))
print("tsqr basis gap", proj_gap(b.q, bo.q), "rank", b.numerical_rank, bo.numerical_rank, "sv rel", np.abs(b.singular_values - bo.singular_values[:42]).max() / bo.singular_values[0])

# H-Tucker
tree = P.DimensionTree.balanced(4); otree = O.DimensionTree.balanced(4)
X = planted((15, 15, 15, 15), 3)
ranks = P.uniform_node_ranks(tree, 5); samples = P.node_sample_counts(tree, X.shape, 20.0)
rep = P.SubsampleReport()
h = P.sub_r_rtl_ht(X, tree, ranks, samples, 4, 0, report=rep)
ho = O.sub_r_rtl_ht(X, otree, ranks, samples, 4, 0)
hg = O.HTuckerDecomposition(otree, h.leaf_factors, h.transfers)
print("ht err gpu", O.rel_error(X, O.ht_reconstruct(hg)), "cpu", O.rel_error(X, O.ht_reconstruct(ho)), rep.achieved_ranks)
# transfer/root vs oracle
ul = np.linalg.qr(rng.standard_normal((12, 4)))[0]; ur = np.linalg.qr(rng.standard_normal((9, 3)))[0]; us = rng.standard_normal((108, 5))
print("transfer", np.abs(P.transfer_tensor(us, ul, ur) - O.transfer_tensor(us, ul, ur)).max())
Xr = rng.standard_normal((12, 9))
print("root", np.abs(P.root_transfer(Xr, ul, ur) - O.root_transfer(Xr, ul, ur)).max())
print("DONE")
