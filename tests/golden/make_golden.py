"""Generates tests/golden/sampling_golden.json from the REFERENCE's own
srtt::RngStream / sample_indices[_partitioned] (rng.hpp, sampling.hpp),
compiled from /root/reference by oracle/Makefile into
oracle/_ref/libsrtt_ref_sampling.so. Run here (the reference tree is not on
the GPU box); the JSON is committed.

    make -C oracle ref && python tests/golden/make_golden.py
"""
import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libsrtt_ref_sampling.so"))
vp, u64, i64 = C.c_void_p, C.c_uint64, C.c_int64
lib.ref_sample_then_normals.argtypes = [u64, u64, i64, i64, i64, vp, i64, vp]
lib.ref_next_u64.argtypes = [u64, u64, i64, vp]
lib.ref_child_u64.argtypes = [u64, u64, u64, i64, vp]
lib.ref_mixed_draws.argtypes = [u64, u64, i64, vp, vp]


def sample(seed, sid, m, s, parts, nn):
    idx = np.zeros(s, np.int64)
    nor = np.zeros(nn)
    rc = lib.ref_sample_then_normals(seed, sid, m, s, parts, idx.ctypes.data, nn, nor.ctypes.data)
    return rc, idx, nor


cases = []
# BASELINE config targets + reference test shapes
fixed = [(0, 0, 16384, 52, 1), (0, 1, 16384, 52, 1), (0, 2, 16384, 52, 1), (0, 0, 2560000, 44, 1),
         (0, 4, 2560000, 44, 1), (0, 0, 8000000, 80, 1), (0, 3, 8000000, 80, 1), (0, 1, 20736, 60, 1),
         (0, 2, 20736, 60, 1), (0, 3, 2985984, 60, 1), (0, 7, 35831808, 60, 1), (0, 14, 35831808, 60, 1),
         (0, 0, 4194304, 168, 1), (0, 2, 4194304, 168, 1), (1, 0, 100, 10, 1), (2, 0, 12, 12, 1),
         (3, 0, 1000, 1, 1), (42, 7, 100, 10, 1), (5, 0, 103, 10, 4), (6, 0, 100, 8, 4), (7, 3, 50, 6, 1),
         (5, 1, 1000, 21, 3), (9, 2, 3375, 75, 1), (0, 0, 3375, 75, 1)]
rng = np.random.default_rng(2026)
for _ in range(60):
    m = int(rng.integers(1, 10**8))
    s = int(rng.integers(1, min(m, 200) + 1))
    parts = int(rng.integers(1, min(s, 6) + 1)) if rng.random() < 0.3 else 1
    fixed.append((int(rng.integers(0, 2**63)), int(rng.integers(0, 2**20)), m, s, parts))
for seed, sid, m, s, parts in fixed:
    nn = 9
    rc, idx, nor = sample(seed, sid, m, s, parts, nn)
    cases.append({"seed": seed, "stream": sid, "m": m, "s": s, "partitions": parts, "rc": rc,
                  "indices": idx.tolist(), "normals_after": [float.hex(float(v)) for v in nor]})
raw = []
for seed, sid in [(0, 0), (123456789, 42), (9, 1), (2**63 + 5, 2**40)]:
    out = np.zeros(16, np.uint64)
    lib.ref_next_u64(seed, sid, 16, out.ctypes.data)
    child = np.zeros(4, np.uint64)
    lib.ref_child_u64(seed, sid, 3, 4, child.ctypes.data)
    raw.append({"seed": seed, "stream": sid, "u64": [int(v) for v in out], "child3_u64": [int(v) for v in child]})
kinds = np.array([0, 7, 0, 100, 2**62 + 3, 0, 1, 5], np.uint64)
mixed = np.zeros(len(kinds))
lib.ref_mixed_draws(11, 2, len(kinds), kinds.ctypes.data, mixed.ctypes.data)
doc = {"generator": "oracle/_ref (reference rng.hpp + sampling.hpp)", "sampling": cases, "raw": raw,
       "mixed": {"seed": 11, "stream": 2, "kinds": [int(k) for k in kinds],
                 "values": [float.hex(float(v)) for v in mixed]}}
with open(os.path.join(HERE, "sampling_golden.json"), "w") as f:
    json.dump(doc, f, indent=0)
print("wrote", len(cases), "sampling cases")
