"""Pins the oracle's RNG/sampler restatement (oracle/rng_oracle.c) against
(1) the SURVEY Appendix-A known answers, produced by the reference's own
rng.hpp/sampling.hpp, (2) the committed golden fixtures generated from the
reference (tests/golden/make_golden.py), and (3) the reference library
itself when oracle/_ref is built here."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import srtt_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "sampling_golden.json")))

# (stream id, m, s, idx[0..2], idx[s-1], normal0, normal1)
APPENDIX_A = [
    (0, 16384, 52, (14177, 12504, 9324), 6713, -0.16178674819383701, -0.29063593100948915),
    (1, 16384, 52, (6532, 7759, 2602), 13172, -0.58914625180728386, 1.3864059732056599),
    (2, 16384, 52, (11587, 16088, 15943), 3874, 1.3434290453467079, -0.21798109082237663),
    (0, 2560000, 44, (11326, 1043782, 294888), 2298096, -0.097215114788188478, -1.140857080327754),
    (0, 8000000, 80, (1945958, 1598104, 5764188), 2016660, -0.066854775985292422, 1.6652668594934044),
    (1, 20736, 60, (8519, 15701, 10933), 13640, 2.3142352468726108, 0.058248384331463073),
    (7, 35831808, 60, (22611679, 18605699, 26736352), 4089621, 0.95347861985124494, -0.34204672577241679),
    (0, 4194304, 168, (1480808, 2780864, 3707388), 4035639, 0.76969009971477376, -0.43747745678138156),
]


@pytest.mark.parametrize("sid,m,s,first,last,n0,n1", APPENDIX_A)
def test_appendix_a_known_answers(sid, m, s, first, last, n0, n1):
    rng = O.RngStream(0, sid)
    idx = O.sample_indices(m, s, rng)
    assert tuple(idx[:3]) == first and idx[-1] == last
    nor = rng.normals(2)
    assert nor[0] == n0 and nor[1] == n1  # bit-exact (same libm on this host)


def test_golden_sampling_fixtures():
    for c in GOLDEN["sampling"]:
        rng = O.RngStream(c["seed"], c["stream"])
        if c["rc"] != 0:
            with pytest.raises(ValueError):
                O.sample_indices(c["m"], c["s"], rng, c["partitions"])
            continue
        idx = O.sample_indices(c["m"], c["s"], rng, c["partitions"])
        assert idx.tolist() == c["indices"], c
        nor = rng.normals(len(c["normals_after"]))
        assert [float.hex(float(v)) for v in nor] == c["normals_after"]


def test_golden_raw_draws():
    for r in GOLDEN["raw"]:
        assert [int(v) for v in O.RngStream(r["seed"], r["stream"]).next_u64(16)] == r["u64"]


def test_draw_counter_matches_sampling_consumption():
    # the device generator starts after the sampling draws: count them
    rng = O.RngStream(0, 0)
    O.sample_indices(16384, 52, rng)
    d = rng.draws
    assert d >= 52
    raw = O.RngStream(0, 0).next_u64(d + 2)
    nxt = rng.next_u64(1)[0]
    assert nxt == raw[d]


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(HERE), "oracle", "_ref",
                                                    "libsrtt_ref_sampling.so")),
                    reason="reference sampler not built here (make -C oracle ref)")
def test_against_reference_library_random_sweep():
    lib = C.CDLL(os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libsrtt_ref_sampling.so"))
    lib.ref_sample_then_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_void_p, C.c_int64, C.c_void_p]
    r = np.random.default_rng(7)
    for _ in range(500):
        m = int(r.integers(1, 10**9))
        s = int(r.integers(1, min(m, 400) + 1))
        parts = int(r.integers(1, min(s, 5) + 1)) if r.random() < 0.3 else 1
        seed, sid = int(r.integers(0, 2**63)), int(r.integers(0, 2**32))
        idx = np.zeros(s, np.int64)
        nor = np.zeros(7)
        rc = lib.ref_sample_then_normals(seed, sid, m, s, parts, idx.ctypes.data, 7, nor.ctypes.data)
        rng = O.RngStream(seed, sid)
        if rc:
            with pytest.raises(ValueError):
                O.sample_indices(m, s, rng, parts)
            continue
        assert np.array_equal(O.sample_indices(m, s, rng, parts), idx)
        assert np.array_equal(rng.normals(7), nor)


def test_gaussian_moments():
    """test_sampling.cpp:86-101: mean within 5 sigma, variance within 2%."""
    g = O.gaussian_matrix(1000, 1000, O.RngStream(13, 0))
    assert abs(g.mean()) <= 5.0 / 1000.0
    assert abs(g.var(ddof=1) - 1.0) <= 0.02
