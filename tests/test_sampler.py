"""The PRODUCT's host sampler (libsrtt_b200.so, srtt_sample_indices) is
bit-exact with the reference (golden fixtures generated from the
reference's own code) and reports the draw offset the device Gaussian
generator starts from. Host-only: runs without a GPU."""
import json
import os

import numpy as np
import pytest

import paper_2603_21379_b200 as P
import srtt_oracle as O

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sampling_golden.json")))


def test_golden_indices_bit_exact():
    for c in GOLDEN["sampling"]:
        if c["rc"] != 0:
            with pytest.raises(P.InvalidArgument):
                P.sample_indices(c["m"], c["s"], c["seed"], c["stream"], c["partitions"])
            continue
        idx, draws = P.sample_indices(c["m"], c["s"], c["seed"], c["stream"], c["partitions"])
        assert idx.tolist() == c["indices"], c


def test_draw_offsets_match_oracle():
    r = np.random.default_rng(3)
    for _ in range(200):
        m = int(r.integers(1, 10**8))
        s = int(r.integers(1, min(m, 300) + 1))
        seed, sid = int(r.integers(0, 2**62)), int(r.integers(0, 1000))
        idx, draws = P.sample_indices(m, s, seed, sid)
        rng = O.RngStream(seed, sid)
        assert np.array_equal(O.sample_indices(m, s, rng), idx)
        assert draws == rng.draws


def test_partition_counts():
    """test_sampling.cpp:51-76: 103 = 4*25 + 3 -> counts (2, 2, 2, 4)."""
    idx, draws = P.sample_indices(103, 10, 5, 0, 4)
    assert len(set(idx.tolist())) == 10
    counts = np.bincount(np.minimum(idx // 25, 3), minlength=4)
    assert counts.tolist() == [2, 2, 2, 4]
    assert draws == 0  # parent stream untouched (child streams)
    idx, _ = P.sample_indices(100, 8, 6, 0, 4)
    assert np.bincount(idx // 25, minlength=4).tolist() == [2, 2, 2, 2]


def test_sampling_properties_and_errors():
    """test_sampling.cpp:11-49."""
    idx, _ = P.sample_indices(100, 10, 1, 0)
    assert len(set(idx.tolist())) == 10 and idx.min() >= 0 and idx.max() < 100
    idx, _ = P.sample_indices(12, 12, 2, 0)
    assert sorted(idx.tolist()) == list(range(12))
    a, _ = P.sample_indices(100, 10, 42, 7)
    b, _ = P.sample_indices(100, 10, 42, 7)
    c, _ = P.sample_indices(100, 10, 42, 8)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    with pytest.raises(P.InvalidArgument):
        P.sample_indices(5, 6, 42, 7)
    with pytest.raises(P.InvalidArgument):
        P.sample_indices(50, 3, 7, 3, 4)  # more partitions than samples
    one, _ = P.sample_indices(50, 6, 7, 3, 1)
    plain, _ = P.sample_indices(50, 6, 7, 3)
    assert np.array_equal(one, plain)
