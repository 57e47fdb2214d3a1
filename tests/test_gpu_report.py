"""Experiment driver end to end on the GPU (reference
test_experiment.cpp:58-208 for the hot-path methods)."""
import io

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_one_row_per_seed_with_tiny_planted_errors():
    from paper_2603_21379_b200 import report as R

    spec = R.ExperimentSpec(generator="tucker-planted", shape=[8, 8, 8], rank=3, method="sub-r-hosvd",
                            samples=20, runs=3, base_seed=5)
    rep = R.run_experiment(spec)
    assert len(rep.rows) == 3
    assert all(r.rel_error <= 1e-10 for r in rep.rows)
    assert rep.rows[0].seed == 5 and rep.rows[2].seed == 7
    assert R.join_x(rep.shape) == "8x8x8"


def test_identical_specs_reproduce_identical_errors_and_bytes():
    from paper_2603_21379_b200 import report as R

    spec = R.ExperimentSpec(shape=[8, 8, 8], rank=3, method="sub-r-hosvd", samples=20, runs=4, base_seed=11)
    a, b = R.run_experiment(spec), R.run_experiment(spec)
    assert [r.rel_error for r in a.rows] == [r.rel_error for r in b.rows]
    spec.timings = False
    assert R.csv_string(R.run_experiment(spec)) == R.csv_string(R.run_experiment(spec))


def test_sampling_fractions_and_summary():
    from paper_2603_21379_b200 import report as R

    spec = R.ExperimentSpec(shape=[6, 6, 6], rank=2, method="sub-r-hosvd", alpha=3.0, runs=1)
    rep = R.run_experiment(spec)
    assert len(rep.fractions) == 3
    for ln in rep.fractions:
        assert (ln.samples, ln.columns, ln.percent_text) == (18, 36, "50%")
    buf = io.StringIO()
    R.write_json_summary(rep, buf)
    assert "sampling_fractions" in buf.getvalue() and "50%" in buf.getvalue()


def test_strict_mode_rejects_rank_shortfall(tmp_path, O):
    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import report as R

    rng = np.random.default_rng(1)
    core = rng.standard_normal((2, 2, 2))
    fac = [np.linalg.qr(rng.standard_normal((8, 2)))[0] for _ in range(3)]
    x = O.reconstruct(O.TuckerDecomposition(core, fac))
    path = tmp_path / "strict.srtt"
    P.write_tensor(path, x)
    spec = R.ExperimentSpec(generator="file", input_path=str(path), rank=4, method="sub-r-hosvd", samples=20,
                            strict=True)
    with pytest.raises(R.CheckFailure):
        R.run_experiment(spec)


def test_file_generator_errors_match_oracle(tmp_path, O):
    """Rows from a file input: the GPU rel_error equals the oracle's error of
    the same decomposition (parity of the reporting step)."""
    import paper_2603_21379_b200 as P
    from paper_2603_21379_b200 import report as R

    x = np.random.default_rng(4).standard_normal((12, 10, 9))
    path = tmp_path / "x.srtt"
    P.write_tensor(path, x)
    spec = R.ExperimentSpec(generator="file", input_path=str(path), rank=3, method="sub-r-hosvd", samples=20,
                            oversampling=4, runs=2, base_seed=3)
    rep = R.run_experiment(spec)
    for row in rep.rows:
        t = O.sub_r_hosvd(x, [3, 3, 3], 4, rep.sample_counts, row.seed)
        want = O.rel_error(x, O.reconstruct(t))
        assert abs(row.rel_error - want) <= 1e-10 * max(want, 1.0)
    lines = R.csv_string(rep).splitlines()
    assert len(lines) == 3 and R.parse_csv_line(lines[1])[3] == "12x10x9"


def test_hierarchical_experiment_runs_end_to_end():
    from paper_2603_21379_b200 import report as R

    spec = R.ExperimentSpec(generator="htucker-planted", shape=[8, 8, 8, 8], rank=3, method="sub-r-rtl-ht",
                            alpha=10.0, runs=2)
    rep = R.run_experiment(spec)
    assert len(rep.rows) == 2
    assert all(r.rel_error <= 1e-7 for r in rep.rows)
    assert rep.fractions and "sub-r-rtl-ht" in R.csv_string(rep)
