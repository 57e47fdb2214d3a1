"""Report layer (reference test_experiment.cpp:10-56 and the CSV/JSON
schema of experiment.cpp:367-497): formatting helpers on CPU."""
import io
import json
import math

import pytest

from paper_2603_21379_b200 import report as R


def test_method_flags():
    for m in R.METHODS:
        assert m in R.METHODS
    assert R.method_needs_samples("sub-r-hosvd") and R.method_needs_samples("sub-r-rtl-ht")
    assert not R.method_needs_samples("t-hosvd")
    assert R.method_is_hierarchical("rtl-ht") and not R.method_is_hierarchical("r-hosvd")


def test_format_percent_ceil():
    """test_experiment.cpp:27-36."""
    assert R.format_percent_ceil(75.0 / 15.0 ** 7) == "0.00005%"
    assert R.format_percent_ceil(1e4 / 16.0 ** 7) == "0.004%"
    assert R.format_percent_ceil(1e4 / 20.0 ** 7) == "0.0008%"
    assert R.format_percent_ceil(0.0) == "0%"
    assert R.format_percent_ceil(1.0) == "100%"
    assert R.format_percent_ceil(0.0035) == "0.4%"
    assert R.format_percent_ceil(0.004) == "0.4%"
    assert R.format_percent_ceil(0.01) == "1%"
    assert R.format_percent_ceil(0.5) == "50%"


def test_parse_csv_line():
    """test_experiment.cpp:38-51."""
    assert R.parse_csv_line("a,b,c") == ["a", "b", "c"]
    q = R.parse_csv_line('1,"x,y",3,"say ""hi"""')
    assert q[1] == "x,y" and q[3] == 'say "hi"'
    j = R.parse_csv_line('7,"[{""stage"":""svd"",""seconds"":0.5}]"')
    assert j[1] == '[{"stage":"svd","seconds":0.5}]'


def test_median():
    assert R.median([3.0, 1.0, 2.0]) == 2.0
    assert R.median([4.0, 1.0, 3.0, 2.0]) == 2.5
    with pytest.raises(ValueError):
        R.median([])


def _fake_report():
    spec = R.ExperimentSpec(shape=[6, 6, 6], rank=2, method="sub-r-hosvd", samples=12, runs=2)
    rep = R.RunReport(spec=spec, shape=[6, 6, 6], ranks=[2, 2, 2], sample_counts=[12, 12, 12], environment="env")
    rep.rows = [R.SeedResult(seed=1, rel_error=1.25e-9, total_seconds=0.0012345,
                             timings=[{"seconds": 1e-4, "stage": "sketch", "worker": 0}]),
                R.SeedResult(seed=2, rel_error=2.5e-9, total_seconds=0.002, timings=[])]
    rep.fractions = [R.SamplingFractionLine("mode 0", 18, 36, 0.5, "50%")]
    return rep


def test_csv_schema_round_trips():
    """test_experiment.cpp:108-141."""
    rep = _fake_report()
    text = R.csv_string(rep)
    lines = text.splitlines()
    assert lines[0] == R.CSV_HEADER
    hdr = R.parse_csv_line(lines[0])
    assert len(hdr) == 11 and hdr[0] == "seed" and hdr[10] == "stage_json"
    f = R.parse_csv_line(lines[1])
    assert len(f) == 11
    assert f[1] == "sub-r-hosvd" and f[3] == "6x6x6" and f[4] == "2x2x2" and f[5] == "12x12x12"
    assert f[6] == "4" and f[7] == "1"
    assert float(f[8]) == 1.25e-9 and f[9] == "0.001234"
    assert json.loads(f[10]) == [{"seconds": 1e-4, "stage": "sketch", "worker": 0}]
    assert R.parse_csv_line(lines[2])[10] == "[]"


def test_json_summary_and_scaling():
    rep = _fake_report()
    buf = io.StringIO()
    R.write_json_summary(rep, buf)
    j = json.loads(buf.getvalue())
    assert j["errors"]["median"] == pytest.approx(1.875e-9)
    assert j["sampling_fractions"][0]["percent"] == "50%"
    assert j["shape"] == "6x6x6" and j["order"] == 3 and j["runs"] == 2
    assert list(j) == sorted(j)                       # nlohmann key order
    buf = io.StringIO()
    R.write_scaling_json([(1, rep), (2, rep)], buf)
    s = json.loads(buf.getvalue())["scaling"]
    assert s[0]["workers"] == 1 and s[1]["speedup_total"] == pytest.approx(1.0)
    assert R.factor_stage_seconds(rep.rows[0]) == pytest.approx(1e-4)


def test_out_of_scope_methods_are_refused():
    import paper_2603_21379_b200 as P

    with pytest.raises(P.InvalidArgument, match="outside the B200 hot path"):
        R.resolve_problem(R.ExperimentSpec(method="t-hosvd", shape=[4, 4, 4], rank=2))
    with pytest.raises(P.InvalidArgument, match="unknown method"):
        R.resolve_problem(R.ExperimentSpec(method="nope"))
