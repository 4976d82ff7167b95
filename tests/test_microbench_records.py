"""B200 microbench records: the emitter's CSV is read and fitted
by the REFERENCE's own load_records_csv + CostModel fit (oracle/_ref)."""
import importlib.util
import os

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tool():
    spec = importlib.util.spec_from_file_location(
        "microbench_records", os.path.join(ROOT, "tools", "microbench_records.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_records_csv_fits_with_reference(tmp_path):
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    ref = O.Reference()
    recs = [("WeightCopy", 1, 6.9, 0), ("WeightCopy", 1, 7.1, 0), ("ActivationCopy", 1, 0.004, 0),
            ("FastExec", 1, 0.06, 0), ("SlowExec", 1, 210.0, 0), ("SlowExec", 2, 420.0, 0),
            ("SlowExec", 3, 630.0, 0)]
    path = str(tmp_path / "r.csv")
    _tool().write_records(recs, path)
    fit = ref.fit_records(path, 2.0)
    assert fit["weight_copy_ms"] == pytest.approx(7.0)
    assert fit["activation_copy_ms"] == pytest.approx(0.004)
    assert fit["fast_exec_ms"] == pytest.approx(0.06)
    assert fit["slow_ms_per_token"] == pytest.approx(210.0)
    assert fit["slow_intercept_ms"] == pytest.approx(0.0, abs=1e-9)
    # on a B200 the paper's decode premise (CPU expert beats fetching it) fails
    assert fit["decode_assumption_check"] is False
    with open(path, "a") as f:
        f.write("Bogus,1,1.0,0\n")
    with pytest.raises(ValueError, match="ValidationError"):
        ref.fit_records(path)
