"""Runs the C++ re-hosting of the reference's test suites (tests/cpp/test_dropin.cpp)
against the drop-in moe_orch library (libmoe_orch_b200.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2402_07033_b200", "_build", "test_dropin")


def _run(which):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} not built (run __graft_entry__.build())")
    p = subprocess.run([BIN, which], capture_output=True, text=True, timeout=900)
    print(p.stdout[-4000:])
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
    return p.stdout


def test_dropin_host_cases():
    out = _run("cpu")
    assert " 0 failed checks" in out


@pytest.mark.gpu
def test_dropin_gpu_cases():
    out = _run("gpu")
    assert " 0 failed checks" in out
