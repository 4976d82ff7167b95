import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# Several peer-linked "ranks" share one GPU in the multi-rank tests, each with
# its own streams.  With CUDA's default 8 hardware work queues, two ranks'
# streams can land on one queue, and a rank's kernel that spins on another
# rank's flags then blocks that rank's kernels queued behind it (a false
# dependency that only times out).  Give every stream its own queue.  (Set
# before the CUDA context exists; on real multi-GPU runs each rank owns a GPU.)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")
    # a fresh checkout: build the in-tree libraries first (nvcc cross-compiles
    # without a GPU); an existing build is left alone
    lib = os.path.join(ROOT, "paper_2402_07033_b200", "_build", "libmoe_b200.so")
    if not os.path.exists(lib) and not os.environ.get("MOE_B200_LIB"):
        import subprocess

        subprocess.run(["make", "-s", "-j", str(os.cpu_count() or 4), "-C",
                        os.path.join(ROOT, "paper_2402_07033_b200", "csrc")], check=True)
    # the checker: the reference compiled from its own sources (here only —
    # /root/reference does not exist on the GPU box, which uses prebuilt files)
    ref = os.path.join(ROOT, "oracle", "_ref", "libmoe_ref.so")
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj"):
        import subprocess

        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle", "ref"], check=False)


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build(ref=False)
    return oracle.Oracle()


@pytest.fixture
def libopts():
    """Set library debug options (moe_debug_set_option) for one test; the
    previous values come back afterwards.  Usage: libopts(stack=0)."""
    import paper_2402_07033_b200 as M

    saved = {}

    def set_(**kw):
        for k, v in kw.items():
            if k not in saved:
                saved[k] = M.get_option(k)
            M.set_option(k, v)

    yield set_
    for k, v in saved.items():
        M.set_option(k, v)
