"""Test configuration: the `gpu` marker (parity tests on a B200) and import
paths for the package and the oracle (test infrastructure)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels through the C-ABI)")


@pytest.fixture(scope="session")
def handle():
    import paper_2603_21379_b200 as P

    return P.default_handle()


@pytest.fixture(scope="session")
def O():
    import srtt_oracle

    return srtt_oracle
