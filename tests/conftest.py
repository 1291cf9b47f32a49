import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build libmb4cu.so and the oracle checkers once (no-op when up to date)."""
    from paper_2003_04345_b200 import _build

    if os.environ.get("MB4_SKIP_BUILD") != "1":
        try:
            _build.build_lib()
        except Exception as exc:  # nvcc absent on a box: use the prebuilt library
            if not os.path.exists(os.path.join(ROOT, "paper_2003_04345_b200", "libmb4cu.so")):
                raise exc
        if os.path.exists("/root/reference") or not os.path.exists(
                os.path.join(ROOT, "oracle", "liboracle.so")):
            _build.build_oracle()
    yield
