import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def refsolver():
    """The reference solver compiled in place (oracle/_ref); built here if the reference
    sources are present, otherwise the prebuilt library that travelled with the snapshot."""
    from oracle import ref
    if not ref.available():
        try:
            ref.build()
        except Exception as e:  # pragma: no cover
            pytest.skip(f"reference oracle unavailable: {e}")
    if not ref.available():
        pytest.skip("reference oracle library not built (oracle/_ref/libmmsim_ref.so)")
    return ref
