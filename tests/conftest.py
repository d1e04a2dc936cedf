import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running case")


import pytest  # noqa: E402


@pytest.fixture
def lsw_opts():
    """Set liblsw variant options (include/lsw_debug.h) for the ctxs a test
    creates: ``lsw_opts(tc_kernel="pt", tc_grid=3)``; cleared afterwards."""
    from paper_2405_17741_b200 import binding
    used = []

    def set_(**kv):
        for k, v in kv.items():
            if v is not None:
                binding.set_option(k, v)
                used.append(k)
    yield set_
    binding.set_option(None)
