import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)



def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; runs the CUDA path")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_sessionstart(session):
    # Build the native artefacts in-tree (idempotent; nvcc cross-compiles without a GPU).
    import __graft_entry__

    lib = __graft_entry__._load_file("_nsg_build_lib", os.path.join(ROOT, "paper_2509_03653_b200", "_lib.py"))
    lib.build_libnsg()
    lib.build_libnsg(debug=True)  # -DNSG_DEBUG_CHECKS variant (tests of the NSG_ERR_INTERNAL readback)
    import gen
    import oracle

    gen.build()
    oracle.build()


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device (the CUDA path has no CPU fallback)")
    return torch.device("cuda", 0)
