import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_report_header(config):
    """The build under test: psg_version() carries the hash of the sources libpsg.so was built from."""
    try:
        import paper_0912_3678_b200 as psg
        return "libpsg: " + psg.lib().psg_version().decode()
    except Exception as e:  # the CPU suite still runs without the library
        return f"libpsg: not loaded ({e})"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    return torch


# Achieved parity values of the -m gpu run, merged into profiles/r02_parity.json
# (and gpurun_out/) as they are recorded.
def record_parity(key, values):
    import json
    for d in (os.path.join(ROOT, "profiles"), os.path.join(ROOT, "gpurun_out")):
        os.makedirs(d, exist_ok=True)
        path = os.path.join(d, "r02_parity.json")
        old = {}
        if os.path.exists(path):
            try:
                old = json.load(open(path))
            except Exception:
                old = {}
        old[key] = values
        with open(path, "w") as fh:
            json.dump(old, fh, indent=1, sort_keys=True)
