import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_workload():
    lib = os.path.join(ROOT, "workload", "_lib", "libpsattn_synth_host.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "workload")], check=True, stdout=subprocess.DEVNULL)


_ensure_workload()


def _ensure_oracle():
    so = os.path.join(ROOT, "oracle", "build", "libpsa_oracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                       stdout=subprocess.DEVNULL)
    return so


@pytest.fixture(scope="session")
def oracle():
    _ensure_oracle()
    from oracle.pyoracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import RefDriver, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefDriver()
