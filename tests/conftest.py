"""Shared test setup: markers, import paths, oracle build.

The oracle (``oracle/``) is the checker only; the product under test is the
native library loaded by ``paper_2602_08923_b200``.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")
    lib = os.path.join(ROOT, "oracle", "build", "libdqoracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)


def pytest_terminal_summary(terminalreporter):
    """Which native library the run loaded (DQ_LIB_VARIANT selects a build variant)."""
    mod = sys.modules.get("paper_2602_08923_b200._lib")
    if mod is None or getattr(mod, "_lib", None) is None:
        return
    try:
        flags = mod.lib().dq_build_flags()
        terminalreporter.write_line(f"dynamiq_b200 library: {mod.LIB_PATH} (build flags {flags:#x}; bit 0: device checks)")
    except Exception:
        pass


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref (the reference library) is not built here")
    return Oracle("reference")
