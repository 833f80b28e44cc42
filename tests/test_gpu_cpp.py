"""Build and run tests/cpp/test_dropin.cpp: the reference-style C++ tests against the
drop-in header include/dynamiq_b200.hpp (C++20, links libdynamiq_b200.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_dropin_test() -> str:
    out = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    lib = os.path.join(ROOT, "paper_2602_08923_b200")
    orc = os.path.join(ROOT, "oracle", "build")
    cmd = ["g++", "-std=c++20", "-O2", os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-o", out,
           "-I/usr/local/cuda/include", f"-L{lib}", "-ldynamiq_b200", f"-L{orc}", "-ldqoracle",
           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}:{orc}:/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return out


def test_dropin_header_compiles():
    """C++ compile check of the header + test (no GPU needed to build)."""
    assert os.path.exists(build_dropin_test())


@pytest.mark.gpu
def test_dropin_reference_style_suite():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = build_dropin_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
