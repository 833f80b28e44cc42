"""The Fisher-Yates draw's r % k (k = 3, 5, 6) computed by 32-bit folds (mod_const in
csrc/dq_device.cuh): equal to the 64-bit remainder on edge cases and 10^7 random values.
Host-side: nvcc compiles a small host program against the same header (no GPU needed)."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r'''
#include <cstdio>
#include <random>
#include "dq_device.cuh"
int main() {
  std::mt19937_64 g(7);
  unsigned long long bad = 0;
  auto chk = [&](uint64_t r) {
    bad += dq::mod_const<3>(r) != r % 3;
    bad += dq::mod_const<5>(r) != r % 5;
    bad += dq::mod_const<6>(r) != r % 6;
    bad += dq::mod_const<4>(r) != r % 4;
    bad += dq::mod_const<7>(r) != r % 7;
  };
  const uint64_t edge[] = {0ull, 0xffffffffull, 0x100000000ull, 0x1ffffffffull, 0xffffffff00000000ull,
                           0xffffffffffffffffull, 0x8000000000000000ull, 0x7fffffffffffffffull};
  for (uint64_t e : edge)
    for (int d = -8; d <= 8; ++d) chk(e + static_cast<uint64_t>(d));
  for (long i = 0; i < 10000000; ++i) chk(g());
  std::printf("%llu\n", bad);
  return 0;
}
'''


def test_mod_fold_matches_64bit_remainder():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "m.cu")
        exe = os.path.join(d, "m")
        open(src, "w").write(SRC)
        inc = os.path.join(ROOT, "paper_2602_08923_b200", "csrc")
        subprocess.run([nvcc, "-std=c++17", "-O2", "-I", inc, "-o", exe, src], check=True, capture_output=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.strip()
    assert out == "0"
