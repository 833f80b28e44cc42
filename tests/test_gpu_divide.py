"""Device self-checks of the arithmetic shortcuts inside the codec kernels.

* the shared-reciprocal division (dq_codec.cu div_rn) must equal IEEE div.rn.f32
  (the reference divides with x86 SSE divss, correctly rounded) on every input;
* the O(1) codebook bracket must equal lower_bound (proj/src/codebook.cpp:77-85);
* the decode's scale factor code * sg_scale / 255 (codec.cpp:146-149) through the fast
  reciprocal sequence must equal div.rn.f32 for every code and every bf16 sg_scale.
"""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_08923_b200._lib import lib
    return lib()


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_division_matches_ieee(L, seed):
    bad = C.c_uint64()
    from paper_2602_08923_b200._lib import check
    check(L.dq_selftest(0, 1 << 28, seed, C.byref(bad)))
    assert bad.value == 0, L.dq_last_error().decode()


@pytest.mark.parametrize("seed", [1, 2])
def test_bracket_matches_lower_bound(L, seed):
    bad = C.c_uint64()
    from paper_2602_08923_b200._lib import check
    check(L.dq_selftest(1, 1 << 26, seed, C.byref(bad)))
    assert bad.value == 0, L.dq_last_error().decode()


def test_div255_exhaustive(L):
    """all 256 codes x 65536 bf16 super-group scales (finite, positive)"""
    bad = C.c_uint64()
    from paper_2602_08923_b200._lib import check
    check(L.dq_selftest(2, 256 << 16, 0, C.byref(bad)))
    assert bad.value == 0, L.dq_last_error().decode()
