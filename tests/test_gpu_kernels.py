"""GPU: numerical building blocks of the kernels."""
import pytest

from paper_1410_0925_b200 import _abi

pytestmark = pytest.mark.gpu


def test_branch_free_division_matches_ieee_for_constant_divisors():
    """div_rr (integration's division) == IEEE a / b for a = 0 and every float
    numerator with 2^-60 <= |a| <= 256 -- the operand domain: eta = d - z is 0
    or at least ulp(0.1) ~ 7e-9, the blend numerator is a sum of such terms --
    for every divisor the kernel divides by a constant: the truncation bands
    mu of the configs and every weight count 1..256."""
    L = _abi.load()
    lo = 2.0 ** -60
    for mu in (0.02, 0.06, 0.03, 0.004, 0.005):
        assert L.vf_selftest_division(0, 0, mu, 16.0, lo, 0) == 0, f"mu={mu}"
    for w in range(1, 257):
        assert L.vf_selftest_division(0, 0, float(w), 256.0, lo, 0) == 0, f"w={w}"


def test_branch_free_division_matches_ieee_projection_range():
    """The projection divides fx * x by z: 2^30 random pairs, |a| <= 1e5,
    1e-3 <= |z| <= 64."""
    L = _abi.load()
    assert L.vf_selftest_division(0, 1, 1e5, 1e-3, 64.0, 1 << 30) == 0
