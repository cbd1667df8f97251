"""CPU proofs of the exact-division shortcuts used by the integration kernel
(paper_1410_0925_b200/csrc/vf_integrate.cu): with y = RN(1/b), the quotient
q = RN(a*y) corrected once, RN(q + RN(a - b*q)*y), equals the IEEE quotient
RN(a/b) for every operand the kernel feeds it:

* sdf_value_to_float (voxel.hpp:11): a = every int16, b = 32767;
* the colour blend (integration.hpp:94-97): a = clr*w + sample, an integer in
  [0, 255*255 + 255], b = w + 1 in [1, 256].

Exhaustive, in C with fmaf (gcc, -ffp-contract=off)."""
import shutil
import subprocess

import pytest

SRC = r"""
#include <math.h>
#include <stdio.h>
static float div_rr(float a, float b, float rb) {
  const float q = a * rb;
  const float r = fmaf(-b, q, a);
  return fmaf(r, rb, q);
}
int main(void) {
  long bad = 0, n = 0;
  volatile float b32767 = 32767.0f;
  const float r32767 = 1.0f / b32767;
  for (int v = -32768; v <= 32767; ++v, ++n)
    if (div_rr((float)v, b32767, r32767) != (float)v / b32767) ++bad;
  for (int w = 0; w < 256; ++w) {
    volatile float den = (float)(w + 1);
    const float rd = 1.0f / den;
    for (int a = 0; a <= 255 * 255 + 255; ++a, ++n)
      if (div_rr((float)a, den, rd) != (float)a / den) ++bad;
  }
  printf("%ld %ld\n", n, bad);
  return 0;
}
"""


def test_refined_quotients_are_exact(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    c = tmp_path / "divid.c"
    c.write_text(SRC)
    exe = tmp_path / "divid"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), str(c), "-lm"], check=True)
    n, bad = map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split())
    assert n == 65536 + 256 * (255 * 255 + 256)
    assert bad == 0
