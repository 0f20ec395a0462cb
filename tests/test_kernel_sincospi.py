"""Host-side checks of the kernel's table-driven sin/cos(pi x) (paper_2412_11614_b200/csrc/kernels.cu,
`sincospi_d`, ISRS_CISTAB): the 256-entry table in csrc/cis_table.h and the reduction + polynomial
constants are read from the CUDA sources themselves and checked against the mathematics (no GPU):

* table: quarter points exact, the quarter-turn symmetry cos(pi(j+64)/128) = -sin(pi j/128) exact,
  every entry within 1 ulp of x87 long-double cos/sin, |T|^2 = 1 within 2 ulp;
* formula: the kernel's steps (rounding constant, exact reduction, degree-6 polynomials, complex
  product with the table entry) replayed with libm's fused multiply-add agree with x87 long-double
  sin/cos(pi x) within 2.5e-16 over |x| up to 3e4 (the largest chi h / pi of c5).
The kernel path itself is checked against the oracle by the GPU parity tests and the cistab_* kernel
mutants (tests/tools/kernel_mutants.py)."""
import ctypes
import ctypes.util
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2412_11614_b200", "csrc")
PI = np.longdouble("3.14159265358979323846264338327950288419716939937510")


def table():
    src = open(os.path.join(CSRC, "cis_table.h")).read()
    rows = re.findall(r"\{(\S+), (\S+)\},\s+// j = (\d+)", src)
    assert [int(r[2]) for r in rows] == list(range(256))
    return np.array([[float.fromhex(c), float.fromhex(s)] for c, s, _ in rows])


def kernel_block():
    src = open(os.path.join(CSRC, "kernels.cu")).read()
    m = re.search(r"#if ISRS_CISTAB(.*?)#else", src, re.S)
    assert m, "table-driven sincospi block not found in kernels.cu"
    return "\n".join(line.split("//")[0] for line in m.group(1).splitlines())   # code only


def test_table_entries():
    t = table()
    assert tuple(t[0]) == (1.0, 0.0) and tuple(t[64]) == (0.0, 1.0)
    assert tuple(t[128]) == (-1.0, 0.0) and tuple(t[192]) == (0.0, -1.0)
    j = np.arange(256)
    # cos(a + pi/2) = -sin(a), sin(a + pi/2) = cos(a): the same real numbers, so the same doubles
    np.testing.assert_array_equal(t[(j + 64) % 256, 0], -t[j, 1])
    np.testing.assert_array_equal(t[(j + 64) % 256, 1], t[j, 0])
    a = PI * j.astype(np.longdouble) / np.longdouble(128)
    ref = np.stack([np.cos(a), np.sin(a)], axis=1)
    # (the exact zeros of the quarter points against long double cos/sin at multiples of pi/2, |.| < 2e-19)
    ulp = np.maximum(np.spacing(np.abs(t)), 1e-18)
    assert np.all(np.abs(t.astype(np.longdouble) - ref) <= 0.5 * ulp)    # correctly rounded
    assert np.max(np.abs(t[:, 0] ** 2 + t[:, 1] ** 2 - 1.0)) <= 4.5e-16


def test_formula_matches_long_double():
    blk = kernel_block()
    nums = [float(x) for x in re.findall(r"-?\d+\.\d+(?:e[-+]?\d+)?", blk)]
    # order in the source: M, 128, -1/128, then sin coefficients (3 in Horner order + pi), cos (3)
    M, s7, s5, s3, s1, c6, c4, c2 = (nums[0], nums[3], nums[4], nums[5], nums[6], nums[7], nums[8],
                                     nums[9])
    assert M == 1.5 * 2 ** 52 and nums[1] == 128.0 and nums[2] == -0.0078125
    p = PI
    for got, want in ((s1, p), (s3, -p ** 3 / 6), (s5, p ** 5 / 120), (s7, -p ** 7 / 5040),
                      (c2, -p ** 2 / 2), (c4, p ** 4 / 24), (c6, -p ** 6 / 720)):
        assert abs(np.longdouble(got) - want) <= abs(want) * 1.2e-16
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.fma.restype = ctypes.c_double
    libm.fma.argtypes = [ctypes.c_double] * 3
    fma = libm.fma
    t = table()
    rng = np.random.default_rng(20241211)
    xs = np.concatenate([rng.uniform(-1, 1, 3000), rng.uniform(-3e4, 3e4, 3000),
                         rng.uniform(-1e-3, 1e-3, 500), np.arange(-4, 4.01, 1 / 256)])
    worst = 0.0
    for x in xs:
        x = float(x)
        tt = fma(x, 128.0, M)
        r = fma(tt - M, -0.0078125, x)
        n = int(np.float64(tt).view(np.int64)) & 255
        ex, ey = t[n]
        r2 = r * r
        ps = fma(fma(fma(r2, s7, s5), r2, s3), r2, s1)
        s = r * ps
        cm1 = fma(fma(r2, c6, c4), r2, c2) * r2
        c = fma(ex, cm1, fma(-ey, s, ex))
        sn = fma(ey, cm1, fma(ex, s, ey))
        xr = np.fmod(np.longdouble(x), np.longdouble(2))          # exact
        err = max(abs(np.longdouble(c) - np.cos(PI * xr)), abs(np.longdouble(sn) - np.sin(PI * xr)))
        worst = max(worst, float(err))
    assert worst <= 2.5e-16, worst
