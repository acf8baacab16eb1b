"""Fit the tcgen05 kind::f16 accumulation to the raw results of tools/f16acc_micro
(gpurun_out/f16acc*.bin): which alignment / truncation model reproduces every fp32 result.
Exact integer arithmetic in units of 2^-160."""
import sys
from fractions import Fraction

import numpy as np

M, N, KT = 128, 64, 64
U = 160  # value = int * 2^-U


def load(path):
    raw = open(path, "rb").read()
    a = np.frombuffer(raw[: M * KT * 2], dtype=np.float16).astype(np.float64).reshape(M, KT)
    b = np.frombuffer(raw[M * KT * 2: (M + N) * KT * 2], dtype=np.float16).astype(np.float64).reshape(N, KT)
    d = np.frombuffer(raw[(M + N) * KT * 2:], dtype=np.float32).reshape(M, N)
    return a, b, d


def to_int(x):  # exact double -> int units
    return int(Fraction(float(x)) * (1 << U))


def rz24(v):  # truncate an integer-unit value to a 24-bit significand (fp32, toward zero)
    if v == 0:
        return 0
    s = -1 if v < 0 else 1
    a = abs(v)
    n = a.bit_length()
    if n > 24:
        a = (a >> (n - 24)) << (n - 24)
    return s * a


def trunc_to(v, lsb_exp):  # truncate toward zero to a multiple of 2^lsb_exp (units)
    q = 1 << max(lsb_exp, 0)
    if lsb_exp <= 0:
        return v
    return (abs(v) // q) * q * (1 if v >= 0 else -1)


def model(prods, acc, F, acc_in_align=True, group=16):
    """prods: 16 ints; acc: int.  Addends aligned to the largest one's leading bit
    (of the group, then of the group sums and acc), truncated F bits below it."""
    def align_sum(vals):
        nz = [abs(v) for v in vals if v]
        if not nz:
            return 0
        top = max(nz).bit_length()  # leading bit position + 1
        lsb = top - F
        return sum(trunc_to(v, lsb) for v in vals)
    if group == 16:
        vals = list(prods) + ([acc] if acc_in_align else [])
        s = align_sum(vals)
        if not acc_in_align:
            s = s + acc
        return rz24(s)
    parts = [align_sum(prods[g:g + group]) for g in range(0, 16, group)]
    vals = parts + ([acc] if acc_in_align else [])
    s = align_sum(vals)
    if not acc_in_align:
        s += acc
    return rz24(s)


def main(paths):
    cases = []
    for path in paths:
        a, b, d = load(path)
        for r in range(8, M):
            for c in range(N):
                pr = [to_int(a[r, k] * b[c, k]) for k in range(KT)]
                cases.append((pr, to_int(float(d[r, c]))))
    print(f"{len(cases)} random dot products from {len(paths)} dumps")
    for group in (16, 8, 4, 2):
        for acc_in in (True, False):
            for F in range(23, 34):
                ok = 0
                for pr, got in cases:
                    acc = 0
                    for kk in range(4):
                        acc = model(pr[16 * kk: 16 * kk + 16], acc, F, acc_in, group)
                    ok += acc == got
                if ok > 0.9 * len(cases) or F in (24, 26, 28):
                    print(f"group {group:2d} acc_in_align {acc_in!s:5} F {F}: {ok}/{len(cases)}")


if __name__ == "__main__":
    main(sys.argv[1:] or ["gpurun_out/f16acc.bin"])
