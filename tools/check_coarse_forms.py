"""Brute-force equivalence checks behind three integer-arithmetic rewrites in sph_wide.cu (Python
mirrors of the device code; run: python tools/check_coarse_forms.py, ~1 min):
  coarse_range  -- the closed form against the original loop "cells from the one holding a, while
                   coarse_meets", every n < 70, F <= n, k <= n, a in [-2n, 2n);
  coarse_meets  -- two conditional corrections against ((f0 - a) % n + n) % n over its callers' range
                   a = c - k, c in [0, n), k <= (n - 1) / 2 + 1;
  div_small     -- f32 quotient (+-3e-7 relative error) with the +-1 correction against x // F."""
import numpy as np


def meets(ci, a, k, n, F, fast=False):
    f0 = ci * F
    w = min(F, n - f0)
    if 2 * k + 1 >= n:
        return True
    if fast:
        d0 = f0 - a
        d0 += n if d0 < 0 else 0
        d0 -= n if d0 >= n else 0
    else:
        d0 = ((f0 - a) % n + n) % n
    return d0 <= 2 * k or d0 + w > n


def range_loop(a, k, n, F, cn):
    am = ((a % n) + n) % n
    c0 = 0 if 2 * k + 1 >= n else am // F
    cnt, ci = 0, c0
    while cnt < cn and meets(ci, a, k, n, F):
        cnt += 1
        ci = 0 if ci + 1 == cn else ci + 1
    return c0, cnt


def range_closed(a, k, n, F, cn):
    if 2 * k + 1 >= n:
        return 0, cn
    am = a % n
    e = am + 2 * k
    c0 = am // F
    return c0, (e // F - c0 + 1 if e < n else min(cn - c0 + (e - n) // F + 1, cn))


def main():
    bad = tot = 0
    for n in range(3, 70):
        for F in range(1, n + 1):
            cn = (n + F - 1) // F
            for k in range(0, n + 1):
                for a in range(-2 * n, 2 * n):
                    tot += 1
                    bad += range_loop(a, k, n, F, cn) != range_closed(a, k, n, F, cn)
    print(f"coarse_range: {tot} cases, {bad} mismatches")
    bad = tot = 0
    for n in range(3, 60):
        for F in range(1, n + 1):
            for k in range(0, (n - 1) // 2 + 2):
                for c in range(n):
                    for ci in range((n + F - 1) // F):
                        tot += 1
                        bad += meets(ci, c - k, k, n, F) != meets(ci, c - k, k, n, F, fast=True)
    print(f"coarse_meets: {tot} cases, {bad} mismatches")
    bad = 0
    x = np.arange(0, 4096, dtype=np.int64)
    for F in range(1, 1025):
        for eps in (-3e-7, 0.0, 3e-7):
            q = np.trunc((x.astype(np.float32) / np.float32(F)) * np.float32(1 + eps)).astype(np.int64)
            q += (q + 1) * F <= x
            q -= q * F > x
            bad += int((q != x // F).sum())
    print(f"div_small: {4096 * 1024 * 3} cases, {bad} mismatches")


if __name__ == "__main__":
    main()
