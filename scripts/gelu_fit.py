#!/usr/bin/env python3
"""Fit and check the branch-free erf used by the fused GELU epilogue (gelu2_fast,
paper_2603_28708_b200/csrc/common.cuh).

erfc(t) = 2^(-t^2 log2 e + P(t)), P = Chebyshev least-squares fit of log2(erfcx(t)) on
[0, 4.5] in the centred variable xc = t * 2/4.5 - 1 (monomial coefficients printed).
Then every finite binary16 input x is pushed through the GPU formula (fp32 ops
emulated, FMA fused) and through the reference formula 0.5f*x*(1+erff(x*0.70710678f))
(src/kernels.cpp:221-235) with a correctly rounded erff, and the fp16 outputs are
compared.  Needs scipy (this container); not used at run time."""
import numpy as np
from scipy.special import erf, erfcx

T = 4.5
DEG = 12


def fit():
    t = np.linspace(0, T, 400001)
    f = np.log2(erfcx(t))
    c = np.polynomial.chebyshev.Chebyshev.fit(t * (2 / T) - 1, f, DEG, domain=[-1, 1])
    return c.convert(kind=np.polynomial.Polynomial).coef.astype(np.float32)


def fma(a, b, c):
    return (a.astype(np.float64) * b + c).astype(np.float32)


def main():
    co = fit()
    print("coefficients (ascending):", [f"{v:.9e}" for v in co])
    f32 = np.float32
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16).view(np.float16)
    x = h.astype(np.float32)
    x = x[np.isfinite(x)]
    u = (x * f32(0.70710678118654752440)).astype(np.float32)
    t = np.minimum(np.abs(u), f32(T))
    xc = fma(t, np.float64(f32(2 / T)), np.float64(-1))
    acc = np.full_like(xc, co[-1])
    for a in co[-2::-1]:
        acc = fma(acc, xc, np.float64(a))
    e = fma((t * t).astype(np.float32), np.float64(f32(-1.4426950408889634)), acc)
    q = np.exp2(e.astype(np.float64)).astype(np.float32)
    a = (f32(1) - q).astype(np.float32)
    mine_erf = np.where(u < 0, -a, a).astype(np.float32)

    def gelu(er):
        return ((f32(0.5) * x).astype(np.float32) * (f32(1) + er).astype(np.float32)).astype(np.float32).astype(np.float16)

    mine = gelu(mine_erf)
    ref = gelu(erf(u.astype(np.float64)).astype(np.float32))
    d = mine != ref
    print(f"finite binary16 inputs {x.size}, fp16 GELU outputs differing from the reference formula: {int(d.sum())}")
    for i in np.where(d)[0]:
        print(f"  x={x[i]!r} fast={float(mine[i])!r} ref={float(ref[i])!r}")


if __name__ == "__main__":
    main()
