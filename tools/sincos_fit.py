"""Fit and validate the fp32 polynomials of sincos_2pi_u24 (csrc/vndf_device.cuh).

The config-4 azimuth is phi = 2 pi k 2^-24 for a 24-bit integer k.  The kernel
reduces it EXACTLY with integer arithmetic to phi = q pi/2 + theta, theta =
r 2 pi 2^-24, r in [-2^21, 2^21) (|theta| <= pi/4), then evaluates
    sin(theta) = theta + theta x (s1 + x (s2 + x s3)),        x = theta^2
    cos(theta) = 1 + x (c1 + x (c2 + x (c3 + x c4)))
in fp32 with fused multiply-adds.  This script fits the coefficients
(least squares on Chebyshev nodes for the RELATIVE error, iterated with
Lawson-style reweighting towards minimax), rounds them to fp32, and then
evaluates the kernel's exact fp32 operation sequence on EVERY one of the 2^22
reduced arguments (numpy, fma emulated as one rounding of the exact float64
result), reporting the worst error in units of the result's ulp.

    python tools/sincos_fit.py
"""
import numpy as np

F = np.float32


def fma32(a, b, c):
    # a*b is exact in float64 for fp32 inputs; the sum rounds once in float64
    # (<= 2^-53 relative) before the fp32 rounding: a faithful emulation
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(F)


def mul32(a, b):
    return (a.astype(np.float64) * b.astype(np.float64)).astype(F)


def fit(kind, deg, iters=30):
    t = np.cos(np.linspace(0, np.pi, 4001)) * 0.5 + 0.5   # Chebyshev-ish nodes on [0, 1]
    th = t * (np.pi / 4)
    x = th * th
    if kind == "sin":
        target = np.where(th > 0, np.sin(th) / np.where(th > 0, th, 1) - 1.0, 0.0)  # s1 x + s2 x^2 + ...
        scale = np.ones_like(th)
        A = np.stack([x ** (j + 1) for j in range(deg)], axis=1)
    else:
        target = np.cos(th) - 1.0
        scale = 1.0 / np.cos(th)          # relative error of cos
        A = np.stack([x ** (j + 1) for j in range(deg)], axis=1)
    w = np.ones_like(th)
    for _ in range(iters):
        W = (w * scale)[:, None]
        coef, *_ = np.linalg.lstsq(A * W, target * W[:, 0], rcond=None)
        err = np.abs((A @ coef - target) * scale)
        w = w * (err / err.max() + 1e-3) ** 0.5
        w /= w.max()
    return coef


def evaluate(s, c):
    r = np.arange(-(1 << 21), 1 << 21, dtype=np.int64)
    th = mul32((r * 1024).astype(np.int32).astype(F), np.array(2 * np.pi * 2.0**-34, dtype=F))
    x = mul32(th, th)
    p = fma32(x, np.full_like(th, s[2]), np.full_like(th, s[1]))
    p = fma32(x, p, np.full_like(th, s[0]))
    sn = fma32(mul32(th, x), p, th)
    q = fma32(x, np.full_like(th, c[3]), np.full_like(th, c[2]))
    q = fma32(x, q, np.full_like(th, c[1]))
    q = fma32(x, q, np.full_like(th, c[0]))
    cs = fma32(x, q, np.ones_like(th))
    exact = 2 * np.pi * r.astype(np.float64) * 2.0**-24
    es, ec = np.sin(exact), np.cos(exact)
    ulp = lambda v: np.spacing(np.abs(v).astype(F)).astype(np.float64)
    nz = r != 0
    err_s = np.abs(sn.astype(np.float64) - es)[nz] / ulp(es)[nz]
    err_c = np.abs(cs.astype(np.float64) - ec) / ulp(ec)
    rel_s = (np.abs(sn.astype(np.float64) - es)[nz] / np.abs(es[nz])).max()
    rel_c = (np.abs(cs.astype(np.float64) - ec) / np.abs(ec)).max()
    return err_s.max(), err_c.max(), rel_s, rel_c, (sn[~nz] == 0).all()


def main():
    s = fit("sin", 3).astype(F)
    c = fit("cos", 4).astype(F)
    es, ec, rs, rc, zero_ok = evaluate(s, c)
    print("sin coefficients (s1, s2, s3):", ", ".join(f"{v:.9e}f" for v in s))
    print("cos coefficients (c1, c2, c3, c4):", ", ".join(f"{v:.9e}f" for v in c))
    print(f"over all 2^22 reduced arguments: sin max {es:.3f} ulp (rel {rs:.3e}), "
          f"cos max {ec:.3f} ulp (rel {rc:.3e}); sin(0) == 0: {zero_ok}")


if __name__ == "__main__":
    main()
