"""Near-minimax polynomials for sin(pi r), cos(pi r) on |r| <= 1/4
(weighted least squares on Chebyshev nodes in mpmath, refined with a few
Lawson iterations), and the max error of their double-precision Horner/FMA
evaluation.  Used to size hk_math.cuh's generator sincospi."""
import sys

import mpmath as mp
import numpy as np

mp.mp.dps = 50


def fit(fn, parity, nterms, a=mp.mpf(0), b=mp.mpf(1) / 4, npts=400, iters=30):
    xs = [(a + b) / 2 + (b - a) / 2 * mp.cos(mp.pi * (2 * i + 1) / (2 * npts)) for i in range(npts)]
    w = [mp.mpf(1)] * npts
    pw = [2 * k + parity for k in range(nterms)]
    coef = None
    for _ in range(iters):
        A = mp.matrix(npts, nterms)
        y = mp.matrix(npts, 1)
        for i, x in enumerate(xs):
            sw = mp.sqrt(w[i])
            for k, p in enumerate(pw):
                A[i, k] = sw * x ** p
            y[i] = sw * fn(x)
        coef = mp.lu_solve(A.T * A, A.T * y)
        err = [abs(fn(x) - sum(coef[k] * x ** p for k, p in enumerate(pw))) for x in xs]
        tot = sum(wi * ei for wi, ei in zip(w, err))
        w = [wi * ei / tot for wi, ei in zip(w, err)]
    return [coef[k] for k in range(nterms)]


def eval_double(c, parity, r):
    r2 = r * r
    p = np.full_like(r, float(c[-1]))
    for k in range(len(c) - 2, -1, -1):
        p = np.fma(p, r2, float(c[k])) if hasattr(np, "fma") else p * r2 + float(c[k])
    return r * p if parity == 1 else p


def main():
    rs = np.linspace(-0.25, 0.25, 400001)
    ref_s = np.array([float(mp.sin(mp.pi * mp.mpf(float(x)))) for x in rs[::50]])
    ref_c = np.array([float(mp.cos(mp.pi * mp.mpf(float(x)))) for x in rs[::50]])
    for ns in range(5, 10):
        c = fit(lambda x: mp.sin(mp.pi * x), 1, ns)
        e = np.max(np.abs(eval_double(c, 1, rs[::50]) - ref_s))
        print(f"sin terms {ns} (degree {2 * ns - 1}): max abs err {e:.3g}")
    for nc in range(5, 11):
        c = fit(lambda x: mp.cos(mp.pi * x), 0, nc)
        e = np.max(np.abs(eval_double(c, 0, rs[::50]) - ref_c))
        print(f"cos terms {nc} (degree {2 * nc - 2}): max abs err {e:.3g}")
    if len(sys.argv) > 2:
        ns, nc = int(sys.argv[1]), int(sys.argv[2])
        cs = fit(lambda x: mp.sin(mp.pi * x), 1, ns)
        cc = fit(lambda x: mp.cos(mp.pi * x), 0, nc)
        print("sin", [mp.nstr(v, 20) for v in cs])
        print("sin_hex", [float(v).hex() for v in cs])
        print("cos_hex", [float(v).hex() for v in cc])


if __name__ == "__main__":
    main()


def fit_exp(nterms: int):
    """exp(r) on |r| <= ln2/2 as sum c_k r^k (near-minimax), for the FCN's
    factored density (hk_fcn.cu fcn_exp_neg)."""
    half = mp.log(2) / 2
    xs = [half * mp.cos(mp.pi * (2 * i + 1) / 800) for i in range(400)]
    w = [mp.mpf(1)] * len(xs)
    for _ in range(30):
        A = mp.matrix(len(xs), nterms)
        y = mp.matrix(len(xs), 1)
        for i, x in enumerate(xs):
            sw = mp.sqrt(w[i])
            for k in range(nterms):
                A[i, k] = sw * x ** k
            y[i] = sw * mp.exp(x)
        c = mp.lu_solve(A.T * A, A.T * y)
        err = [abs(mp.exp(x) - sum(c[k] * x ** k for k in range(nterms))) / mp.exp(x) for x in xs]
        tot = sum(wi * ei for wi, ei in zip(w, err))
        w = [wi * ei / tot for wi, ei in zip(w, err)]
    return [c[k] for k in range(nterms)], max(err)
