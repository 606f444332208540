"""Derive the fp32 arithmetic-contract polynomial coefficients.

Offline tool: run once, its printed hex-float constants are typed into the
contract table of DESIGN.md and, independently, into oracle/contract32.c and
paper_2305_05286_b200/csrc/contract.cuh.  Neither side imports this file.

Method: weighted least squares (relative error) on Chebyshev nodes in
50-digit mpmath, then coefficients rounded to binary32 highest-degree first,
re-fitting the lower ones after each rounding.
"""
import sys
import mpmath as mp
import numpy as np

mp.mp.dps = 50


def fit(fun, lo, hi, deg, nodes=600, fixed=None):
    xs = [mp.mpf(lo) + (mp.mpf(hi) - mp.mpf(lo)) * (1 - mp.cos(mp.pi * (k + 0.5) / nodes)) / 2
          for k in range(nodes)]
    ys = [fun(x) for x in xs]
    fixed = dict(fixed or {})
    free = [k for k in range(deg + 1) if k not in fixed]
    if not free:
        return [fixed[k] for k in range(deg + 1)], xs, ys
    A = mp.matrix(nodes, len(free))
    b = mp.matrix(nodes, 1)
    for r, (x, y) in enumerate(zip(xs, ys)):
        w = 1 / abs(y)
        rhs = y - sum(c * x ** k for k, c in fixed.items())
        for ci, k in enumerate(free):
            A[r, ci] = w * x ** k
        b[r] = w * rhs
    sol = mp.lu_solve(A.T * A, A.T * b)
    coef = dict(fixed)
    for ci, k in enumerate(free):
        coef[k] = sol[ci]
    return [coef[k] for k in range(deg + 1)], xs, ys


def fit_f32(fun, lo, hi, deg, fixed_exact=None):
    fixed = dict(fixed_exact or {})
    for k in range(deg, -1, -1):
        if k in fixed:
            continue
        c, _, _ = fit(fun, lo, hi, deg, fixed=fixed)
        fixed[k] = mp.mpf(float(np.float32(float(c[k]))))
    c, xs, ys = fit(fun, lo, hi, deg, fixed=fixed)
    err = max(abs((sum(ck * x ** k for k, ck in enumerate(c)) - y) / y) for x, y in zip(xs, ys))
    return [float(np.float32(float(ck))) for ck in c], float(err)


def show(name, coefs, err):
    print(f"{name}: max rel err (exact eval, f32 coefs) = {err:.3e}")
    for k, ck in enumerate(coefs):
        print(f"   c{k} = {float(ck).hex():>24s}  /* {ck:.9e} */")


XA = 1.0
targets = {
    # ln(1+f) = f + f^2 * P(f)
    "P_ln": (lambda f: (mp.log1p(f) - f) / f ** 2 if f != 0 else mp.mpf(-0.5),
             float(mp.sqrt(2) / 2 - 1) - 1e-4, float(mp.sqrt(2) - 1) + 1e-4),
    # g(y)/y, g(y) = ln((sqrt(y)/2) coth(sqrt(y)/2))
    "G_A": (lambda y: mp.log((mp.sqrt(y) / 2) * mp.coth(mp.sqrt(y) / 2)) / y if y != 0 else mp.mpf(1) / 12,
            0.0, XA * XA),
    # exp(-r)
    "E_exp": (lambda r: mp.exp(-r), -0.3480, 0.3480),
    # atanh(sqrt(w))/sqrt(w)
    "H_B": (lambda w: mp.atanh(mp.sqrt(w)) / mp.sqrt(w) if w != 0 else mp.mpf(1),
            0.0, float(mp.exp(-2 * XA)) * 1.0001),
    # sin(pi/2 sqrt(z))/sqrt(z), cos(pi/2 sqrt(z))  (Box-Muller)
    "S_sin": (lambda z: mp.sin(mp.pi / 2 * mp.sqrt(z)) / mp.sqrt(z) if z != 0 else mp.pi / 2, 0.0, 0.25),
    "C_cos": (lambda z: mp.cos(mp.pi / 2 * mp.sqrt(z)), 0.0, 0.25),
}

if __name__ == "__main__":
    degs = dict(a.split("=") for a in sys.argv[1:])
    for name, (fun, lo, hi) in targets.items():
        if name not in degs:
            continue
        fixed = {0: mp.mpf(1)} if name in ("E_exp", "H_B", "C_cos") else None
        c, e = fit_f32(fun, lo, hi, int(degs[name]), fixed)
        show(name, c, e)
