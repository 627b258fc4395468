"""Chebyshev-economised series tables of problems.cuh (econ_trig / econ_exp).

For each (N, r): start from the Taylor series of degree N + extra and remove
the top terms one at a time through T_m(z / r) on [-r, r] (telescoping
economisation), leaving degree N.  The shipped tables (no arguments) use
extra = 1, except trig N = 5 and N = 6 with extra = 2.  Trig: the even coefficients come from
cos z, the odd ones from sin z (sin(t0 + z) = sin t0 cos z + cos t0 sin z and
cos(t0 + z) likewise, so one table of magnitudes serves both with the signs
of the derivative cycle); exp: e^z.  Prints the C++ hex tables and the max
absolute error on [-r, r] for unit amplitude (relative for exp), measured at
4001 points with 50-digit mpmath arithmetic on the coefficients as rounded
to double.

usage: python tools/econ_tables.py [--extra=K] [N:r ...]   (default: the shipped classes)
"""
import sys

import mpmath as mp

mp.mp.dps = 60


def cheb_T(m):
    """Coefficients (ascending) of the Chebyshev polynomial T_m."""
    a, b = [mp.mpf(1)], [mp.mpf(0), mp.mpf(1)]
    if m == 0:
        return a
    for _ in range(m - 1):
        c = [mp.mpf(0)] + [2 * x for x in b]
        for i, x in enumerate(a):
            c[i] -= x
        a, b = b, c
    return b


def economise(coef, n, r):
    c = list(coef)
    for m in range(len(c) - 1, n, -1):
        if c[m] == 0:
            continue
        t = cheb_T(m)  # leading coefficient 2^(m-1)
        k = c[m] * r ** m / t[m]  # c_m z^m - k T_m(z / r) has degree < m
        for i in range(m + 1):
            c[i] -= k * t[i] / r ** i
        c[m] = mp.mpf(0)
    return c[: n + 1]


def taylor(kind, m):
    out = []
    for i in range(m + 1):
        f = mp.factorial(i)
        if kind == "exp":
            out.append(1 / f)
        elif kind == "cos":
            out.append(((-1) ** (i // 2)) / f if i % 2 == 0 else mp.mpf(0))
        else:
            out.append(((-1) ** (i // 2)) / f if i % 2 == 1 else mp.mpf(0))
    return out


def to_double(x):
    return float(x)


def poly(c, z):
    s = mp.mpf(0)
    for x in reversed(c):
        s = s * z + x
    return s


def table(n, r, extra=1, extra_exp=None):
    r = mp.mpf(r)
    ec = economise(taylor("cos", n + extra), n, r)
    es = economise(taylor("sin", n + extra), n, r)
    ee = economise(taylor("exp", n + (extra if extra_exp is None else extra_exp)), n, r)
    trig = [abs(ec[i]) if i % 2 == 0 else abs(es[i]) for i in range(n + 1)]
    trig_d = [to_double(x) for x in trig]
    exp_d = [to_double(x) for x in ee]
    err = {"cos": 0, "sin": 0, "exp": 0}
    for j in range(4001):
        z = r * (mp.mpf(j) / 2000 - 1)
        pc = poly([(-1) ** (i // 2) * mp.mpf(trig_d[i]) if i % 2 == 0 else 0 for i in range(n + 1)], z)
        ps = poly([(-1) ** (i // 2) * mp.mpf(trig_d[i]) if i % 2 == 1 else 0 for i in range(n + 1)], z)
        pe = poly([mp.mpf(x) for x in exp_d], z)
        err["cos"] = max(err["cos"], abs(pc - mp.cos(z)))
        err["sin"] = max(err["sin"], abs(ps - mp.sin(z)))
        err["exp"] = max(err["exp"], abs(pe - mp.exp(z)) / mp.exp(z))
    return trig_d, exp_d, err


def main():
    args = sys.argv[1:]
    extra = None
    if args and args[0].startswith("--extra="):
        extra = int(args.pop(0).split("=")[1])
    # the shipped classes: (N, r, trig extra, exp extra)
    specs = [(int(n), r, extra or 1, extra or 1) for n, r in (a.split(":") for a in args)] or [
        (5, "0.0125", 2, 1), (6, "0.028", 2, 1), (7, "0.05", 1, 1), (9, "0.12", 1, 1)]
    for n, r, xt, xe in specs:
        trig, ex, err = table(n, r, xt, xe)
        print(f"// N = {n}, |z| <= {r}: cos {float(err['cos']):.1e}, sin {float(err['sin']):.1e}, "
              f"exp {float(err['exp']):.1e}")
        print("trig", ", ".join(x.hex() for x in trig))
        print("exp ", ", ".join(x.hex() for x in ex))


if __name__ == "__main__":
    main()
