"""Test helpers: build oracle instances of the seeded workloads, exact polynomial
integrals on the reference triangle, parity norms (reading A23)."""
from __future__ import annotations

from fractions import Fraction
from math import comb, factorial

import numpy as np

import oracle
import swe_inputs as si


def make_oracle(w: si.Workload, **over):
    """Oracle for workload w, with B and the initial state sampled at the oracle's nodes."""
    prm = dict(w.params)
    prm.update(over)
    m = w.mesh
    Np = (w.N + 1) * (w.N + 2) // 2
    probe = oracle.Oracle(m.vx, m.vy, m.etov, np.zeros((m.K, Np)), w.N, w.g, vper=m.vper, **prm)
    x, y = probe.nodes()
    del probe
    B, h, hu, hv = w.fields(x, y)
    o = oracle.Oracle(m.vx, m.vy, m.etov, B, w.N, w.g, vper=m.vper, vbc=m.vbc, **prm)
    return o, dict(x=x, y=y, B=B, h=h, hu=hu, hv=hv)


def tri_monomial_integral(a: int, b: int) -> Fraction:
    """Exact  int_T r^a s^b dr ds  over the reference triangle (-1,-1),(1,-1),(-1,1).
    r = 2 xi - 1, s = 2 eta - 1, dA = 4 dxi deta,  int_simplex xi^i eta^j = i! j! / (i+j+2)!."""
    tot = Fraction(0)
    for i in range(a + 1):
        for j in range(b + 1):
            c = comb(a, i) * comb(b, j) * (2 ** i) * (2 ** j) * ((-1) ** (a - i)) * ((-1) ** (b - j))
            tot += c * Fraction(factorial(i) * factorial(j), factorial(i + j + 2))
    return 4 * tot


def poly_eval(coef: dict, r, s):
    """coef[(a,b)] -> sum c r^a s^b"""
    return sum(c * r ** a * s ** b for (a, b), c in coef.items())


def poly_dr(coef: dict):
    return {(a - 1, b): c * a for (a, b), c in coef.items() if a > 0}


def poly_ds(coef: dict):
    return {(a, b - 1): c * b for (a, b), c in coef.items() if b > 0}


def poly_mul(p: dict, q: dict):
    out: dict = {}
    for (a, b), c in p.items():
        for (d, e), f in q.items():
            out[(a + d, b + e)] = out.get((a + d, b + e), 0.0) + c * f
    return out


def poly_integral(p: dict) -> float:
    return float(sum(Fraction(c) * tri_monomial_integral(a, b) for (a, b), c in p.items()))


def random_poly(deg: int, rng) -> dict:
    return {(a, b): float(rng.standard_normal()) for a in range(deg + 1) for b in range(deg + 1 - a)}


def parity_rel(gpu, orc, g):
    """Per-field relative Linf distance with the A23 scales."""
    hs = max(np.abs(orc[0]).max(), 1e-300)
    scales = [hs, hs * np.sqrt(g * hs), hs * np.sqrt(g * hs)]
    return [float(np.abs(a - b).max() / max(np.abs(b).max(), s)) for a, b, s in zip(gpu, orc, scales)]
