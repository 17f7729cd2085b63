"""The reference's acceptance problems, restated for the GPU tests (test
infrastructure; the package has no problem catalogue).

helmholtz: on [0, pi]^3, k(z) = a - b sin(cz), exact u = sin(beta x) sin(gamma y)
g(z) with g = exp(-k/c) (beta^2 + gamma^2 = a^2 + b^2) and source
f = -b (2a + c) sin(beta x) sin(gamma y) sin(cz) g(z)   (problems.py:89-185).
convdiff: on [0, sqrt2]^2 x [0, 1], zero source, u = sin(pi x/sqrt2) sin(pi y/sqrt2)
Z(z), Z = A+ e^{r+ z} + A- e^{r- z} matching 1x / 2x the horizontal mode at
z = 0 / 1 (problems.py:188-246).

The z-derivatives the 4th/6th-order right-hand sides need (up to f_zzzz) come
from truncated Taylor arithmetic ("jets") instead of closed forms.
"""
import math

import numpy as np

import paper_1912_03565_b200 as hb

K = 4  # highest derivative order carried


class Jet:
    """Taylor coefficients c[k] = f^(k)(z) / k!, k <= K, vectorised over z."""

    def __init__(self, coeffs):
        self.c = coeffs

    @staticmethod
    def var(z):
        z = np.asarray(z, dtype=float)
        c = [z, np.ones_like(z)] + [np.zeros_like(z) for _ in range(K - 1)]
        return Jet(c)

    def __add__(self, o):
        if isinstance(o, Jet):
            return Jet([a + b for a, b in zip(self.c, o.c)])
        return Jet([self.c[0] + o] + self.c[1:])

    __radd__ = __add__

    def __mul__(self, o):
        if isinstance(o, Jet):
            return Jet([sum(self.c[i] * o.c[k - i] for i in range(k + 1)) for k in range(K + 1)])
        return Jet([a * o for a in self.c])

    __rmul__ = __mul__

    def __neg__(self):
        return self * -1.0

    def __sub__(self, o):
        return self + (-o)

    def derivative(self, k):
        return math.factorial(k) * self.c[k]


def jexp(a):
    e = [np.exp(a.c[0])]
    for k in range(1, K + 1):
        e.append(sum(i * a.c[i] * e[k - i] for i in range(1, k + 1)) / k)
    return Jet(e)


def jsincos(a):
    s, c = [np.sin(a.c[0])], [np.cos(a.c[0])]
    for k in range(1, K + 1):
        s.append(sum(i * a.c[i] * c[k - i] for i in range(1, k + 1)) / k)
        c.append(-sum(i * a.c[i] * s[k - i] for i in range(1, k + 1)) / k)
    return Jet(s), Jet(c)


def helmholtz_case(a, b, c, beta, gamma, scheme, n):
    """(grid, profile, source, boundary, exact u) of the variable-k problem."""
    g = hb.make_grid(hb.Domain(0.0, math.pi, 0.0, math.pi, 0.0, math.pi), n, n, n)
    k2 = lambda z: (a - b * np.sin(c * z)) ** 2
    k2z = lambda z: -2.0 * b * c * np.cos(c * z) * (a - b * np.sin(c * z))
    k2zz = lambda z: (2.0 * b**2 * c**2 * np.cos(c * z) ** 2
                      + 2.0 * b * c**2 * np.sin(c * z) * (a - b * np.sin(c * z)))
    prof = hb.sample_profile(k2, k2z, k2zz, 0.0, g)
    c0 = -b * (2.0 * a + c)

    def gz(z):
        s, _ = jsincos(Jet.var(z) * c)
        return jexp((s * b - a) * (1.0 / c))

    def psi(z):  # sin(cz) g(z) as a jet
        s, _ = jsincos(Jet.var(z) * c)
        return s * jexp((s * b - a) * (1.0 / c))

    ang = lambda x, y: np.sin(beta * x) * np.sin(gamma * y)
    u = lambda x, y, z: ang(x, y) * gz(z).c[0]

    def fz(order):
        return lambda x, y, z: c0 * ang(x, y) * psi(z).derivative(order)

    f = fz(0)
    src = hb.SourceSpec(
        f=f, f_z=fz(1), f_zz=fz(2),
        f_xx=lambda x, y, z: -beta**2 * f(x, y, z),
        f_yy=lambda x, y, z: -gamma**2 * f(x, y, z),
        lap_f=lambda x, y, z: -(beta**2 + gamma**2) * f(x, y, z) + fz(2)(x, y, z),
        f_xxyy=lambda x, y, z: beta**2 * gamma**2 * f(x, y, z),
        f_xxzz=lambda x, y, z: -beta**2 * fz(2)(x, y, z),
        f_yyzz=lambda x, y, z: -gamma**2 * fz(2)(x, y, z),
        d4_f=lambda x, y, z: (beta**4 + gamma**4) * f(x, y, z) + fz(4)(x, y, z))
    return g, prof, src, hb.BoundaryData.from_function(u), u


def convdiff_case(gamma, n):
    root2 = math.sqrt(2.0)
    g = hb.make_grid(hb.Domain(0.0, root2, 0.0, root2, 0.0, 1.0), n, n, n)
    prof = hb.constant_profile(0.0, g, gamma=gamma)
    sigma = math.sqrt(math.pi**2 + gamma**2 / 4.0)
    rp, rm = -gamma / 2.0 + sigma, -gamma / 2.0 - sigma
    # Z(0) = 1, Z(1) = 2 with both exponentials kept finite for |gamma| ~ 100:
    # A+ e^{rp} + A- e^{rm} = 2, A+ + A- = 1, solved in decayed form
    decay = math.exp(-2.0 * sigma)
    q = math.exp(gamma / 2.0 - sigma)
    ap = (2.0 * q - decay) / (1.0 - decay)
    am = (1.0 - 2.0 * q) / (1.0 - decay)
    p = math.pi / root2
    u = lambda x, y, z: np.sin(p * x) * np.sin(p * y) * (ap * np.exp(rp * z) + am * np.exp(rm * z))
    return g, prof, hb.SourceSpec.zero(), hb.BoundaryData.from_function(u), u


def error_metrics(values, u, g):
    x = g.x_nodes()[None, None, :]
    y = g.y_nodes()[None, :, None]
    z = g.z_nodes()[:, None, None]
    exact = u(x, y, z)
    d = np.asarray(values).real - exact
    return float(np.abs(d).max()), float(np.linalg.norm(d) / np.linalg.norm(exact))
