"""Fits the FMA-only erf-GELU of ptx.cuh::gelu_poly2 and checks it in fp32:
GELU(x) = x * (1/2 + x_c Q(x_c^2)), x_c = clamp(x, -4, 4), deg Q = 8 (least squares in the
Chebyshev basis over z = x^2 in [0, 16], weighted by x).  Prints the coefficients (float32,
constant term first) and the max |GELU error| over [-20, 20]."""
from math import erf, sqrt

import numpy as np

L, DEG = 4.0, 8
xs = np.linspace(0, L, 40001)[1:]
phi = np.array([0.5 * (1 + erf(x / sqrt(2))) for x in xs])
z = xs ** 2
V = np.polynomial.chebyshev.chebvander(2 * z / (L * L) - 1, DEG)
c, *_ = np.linalg.lstsq(V * xs[:, None], (phi - 0.5) / xs * xs, rcond=None)
coef = np.float32(np.polynomial.Chebyshev(c, domain=[0, L * L]).convert(kind=np.polynomial.Polynomial).coef)
print("coefficients:", [float(v) for v in coef])
x = np.float32(np.linspace(-20, 20, 400001))
xc = np.clip(x, -L, L).astype(np.float32)
zz = xc * xc
q = np.full_like(zz, coef[-1])
for k in range(DEG - 1, -1, -1):
    q = (q * zz + coef[k]).astype(np.float32)
g = x * (np.float32(0.5) + xc * q)
exact = np.array([0.5 * v * (1 + erf(v / sqrt(2))) for v in x.astype(np.float64)])
err = np.abs(g - exact)
inner = np.abs(x) <= L
print(f"max |err| |x|<=4: {err[inner].max():.2e}; max |err|/|x| beyond: {(err[~inner] / np.abs(x[~inner])).max():.2e}")
