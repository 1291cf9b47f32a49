"""Extended-precision energy of a state (test infrastructure): the terms of
observables (lattice.cpp:106-137; the 5-point periodic K with cx = cy = 1 for the
BASELINE lattices) evaluated in long double and summed pairwise, so the result is
free of the O(sqrt(N) eps |H|) rounding of a sequential double sum -- the yardstick
for comparing the GPU's energy monitor with the reference's at 1e6+ sites."""
import numpy as np


def energy_ld(u, V, gamma, nx, ny, cx=1.0, cy=1.0):
    u = np.asarray(u, dtype=np.complex128).reshape(ny, nx)
    p = u.real.astype(np.longdouble)
    q = u.imag.astype(np.longdouble)
    Vl = np.asarray(V, dtype=np.float64).reshape(ny, nx).astype(np.longdouble)

    def k_apply(x):
        return (np.longdouble(2 * cx + 2 * cy) * x - np.longdouble(cx) * (np.roll(x, 1, 1) + np.roll(x, -1, 1))
                - np.longdouble(cy) * (np.roll(x, 1, 0) + np.roll(x, -1, 0)))

    kp, kq = k_apply(p), k_apply(q)
    n2 = p * p + q * q
    kin = np.sum(p * kp + q * kq)
    quart = np.sum(n2 * n2)
    ext = np.sum(Vl * n2)
    return float(kin - np.longdouble(0.5 * gamma) * quart + ext)
