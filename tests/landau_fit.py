"""Landau-damping analysis used by the tests (post-processing of an energy series).

* ``dispersion_root(k)``: root of the linear Vlasov-Poisson dispersion relation
  1 + k^-2 (1 + zeta Z(zeta)) = 0, zeta = omega / (sqrt(2) k), with the plasma
  dispersion function Z(zeta) = i sqrt(pi) w(zeta) (scipy ``wofz``).  This is
  the "expected analytical damping rate" of P:231-232.
* ``fit_damping_rate(t, W)``: S:546-554 -- least squares of ln W at the strict
  interior local maxima against t; returns (slope, n_peaks, peak_times).
"""
from __future__ import annotations

import numpy as np
from scipy.special import wofz


def dispersion_root(k: float = 0.5, omega0: complex = 1.4 - 0.15j) -> complex:
    def D(w):
        z = w / (np.sqrt(2.0) * k)
        Z = 1j * np.sqrt(np.pi) * wofz(z)
        return 1.0 + (1.0 + z * Z) / k ** 2

    w = complex(omega0)
    for _ in range(100):
        h = 1e-7
        dD = (D(w + h) - D(w - h)) / (2 * h)
        step = D(w) / dD
        w -= step
        if abs(step) < 1e-14:
            break
    return w


def fit_damping_rate(t, W, t_max=None, floor=1e-12):
    t = np.asarray(t, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    idx = [i for i in range(1, len(W) - 1) if W[i - 1] < W[i] > W[i + 1] and W[i] > floor]
    if t_max is not None:
        idx = [i for i in idx if t[i] <= t_max]
    if len(idx) < 3:
        raise ValueError(f"InsufficientPeaks: {len(idx)}")
    tp, wp = t[idx], np.log(W[idx])
    slope = np.polyfit(tp, wp, 1)[0]
    return slope, len(idx), tp
