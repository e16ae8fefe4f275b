"""TEST INFRASTRUCTURE — feature-parity metric of SURVEY §8(c).

rel_e = |g - r| / max(|r|, 1e-3 * ||r||_inf), per element; a layer passes when
max(rel_e) <= 1e-2 and mean(rel_e) <= 1e-3 (north_star tolerance for 16-bit operands with
fp32 accumulation). The Frobenius-relative error is reported beside it.
"""
import numpy as np

MAX_TOL, MEAN_TOL = 1e-2, 1e-3


def elementwise_errors(g, r):
    """(max rel_e, mean rel_e, Frobenius-relative error) of g against the reference r."""
    g64 = np.asarray(g, np.float64)
    r64 = np.asarray(r, np.float64)
    assert g64.shape == r64.shape, (g64.shape, r64.shape)
    if r64.size == 0:
        return 0.0, 0.0, 0.0
    d = np.abs(g64 - r64)
    inf = float(np.abs(r64).max())
    floor = max(1e-3 * inf, 1e-30)
    e = d / np.maximum(np.abs(r64), floor)
    fro = float(np.linalg.norm(d) / max(np.linalg.norm(r64), 1e-30))
    return float(e.max()), float(e.mean()), fro


def assert_north_star(g, r, what=""):
    mx, mean, fro = elementwise_errors(g, r)
    assert mx <= MAX_TOL and mean <= MEAN_TOL, f"{what}: max rel_e {mx:.3e}, mean {mean:.3e}, fro {fro:.3e}"
    return mx, mean, fro
