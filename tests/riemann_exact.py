"""Exact solution of the 1-D Euler Riemann problem (ideal gas), for the Sod check
(acceptance criterion 7, reference tests/test_acceptance.py:164-184). Test
infrastructure: the standard two-rarefaction/two-shock pressure function solved
by Newton iteration, then the self-similar sampling of the wave fan.
"""

import numpy as np


def _f_and_df(p, rho, pk, ck, gamma):
    """Velocity change across the wave connecting state k to the star pressure p."""
    if p > pk:   # shock
        A = 2.0 / ((gamma + 1.0) * rho)
        B = (gamma - 1.0) / (gamma + 1.0) * pk
        sq = np.sqrt(A / (p + B))
        return (p - pk) * sq, sq * (1.0 - 0.5 * (p - pk) / (p + B))
    # rarefaction
    pr = p / pk
    f = 2.0 * ck / (gamma - 1.0) * (pr ** ((gamma - 1.0) / (2.0 * gamma)) - 1.0)
    df = 1.0 / (rho * ck) * pr ** (-(gamma + 1.0) / (2.0 * gamma))
    return f, df


def star_state(left, right, gamma=1.4):
    """(p*, u*) of the Riemann problem left = (rho, u, p), right = (rho, u, p)."""
    rl, ul, pl = left
    rr, ur, pr = right
    cl, cr = np.sqrt(gamma * pl / rl), np.sqrt(gamma * pr / rr)
    p = max(1e-8, 0.5 * (pl + pr) - 0.125 * (ur - ul) * (rl + rr) * (cl + cr))
    for _ in range(100):
        fl, dfl = _f_and_df(p, rl, pl, cl, gamma)
        fr, dfr = _f_and_df(p, rr, pr, cr, gamma)
        dp = (fl + fr + ur - ul) / (dfl + dfr)
        pn = max(1e-8, p - dp)
        if abs(pn - p) <= 1e-14 * (pn + p):
            p = pn
            break
        p = pn
    fl, _ = _f_and_df(p, rl, pl, cl, gamma)
    fr, _ = _f_and_df(p, rr, pr, cr, gamma)
    return p, 0.5 * (ul + ur) + 0.5 * (fr - fl)


def riemann_density(x, t, x0=0.5, left=(1.0, 0.0, 1.0), right=(0.125, 0.0, 0.1), gamma=1.4):
    """Exact density at positions x and time t > 0 (Sod defaults)."""
    rl, ul, pl = left
    rr, ur, pr = right
    ps, us = star_state(left, right, gamma)
    cl, cr = np.sqrt(gamma * pl / rl), np.sqrt(gamma * pr / rr)
    g1 = (gamma - 1.0) / (gamma + 1.0)
    out = np.empty_like(np.asarray(x, dtype=np.float64))
    for idx, xi in np.ndenumerate(np.asarray(x, dtype=np.float64)):
        s = (xi - x0) / t
        if s <= us:   # left of the contact
            if ps > pl:   # left shock
                sl = ul - cl * np.sqrt((gamma + 1.0) / (2.0 * gamma) * ps / pl
                                       + (gamma - 1.0) / (2.0 * gamma))
                out[idx] = rl if s < sl else rl * (ps / pl + g1) / (g1 * ps / pl + 1.0)
            else:         # left rarefaction
                cls = cl * (ps / pl) ** ((gamma - 1.0) / (2.0 * gamma))
                if s < ul - cl:
                    out[idx] = rl
                elif s > us - cls:
                    out[idx] = rl * (ps / pl) ** (1.0 / gamma)
                else:
                    out[idx] = rl * (2.0 / (gamma + 1.0) + g1 / cl * (ul - s)) ** (
                        2.0 / (gamma - 1.0))
        else:          # right of the contact
            if ps > pr:   # right shock
                sr = ur + cr * np.sqrt((gamma + 1.0) / (2.0 * gamma) * ps / pr
                                       + (gamma - 1.0) / (2.0 * gamma))
                out[idx] = rr if s > sr else rr * (ps / pr + g1) / (g1 * ps / pr + 1.0)
            else:         # right rarefaction
                crs = cr * (ps / pr) ** ((gamma - 1.0) / (2.0 * gamma))
                if s > ur + cr:
                    out[idx] = rr
                elif s < us + crs:
                    out[idx] = rr * (ps / pr) ** (1.0 / gamma)
                else:
                    out[idx] = rr * (2.0 / (gamma + 1.0) - g1 / cr * (ur - s)) ** (
                        2.0 / (gamma - 1.0))
    return out
