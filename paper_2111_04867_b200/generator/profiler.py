"""The alpha-beta profiler's solver (§4.1, Table 1).

The paper measures each link twice: "We send n chunks one after another on a link and measure
the time to transfer. As per the alpha-beta cost model, the time to transfer is
n * (alpha + beta * s). We then send n chunks all at once on the link and attribute that time to
be alpha + n * beta * s. Using several measurements of time to transfer, we solve for alpha and
beta.". `solve_alpha_beta` is that solve, by linear least squares over every
measurement. On B200 each measurement is one executor call (tools/ab_profile.py: a 2-rank
schedule whose k chunks per rank travel as k steps, or as one k-chunk step), so a fixed per-call
cost c (launch, prologue, exit) that is not a per-transfer cost is fitted beside alpha and beta:
    one after another: t = c + k * (alpha + beta * s)
    all at once:       t = c + alpha + k * beta * s
(fit_c=False drops c, the paper's form.) Units: t and alpha in us, s in MB (2^20 bytes), beta
in us/MB.

`connection_table` summarises the connection-count sweep (the paper's fig:multiconnection,
PAPER.md:405-418: accumulated ingress/egress bandwidth of a fixed volume split over 1..n-1
connections through the switch), measured by tools/nvlink_probe.cu.
"""
from __future__ import annotations

import numpy as np


def solve_alpha_beta(meas, fit_c=True):
    """meas: iterable of (mode, k, s_mb, t_us), mode "seq" (k chunks one after another) or
    "tog" (k chunks at once). Returns {"alpha_us", "beta_us_per_MB", "c_us", "rms_us", "points"}."""
    rows, ts = [], []
    for mode, k, s, t in meas:
        if mode == "seq":
            a_coef, b_coef = k, k * s
        elif mode == "tog":
            a_coef, b_coef = 1, k * s
        else:
            raise ValueError(mode)
        rows.append(([1.0] if fit_c else []) + [float(a_coef), float(b_coef)])
        ts.append(float(t))
    A, y = np.array(rows), np.array(ts)
    if len(y) < A.shape[1]:
        raise ValueError(f"{len(y)} measurements for {A.shape[1]} unknowns")
    x, *_ = np.linalg.lstsq(A, y, rcond=None)
    c, alpha, beta = (x[0], x[1], x[2]) if fit_c else (0.0, x[0], x[1])
    resid = y - A @ x
    return {"alpha_us": float(alpha), "beta_us_per_MB": float(beta), "c_us": float(c),
            "rms_us": float(np.sqrt(np.mean(resid ** 2))), "points": int(len(y)),
            "GBps": float((1 << 20) / (beta * 1e-6) / 1e9) if beta > 0 else None}


def connection_table(rows, volume=None):
    """rows: nvlink_probe JSON objects with probe == "connections". Returns, per number of
    connections c, the accumulated egress GB/s per GPU at `volume` bytes (default: the
    largest measured) and its ratio to one connection."""
    rows = [r for r in rows if r.get("probe") == "connections"]
    if not rows:
        return []
    vol = volume or max(r["volume_bytes"] for r in rows)
    pick = {}
    for r in rows:
        if abs(r["volume_bytes"] - vol) <= 0.01 * vol:
            pick[r["connections"]] = r["egress_GBps"]
    base = pick.get(1)
    return [{"connections": c, "volume_bytes": vol, "egress_GBps": bw,
             "vs_one_connection": round(bw / base, 4) if base else None} for c, bw in sorted(pick.items())]
