"""Parity gates shared by the GPU tests, with a per-session report (printed by conftest).

north_star: max-abs <= 1e-5 (fp32) and <= 2e-2 (bf16) against the fp64 oracle.  A bf16
*output* is itself rounded to the bf16 grid, so (G27) a bf16 element also passes
if |got - ref| <= 2e-2 + ulp_bf16(ref)/2: within the gate of the correctly rounded value's
neighbourhood.  Every check records the plain max-abs and how many elements passed only
through that clause (|got - ref| > 2e-2), so the relaxation's use is visible in the log.
"""
import os

import numpy as np

TOL = {"f32": 1e-5, "bf16": 2e-2}
REPORT = []   # dicts: test, name, dt, maxabs, n, n_clause, bound_max, ok


def bf16_ulp(ref):
    """Spacing of the bf16 grid at |ref| (8 significant bits)."""
    a = np.abs(np.asarray(ref, dtype=np.float64))
    return np.exp2(np.floor(np.log2(np.maximum(a, 2.0 ** -126))) - 7)


def _test_name():
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]


def excess(got, ref, dt, name="", scale=1.0):
    """max over elements of |got - ref| - bound (<= 0 passes) and record the check.
    got, ref: float64 arrays of the same shape; scale multiplies the plain gate (composites,
    reading G24)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if not ref.size:
        return 0.0
    e = np.abs(got - ref)
    plain = TOL[dt] * scale
    bound = plain if dt == "f32" else plain + 0.5 * bf16_ulp(ref)
    ex = float((e - bound).max())
    REPORT.append(dict(test=_test_name(), name=name, dt=dt, maxabs=float(e.max()), n=int(e.size),
                       n_clause=int(((e > plain) & (e <= bound)).sum()), plain=plain, ok=ex <= 0))
    return ex


def summary_lines():
    if not REPORT:
        return []
    out = [f"parity gate report: {len(REPORT)} checks, {sum(not r['ok'] for r in REPORT)} failing"]
    for dt in ("f32", "bf16"):
        rs = [r for r in REPORT if r["dt"] == dt]
        if not rs:
            continue
        worst = max(rs, key=lambda r: r["maxabs"] / r["plain"])
        out.append(f"  {dt}: {len(rs)} checks, worst max-abs/gate = {worst['maxabs'] / worst['plain']:.3f} "
                   f"({worst['maxabs']:.3g} in {worst['test']} {worst['name']}); elements passing only via the "
                   f"1/2-ulp clause: {sum(r['n_clause'] for r in rs)} of {sum(r['n'] for r in rs)}")
    for r in REPORT:
        if r["n_clause"]:
            out.append(f"  clause used: {r['test']} {r['name']}: {r['n_clause']} of {r['n']} elements, "
                       f"max-abs {r['maxabs']:.4g}")
    return out
