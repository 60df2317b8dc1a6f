"""The parity criterion every GPU-vs-oracle test applies (BASELINE.json
north_star; SURVEY §8(d) "parity criterion"), with violation counts reported.

An output entry passes when

    |gpu - ref| <= max(ATOL + RTOL * |ref|,  KAPPA * sum|terms|)

ATOL = 1e-6, RTOL = 1e-4 is the north-star bar. sum|terms| is the oracle's own
per-entry sum of the absolute values of the terms the reference accumulated
into that output (oracle/dipole_oracle.c, *_mag / *_ex entry points; vector
terms by their norm). Where the reference's sum cancels, fp32 interaction
arithmetic carries an error proportional to the terms, not to their
difference: KAPPA = 1e-5 bounds it (about 80 fp32 ulps of every term summed
with the same sign — the per-term error of the fp32 coefficient / distance
arithmetic is a few ulps). Entries without a magnitude (mag=None) get the
plain north-star bar. Zero violations are required everywhere.

Every check is recorded; with PARITY_REPORT=<path> in the environment the
session writes the records (max error, max error / tolerance, violations)
as JSON (tests/conftest.py), the source of DESIGN.md's parity table.
"""
import numpy as np

RTOL, ATOL, KAPPA = 1e-4, 1e-6, 1e-5

RECORDS = []


def check(name, got, want, mag=None, rtol=RTOL, atol=ATOL, kappa=KAPPA):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    err = np.abs(got - want)
    tol = atol + rtol * np.abs(want)
    if mag is not None:
        mag = np.asarray(mag, np.float64)
        tol = np.maximum(tol, kappa * mag)
    ok = err <= tol  # NaN fails
    nviol = int((~ok).sum())
    ratio = float(np.max(err / tol, initial=0.0)) if err.size else 0.0
    rec = {"check": name, "entries": int(err.size), "violations": nviol,
           "max_abs_err": float(np.max(err, initial=0.0)),
           "max_err_over_tol": ratio,
           "max_rel_err_vs_1e-4_bar": float(np.max(err / (atol + rtol * np.abs(want)), initial=0.0)),
           "mag_used": mag is not None}
    if mag is not None:
        rec["entries_needing_mag"] = int((err > atol + rtol * np.abs(want)).sum())
        rec["max_err_over_mag"] = float(np.max(err / np.maximum(mag, 1e-300), initial=0.0))
    RECORDS.append(rec)
    if nviol:
        i = int(np.argmax(np.where(ok, -np.inf, err / tol)))
        raise AssertionError(f"{name}: {nviol} of {err.size} entries violate the parity bar; worst "
                             f"flat index {i}: gpu {got.ravel()[i]!r} ref {want.ravel()[i]!r} tol "
                             f"{tol.ravel()[i]:.3e}")
    return rec


def scalar(name, got, want, mag=None, rtol=RTOL, atol=ATOL, kappa=KAPPA):
    return check(name, np.array([got]), np.array([want]),
                 None if mag is None else np.array([mag]), rtol, atol, kappa)


def counters_equal(name, cnt, wcnt):
    """Identical opening decisions: visited, far-field accepts and leaf-point
    interactions per query (near / far split may differ only by the t < 6.5
    rounding of the same distance, so sums are compared)."""
    cnt, wcnt = np.asarray(cnt), np.asarray(wcnt)
    if wcnt.ndim == 1:
        ok = np.array_equal(cnt[:, 0], wcnt)
    else:
        ok = (np.array_equal(cnt[:, 0], wcnt[:, 0])
              and np.array_equal(cnt[:, 1] + cnt[:, 2], wcnt[:, 1] + wcnt[:, 2])
              and np.array_equal(cnt[:, 3] + cnt[:, 4], wcnt[:, 3] + wcnt[:, 4]))
    RECORDS.append({"check": name, "counters_identical": bool(ok), "queries": int(cnt.shape[0])})
    assert ok, name
