#!/usr/bin/env python
"""Render a PARITY_REPORT JSON (tests/parity.py records) as the markdown table
DESIGN.md §7 carries: per check, entries, violations, max |gpu - ref| and the
worst error as a fraction of the north-star tolerance (1e-6 + 1e-4 |ref|)."""
import json
import sys


def main(path):
    recs = json.load(open(path))
    print("| Check | Entries | Violations | max abs err | max err / (1e-6 + 1e-4 |ref|) | max err / Σ|terms| |")
    print("|---|---|---|---|---|---|")
    for r in recs:
        if "violations" in r:
            mag = f"{r['max_err_over_mag']:.2e}" if r.get("mag_used") else "—"
            print(f"| {r['check']} | {r['entries']:,} | {r['violations']} | {r['max_abs_err']:.2e} | "
                  f"{r['max_rel_err_vs_1e-4_bar']:.3g} | {mag} |")
        elif "counters_identical" in r:
            print(f"| {r['check']} | {r['queries']:,} queries | "
                  f"{0 if r['counters_identical'] else 'MISMATCH'} | identical visited/far/leaf "
                  f"counts: {r['counters_identical']} | | |")
        else:
            print(f"| {r['check']} | | | GPU {r['gpu_max_abs_err']:.4g} / oracle "
                  f"{r['ref_max_abs_err']:.4g} max abs (mean rel {r['gpu_mean_err_over_max_naive']:.2e}) | | |")


if __name__ == "__main__":
    main(sys.argv[1])
