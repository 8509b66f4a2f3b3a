"""Mutation check of the oracle's pins (development aid, CPU only).

Copies oracle/ + tests/ into a scratch directory once per mutant, applies one
plausible mistake to oracle/oracle.c, runs the oracle pin tests there and reports
whether some pin fails (killed) or all pass (survived).

    python tools/oracle_mutants.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTANTS = {
    "holdout known leg selected on the train scope (P:L540, P:L553)":
        ("const uint8_t *sel_mask = pass == 0 ? tr : te;", "const uint8_t *sel_mask = pass == 0 ? tr : tr;"),
    "swap tie-break: first encountered instead of smallest tuple (S:L258-266, reading c5)":
        ("if (!have || precedes(Lt, T, Lb, Tb, k)) {", "if (!have || Lt > Lb) {"),
    "fleet missing cell costs best instead of penalty x best (P:L323-327, reading c4)":
        ("return isfinite(t) ? (double)t : penalty * best[e];", "return isfinite(t) ? (double)t : best[e];"),
    "equal scores ordered by the largest tuple (reading c5)":
        ("if (La < Lb) return 0;\n    for (int u = 0; u < k; u++) {\n        if (a[u] < b[u]) return 1;",
         "if (La < Lb) return 0;\n    for (int u = 0; u < k; u++) {\n        if (a[u] > b[u]) return 1;"),
    "greedy ties to the highest index (reading c5)":
        ("if (c1 < 0 || L > L1) {", "if (c1 < 0 || L >= L1) {"),
    "k-means empty cluster re-seeded with point 0 (S:L276)":
        ("if (dmin[q] > fd) { fd = dmin[q]; far = q; }\n                memcpy(M + (int64_t)j * C",
         "if (q < 0) { fd = dmin[q]; far = q; }\n                memcpy(M + (int64_t)j * C"),
}
PINS = ["tests/test_oracle.py", "tests/test_oracle_swap.py", "tests/test_oracle_fleet.py",
        "tests/test_oracle_kmeans.py"]


def main():
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    rc = 0
    for name, (old, new) in MUTANTS.items():
        if old not in src:
            print(f"SKIP (pattern not found)  {name}")
            continue
        with tempfile.TemporaryDirectory() as d:
            for sub in ("oracle", "tests", "paper_2507_15277_b200"):
                shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
            with open(os.path.join(d, "oracle", "oracle.c"), "w") as f:
                f.write(src.replace(old, new, 1))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"] + PINS,
                               cwd=d, capture_output=True, text=True)
            killed = r.returncode != 0
            if not killed:
                rc = 1
            print(f"{'killed  ' if killed else 'SURVIVED'}  {name}")
    return rc


if __name__ == "__main__":
    sys.exit(main())
