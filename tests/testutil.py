"""Shared test helpers (importable as `testutil`: pytest puts tests/ on sys.path)."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_golden(name):
    """Rows of a whitespace table under tests/golden/ (comment lines start with '#')."""
    rows = {}
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            rows[parts[0]] = [float(x) for x in parts[1:]]
    return rows
