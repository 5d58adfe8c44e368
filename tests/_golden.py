"""Golden-fixture readers for the tests (tests/golden/*.txt carry their citations)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name, dtype=float):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split("\t"))
    return rows


def golden_matrix(name, dtype=float):
    return np.array([[dtype(v) for v in r] for r in load_golden(name)])
