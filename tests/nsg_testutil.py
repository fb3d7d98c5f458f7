"""Helpers shared by the tests (fixture parsing)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name):
    """Parse a tests/golden fixture into [(window, src, dst, expected_rows)]."""
    cases = []
    window = None
    mode = None
    src, dst, exp = [], [], []
    with open(os.path.join(GOLDEN, name)) as f:
        for raw in f:
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("window"):
                if window is not None:
                    cases.append((window, np.array(src, np.uint32), np.array(dst, np.uint32), np.array(exp, np.uint64)))
                window, src, dst, exp = int(line.split()[1]), [], [], []
            elif line in ("packets", "expect"):
                mode = line
            elif mode == "packets":
                a, b = line.split()
                src.append(int(a))
                dst.append(int(b))
            else:
                exp.append([int(x) for x in line.split()])
    cases.append((window, np.array(src, np.uint32), np.array(dst, np.uint32), np.array(exp, np.uint64)))
    return cases
