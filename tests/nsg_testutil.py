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


def load_golden_dist(name):
    """Parse a distributions fixture (tests/golden/dist_*.txt) into [(window, src, dst, expected)], with
    expected = dict of numpy arrays keyed like oracle.window_slices()."""
    cases, cur, mode = [], None, None

    def flush():
        if cur is None:
            return
        ln = np.array(cur["links"], np.uint64).reshape(-1, 3)
        so = np.array(cur["sources"], np.uint64).reshape(-1, 3)
        de = np.array(cur["destinations"], np.uint64).reshape(-1, 3)
        exp = {"link_key": (ln[:, 0] << np.uint64(32)) | ln[:, 1], "link_packets": ln[:, 2],
               "src_node": so[:, 0].astype(np.uint32), "src_packets": so[:, 1], "src_fan": so[:, 2],
               "dst_node": de[:, 0].astype(np.uint32), "dst_packets": de[:, 1], "dst_fan": de[:, 2],
               "ip_sets": np.array(cur["ipsets"][0], np.uint64)}
        cases.append((cur["window"], np.array(cur["src"], np.uint32), np.array(cur["dst"], np.uint32), exp))

    with open(os.path.join(GOLDEN, name)) as f:
        for raw in f:
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("window"):
                flush()
                cur = {"window": int(line.split()[1]), "src": [], "dst": [], "links": [], "sources": [],
                       "destinations": [], "ipsets": []}
            elif line in ("packets", "links", "sources", "destinations", "ipsets"):
                mode = line
            elif mode == "packets":
                a, b = line.split()
                cur["src"].append(int(a))
                cur["dst"].append(int(b))
            else:
                cur[mode].append([int(x) for x in line.split()])
    flush()
    return cases


def load_golden_weighted(name):
    """Parse a weighted-rows fixture into [(window, src, dst, weights, expected_rows)]."""
    cases, cur, mode = [], None, None

    def flush():
        if cur is not None:
            cases.append((cur["window"], np.array(cur["s"], np.uint32), np.array(cur["d"], np.uint32),
                          np.array(cur["w"], np.uint32), np.array(cur["e"], np.uint64)))

    with open(os.path.join(GOLDEN, name)) as f:
        for raw in f:
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("window"):
                flush()
                cur = {"window": int(line.split()[1]), "s": [], "d": [], "w": [], "e": []}
            elif line in ("rows", "expect"):
                mode = line
            elif mode == "rows":
                a, b, c = line.split()
                cur["s"].append(int(a)); cur["d"].append(int(b)); cur["w"].append(int(c))
            else:
                cur["e"].append([int(x) for x in line.split()])
    flush()
    return cases
