"""One call of the per-window path for compute-sanitizer (memcheck / racecheck / synccheck), checked
against the oracle.  usage: python tools/sanitize_case.py {C1|C2r} {flat|legacy|vectors|weighted|anon}
C2r = the first 4 windows of C2 (sanitizer replay is slow)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2509_03653_b200 as nsg  # noqa: E402
from gen.configs import CONFIGS  # noqa: E402

cfg, path = sys.argv[1], sys.argv[2]
c = CONFIGS["C1" if cfg == "C1" else "C2"]
n = c.n_packets if cfg == "C1" else 4 * c.window + 1234
keys = gen.generate_host(c.dist, c.seed, 0, n, packed=True)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
want = oracle.window_stats_sort(keys=keys, window=c.window)
if path == "anon":  # the anonymiser (f2) on the same packets, against oracle/anon.py
    s0, d0 = (keys >> np.uint64(32)).astype(np.uint32), (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    ws, wd, wn = oracle.anonymize(s0, d0, seed=5, rounds=2)
    a, b, N = nsg.anonymize(kd, seed=5, rounds=2)
    ok = (np.array_equal(a.cpu().numpy().view(np.uint32), ws) and np.array_equal(b.cpu().numpy().view(np.uint32), wd)
          and int(N.item()) == wn)
    print(f"{cfg} anon: parity {'OK' if ok else 'FAIL'} (N = {wn})")
    sys.exit(0 if ok else 1)
elif path == "vectors":
    got = nsg.window_vectors(kd, c.window)["stats"]
elif path == "weighted":
    wt = (np.arange(n, dtype=np.uint32) % 7).astype(np.uint32)  # 0..6: rows of weight 0 included
    want = oracle.window_stats_weighted(keys=keys, weights=wt, window=c.window)
    got = nsg.window_stats_weighted(kd, torch.from_numpy(wt.view(np.int32)).cuda(), c.window)
else:
    got = nsg.window_stats_packed(kd, c.window, flags=nsg.api._FLAG_LEGACY_FAST if path == "legacy" else 0)
got = got.cpu().numpy().view(np.uint64)
ok = np.array_equal(got, want)
print(f"{cfg} {path}: parity {'OK' if ok else 'FAIL'}")
sys.exit(0 if ok else 1)
