import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, gen, paper_2509_03653_b200 as nsg
from gen.configs import CONFIGS
c = CONFIGS[os.environ.get("CFG", "C2")]
dev = torch.device("cuda", 0)
keys = gen.generate_host(c.dist, c.seed, 0, c.n_packets, packed=True)
kd = torch.from_numpy(keys.view(np.int64)).to(dev)
for _ in range(int(os.environ.get("REPS", "3"))):
    nsg.window_stats_packed(kd, c.window)
torch.cuda.synchronize()
print("done")
