import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, gen, paper_2509_03653_b200 as nsg
dev = torch.device("cuda", 0)
keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 20), 2, 0, 1 << 17, packed=True)
kd = torch.from_numpy(keys.view(np.int64)).to(dev)
torch.cuda.synchronize()
for i in range(2):
    t0 = time.time()
    nsg.window_stats_packed(kd, 1 << 17)
    torch.cuda.synchronize()
    print("call", i, time.time() - t0, flush=True)
