import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_2509_03653_b200 as nsg
dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
keys = gen.generate_host(gen.Dist("zipf", 1.1, 1 << 16), 72, 0, n, packed=True)
kd = torch.from_numpy(keys.view(np.int64)).to(dev)
ws = nsg.TraceWorkspace(n, n, world, dev)
send, counts = nsg.trace_partition(kd, world, ws)
torch.cuda.synchronize()
print("counts", counts.cpu().tolist())
