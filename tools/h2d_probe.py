import torch, time
dev=torch.device('cuda',0)
for mb in (64,256):
    n=mb<<20
    h=torch.empty(n,dtype=torch.uint8,pin_memory=True); h.fill_(1)
    d=torch.empty(n,dtype=torch.uint8,device=dev)
    for _ in range(3): d.copy_(h,non_blocking=True)
    torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): d.copy_(h,non_blocking=True)
    b.record(); torch.cuda.synchronize()
    print(mb,'MB H2D', n*10/(a.elapsed_time(b)/1e3)/1e9,'GB/s')
    a.record()
    for _ in range(10): h.copy_(d,non_blocking=True)
    b.record(); torch.cuda.synchronize()
    print(mb,'MB D2H', n*10/(a.elapsed_time(b)/1e3)/1e9,'GB/s')
import subprocess
print(subprocess.run(['nvidia-smi','-q','-d','PCIE'],capture_output=True,text=True).stdout[:1500])
