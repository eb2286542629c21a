import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1811_10136_b200 as fr
from paper_1811_10136_b200.permutohedral import PermutohedralLattice
torch.cuda.init()
x = torch.empty(1, device='cuda')
for i in range(5): PermutohedralLattice(3, np.full(3, 0.01))
ts=[]
for i in range(20):
    t0=time.perf_counter(); l=PermutohedralLattice(3, np.full(3, 0.01)); ts.append(time.perf_counter()-t0); del l
print("create idle: median %.1f us" % (1e6*np.median(ts)))
s = torch.cuda.Stream()
ts=[]
big = torch.empty(50_000_000, device='cuda')
for i in range(20):
    with torch.cuda.stream(s):
        big.mul_(1.0001)   # ~ 0.1-0.2 ms of work on a side stream
    t0=time.perf_counter(); l=PermutohedralLattice(3, np.full(3, 0.01)); ts.append(time.perf_counter()-t0); del l
    torch.cuda.synchronize()
print("create with side-stream work pending: median %.1f us" % (1e6*np.median(ts)))
ts=[]
for i in range(20):
    big.mul_(1.0001)
    t0=time.perf_counter(); l=PermutohedralLattice(3, np.full(3, 0.01)); ts.append(time.perf_counter()-t0); del l
    torch.cuda.synchronize()
print("create with default-stream work pending: median %.1f us" % (1e6*np.median(ts)))
