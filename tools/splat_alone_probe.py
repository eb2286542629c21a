"""The observation lattice build alone (float64 planes of the C5 1M
observation cloud, four builds; FR_SPLAT_TIMING=1|2 prints the phases)."""
import os, sys, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from oracle import filterreg_oracle as O
import paper_1811_10136_b200 as fr
from paper_1811_10136_b200 import _rigid
from paper_1811_10136_b200.permutohedral import PermutohedralLattice
model, obs, _ = O.pebble_pair(1000000, outlier_ratio=0.05, seed=0)
Y = obs.astype(np.float32).astype(float)
s = 0.05 * O.bbox_diameter(Y)
soa = _rigid.upload_soa64(Y, torch.device("cuda", 0))
torch.cuda.synchronize()
for r in range(4):
    lat = PermutohedralLattice(3, np.full(3, s))
    print("rep", r, file=sys.stderr)
    lat.splat_points(soa, None, 0)
    lat.blur()
    torch.cuda.synchronize()
