"""C4 (node graph, 100k points, 195 nodes) registration for a launch list
(ncu --metrics gpu__time_duration.sum): the device-resident loop's kernels."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1811_10136_b200 as fr  # noqa: E402
from paper_1811_10136_b200.kinematics import NodeGraph, Skinning  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "config_c4.npz"))
graph = lambda: NodeGraph(g["nodes"], g["edges"], Skinning(g["skin_idx"], g["skin_w"]))  # noqa
cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.02, outlier_ratio=0.1),
                            max_em_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 3,
                            twist_tolerance=1e-5, mstep=fr.MStepOptions(lambda_reg=0.1))
ref, obs = fr.PointCloud(g["X"].astype(float)), fr.PointCloud(g["Y"].astype(float))
res = fr.register(ref, obs, graph(), cfg)
torch.cuda.synchronize()
print(res.iterations, res.termination)
