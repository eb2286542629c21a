"""cProfile of the articulated (C3) and node-graph (C4) registrations on the
GPU box: where the host-side M-step time goes.   python tools/mstep_profile.py"""
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_1811_10136_b200 as fr  # noqa: E402
from configs_timing import cases  # noqa: E402

for name, ref, obs, model, config in cases():
    if name not in sys.argv[1:] and len(sys.argv) > 1:
        continue
    if name in ("C1", "C2"):
        continue
    fr.register(ref, obs, model(), config)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    fr.register(ref, obs, model(), config)
    torch.cuda.synchronize()
    pr.disable()
    print("=====", name)
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
