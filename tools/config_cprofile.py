"""cProfile of one warm register() of C3 or C4 (diagnostic: where the host-side
setup time goes).   python tools/config_cprofile.py c3|c4"""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import configs_timing as C  # noqa: E402

which = sys.argv[1].upper() if len(sys.argv) > 1 else "C4"
torch.cuda.set_device(0)
for name, g, ref, obs, model, config in C.cases():
    if name != which:
        continue
    fr = C.fr
    for _ in range(2):
        fr.register(ref, obs, model(), config)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    m = model()
    pr.enable()
    fr.register(ref, obs, m, config)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats(os.environ.get("SORT", "tottime")).print_stats(int(os.environ.get("TOP", "25")))
    break
