"""cProfile of EegEngine construction from host arrays (the e2e leg's fixed cost)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

prob = synthetic.eeg_problem("c2", device=True)
for _ in range(2):
    EegEngine(prob.mesh, prob.electrodes, prob.sources, PcgConfig(1e-8), prob.B, prob.C, prob.R)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    EegEngine(prob.mesh, prob.electrodes, prob.sources, PcgConfig(1e-8), prob.B, prob.C, prob.R)
    torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
