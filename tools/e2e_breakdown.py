"""Where the e2e step's extra time goes (bench.py e2e vs device-resident build):
engine construction from host arrays (H2D, B/B', G' assembly), build, LF D2H."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

prob = synthetic.eeg_problem("c2", device=True)
cfg = PcgConfig(1e-8)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = EegEngine(prob.mesh, prob.electrodes, prob.sources, cfg, prob.B, prob.C, prob.R)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    A = eng.assemble()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    T = eng.solve(A)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    LF = eng.build()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    h = LF.cpu().numpy()
    t5 = time.perf_counter()
    print(f"engine init {1e3*(t1-t0):.1f} ms | assemble {1e3*(t2-t1):.1f} | solve {1e3*(t3-t2):.1f} | "
          f"full build {1e3*(t4-t3):.1f} | LF D2H {1e3*(t5-t4):.1f} ms", flush=True)
    del eng, A, T, LF
