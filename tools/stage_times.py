"""Where one C2 LF build's time goes, stage by stage (wall clock with a device
synchronize around each stage; diagnostics, not a bench value)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.device import PcgOperator  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.leadfield import response_operator, symmetrize  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig, solve_block  # noqa: E402

prob = synthetic.eeg_problem(sys.argv[1] if len(sys.argv) > 1 else "c2", device=True)
eng = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-8), prob.B, prob.C, prob.R)
eng.build()


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for rep in range(3):
    A, ta = t(eng.assemble)
    op, to = t(lambda: PcgOperator(A, "ldp"))
    (T, info), ts = t(lambda: solve_block(op, eng.Bd, eng.cfg))
    Mr, tm = t(lambda: eng.response_block(T))
    W, tw = t(lambda: response_operator(symmetrize(Mr.cpu().numpy()), eng.R))
    LF, tl = t(lambda: eng.lf_partial(T, W))
    _, tb = t(eng.build)
    it = info.iterations
    print(f"assemble {ta:.1f}  operator {to:.1f}  solve {ts:.1f} (2 x {int(it[:64].max())}/{int(it[64:].max())} "
          f"rounds)  response {tm:.1f}  W {tw:.1f}  tail {tl:.1f}  | build() {tb:.1f} ms", flush=True)
