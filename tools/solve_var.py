"""Diagnostic: repeated identical multi-RHS solves (graph vs direct launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.device import PcgOperator  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig, solve_block  # noqa: E402

prob = synthetic.eeg_problem("c2")
eng = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-8), prob.B, prob.C, prob.R)
op = PcgOperator(eng.assemble(), "ldp")
B = eng.Bd[:, :64].contiguous()
for mode in ("0", "1", "0", "1"):
    os.environ["HFB200_NOGRAPH"] = mode
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        solve_block(op, B, PcgConfig(1e-8))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("nograph" if mode == "1" else "graph  ", " ".join(f"{t:.0f}" for t in ts), flush=True)
