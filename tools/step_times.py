"""Diagnostic: per-step LF build times (CUDA events) on C2 under different
allocation patterns (reused engine, emptied caching allocator, fresh engine)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

prob = synthetic.eeg_problem(sys.argv[1] if len(sys.argv) > 1 else "c2")
mk = lambda: EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-8), prob.B, prob.C, prob.R)
eng = mk()
s = torch.cuda.current_stream()


def timed(f):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    f()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for phase in ("reuse", "empty_cache", "fresh", "reuse2"):
    ts = []
    for i in range(4):
        if phase == "empty_cache":
            torch.cuda.empty_cache()
        if phase == "fresh":
            eng = mk()
        ts.append(timed(lambda: eng.build()))
    print(phase, " ".join(f"{t:.0f}" for t in ts), "ms", flush=True)
