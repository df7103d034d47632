"""Diagnostic: per-step LF build times (CUDA events and wall clock) on C2."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

prob = synthetic.eeg_problem(sys.argv[1] if len(sys.argv) > 1 else "c2")
eng = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-8), prob.B, prob.C, prob.R)
s = torch.cuda.current_stream()
for phase in ("plain", "smi", "plain2"):
    proc = None
    if phase == "smi":
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv",
                                 "-lms", "200"], stdout=subprocess.DEVNULL)
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w = time.perf_counter()
        e0.record(s)
        eng.build()
        e1.record(s)
        torch.cuda.synchronize()
        print(phase, i, f"event {e0.elapsed_time(e1):.1f} ms  wall {(time.perf_counter() - w) * 1e3:.1f} ms",
              flush=True)
    if proc:
        proc.terminate()
