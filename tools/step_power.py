"""Diagnostic: per-step LF build time next to the SM clock / power sampled by
nvidia-smi during that step (is the step-to-step variance power capping?)."""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

prob = synthetic.eeg_problem("c2")
eng = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-8), prob.B, prob.C, prob.R)
samples = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                         "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown",
                         "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)


def reader():
    for line in proc.stdout:
        samples.append((time.time(), line.strip()))


threading.Thread(target=reader, daemon=True).start()
time.sleep(1.0)
for i in range(10):
    torch.cuda.synchronize()
    t0 = time.time()
    eng.build()
    torch.cuda.synchronize()
    t1 = time.time()
    win = [s.split(", ") for (t, s) in samples if t0 <= t <= t1]
    sm = [float(w[0]) for w in win if len(w) >= 6]
    pw = [float(w[2]) for w in win if len(w) >= 6]
    cap = sum(w[4].startswith("Active") for w in win if len(w) >= 6)
    print(f"step {i}: {(t1 - t0) * 1e3:.0f} ms  sm median {np.median(sm):.0f} min {min(sm):.0f} MHz  "
          f"power median {np.median(pw):.0f} max {max(pw):.0f} W  power-cap samples {cap}/{len(win)}",
          flush=True)
proc.terminate()
