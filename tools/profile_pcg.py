"""Short driver for ncu: build the C1/C2 system on the device and run a few PCG
rounds through hf_pcg_profile (k_spmm / k_update_r / k_update_p, k_update_xring),
or one full LF build (--build).  Never used for timing numbers."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--build", action="store_true")
args = ap.parse_args()
prob = synthetic.eeg_problem(args.config, device=True)
eng = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-8), prob.B, prob.C, prob.R)
A = eng.assemble()
if args.build:
    eng.build()
else:
    import bench

    print(bench.kernel_roofline(eng.Bd, A, rounds=args.rounds, config=args.config))
torch.cuda.synchronize()
print("done")
