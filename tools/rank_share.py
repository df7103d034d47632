"""Time one rank's share of a sharded LF build on ONE GPU (no collectives).

Only one GPU is reachable this round, so the N-GPU strong-scaling step is
estimated by running rank 0's electrode block (`engine.column_blocks(L, N)[0]`)
alone: assembly + PCG of L/N columns + its response block + its partial LF
(distributed.sharded_leadfield minus the two NCCL exchanges, which move
128 KB and 31 MB at C2).  CUDA-event timing, median of --steps builds.
Prints one JSON line per N.  An estimate, never a bench value.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine, column_blocks  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()

prob = synthetic.eeg_problem(args.config, device=True)
L = prob.electrodes.count
for N in args.n:
    blk = column_blocks(L, N)[0]
    eng = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-8), prob.B, prob.C, prob.R,
                    columns=blk)
    W = np.eye(L)  # stands in for -R M^-1 (built from the all-gathered M on a real run)

    def rank_step():  # distributed.sharded_leadfield minus its two NCCL exchanges
        A = eng.assemble()
        T = eng.solve(A)
        eng.response_block(T).cpu()
        return eng.lf_partial(T, W)

    rank_step()  # warm-up (graph capture, workspace)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rank_step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    it = eng.last_info.iterations
    print(json.dumps({"config": args.config, "n_gpus_emulated": N, "columns": list(blk),
                      "rank0_build_ms": round(ms, 2), "steps_ms": [round(t, 2) for t in ts],
                      "est_rhs_solves_per_s": round(L / (ms * 1e-3), 2),
                      "iterations": [int(it.min()), int(it.max())]}), flush=True)
    del eng
    torch.cuda.empty_cache()
