"""Two column groups solved concurrently on two streams (two host threads) vs one
streamed solve of all columns: does a second solve fill the first one's
inter-kernel gaps and reduction tails?  (experiment; run on the GPU box)"""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.device import PcgOperator  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig, _run_batch, solve_block  # noqa: E402


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
    torch.cuda.set_device(0)
    prob = synthetic.eeg_problem(cfgname, device=True)
    eng = EegEngine(prob.mesh, prob.electrodes, prob.G, B=prob.B, C=prob.C, R=prob.R)
    op = PcgOperator(eng.assemble(), "ldp")
    cfg = PcgConfig(tolerance=1e-8)
    Bd = eng.Bd.contiguous()
    n, k = Bd.shape
    mi = int(cfg.resolve_max_iterations(n))
    kp = 64
    halves = [Bd[:, :kp].contiguous(), Bd[:, kp:2 * kp].contiguous()]

    def seq():
        torch.cuda.synchronize()
        t = time.perf_counter()
        X, info = solve_block(op, Bd[:, :2 * kp].contiguous(), cfg)
        torch.cuda.synchronize()
        return time.perf_counter() - t, X

    def par():
        streams = [torch.cuda.Stream() for _ in range(2)]
        out = [None, None]

        def work(i):
            with torch.cuda.stream(streams[i]):
                out[i] = _run_batch(op, halves[i], cfg.tolerance, mi)[0]
                streams[i].synchronize()

        torch.cuda.synchronize()
        t = time.perf_counter()
        th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        torch.cuda.synchronize()
        return time.perf_counter() - t, torch.cat(out, dim=1)

    for rep in range(3):
        ts, Xs = seq()
        tp, Xp = par()
        same = bool(torch.equal(Xs, Xp))
        print(f"{cfgname} rep {rep}: streamed {2 * kp} cols {ts * 1e3:.1f} ms, two concurrent batches "
              f"{tp * 1e3:.1f} ms, bitwise equal {same}", flush=True)


if __name__ == "__main__":
    main()
