"""Run a few PCG rounds of the C2 system at one batch width (ncu target).

    python tools/pcg_round_probe.py [--config c2] [--kp 64] [--rounds 8]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_07717_b200 import _native as N, synthetic  # noqa: E402
from paper_1811_07717_b200.device import PcgOperator  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--kp", type=int, default=64)
    ap.add_argument("--rounds", type=int, default=8)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    prob = synthetic.eeg_problem(a.config, device=True)
    eng = EegEngine(prob.mesh, prob.electrodes, prob.G, B=prob.B, C=prob.C, R=prob.R)
    op = PcgOperator(eng.assemble(), "ldp")
    lens = torch.diff(op.Ac.indptr.long()).cpu().numpy()
    import numpy as np
    h = np.bincount(lens)
    print("SpMM copy row lengths:", {int(k): int(v) for k, v in enumerate(h) if v},
          "rows > 8:", int((lens > 8).sum()))
    Bb = eng.Bd[:, :a.kp].contiguous()
    X = torch.empty_like(Bb)
    ws = torch.empty(N.lib.hf_pcg_workspace_bytes(op.n, a.kp, op.Ac.nnz), dtype=torch.uint8, device="cuda")
    ms = (N.C.c_float * 3)()
    f = N.C.c_int32(0)
    N.check("prof", N.lib.hf_pcg_profile(N.C.byref(op.Ac.struct), N.ptr(op.d), N.ptr(Bb), op.n, a.kp,
                                         a.rounds, N.ptr(X), ms, N.C.byref(f), N.ptr(ws), ws.numel(),
                                         N.stream_handle()))
    torch.cuda.synchronize()
    print("ms", [round(float(v), 4) for v in ms])


if __name__ == "__main__":
    main()
