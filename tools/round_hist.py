"""Diagnostic: distribution of per-kernel times over many PCG rounds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_07717_b200 import _native as N  # noqa: E402
from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.device import PcgOperator  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

prob = synthetic.eeg_problem("c2")
eng = EegEngine(prob.mesh, prob.electrodes, prob.G, PcgConfig(1e-8), prob.B, prob.C, prob.R)
op = PcgOperator(eng.assemble(), "ldp")
n, kp = op.n, 64
Bb = eng.Bd[:, :64].contiguous()
X = torch.empty_like(Bb)
ws = torch.empty(N.lib.hf_pcg_workspace_bytes(n, kp, op.Ac.nnz), dtype=torch.uint8, device=Bb.device)
ms = (N.C.c_float * 3)()
fused = N.C.c_int32(0)
res = []
for rep in range(40):
    N.check("p", N.lib.hf_pcg_profile(N.C.byref(op.Ac.struct), N.ptr(op.d), N.ptr(Bb), n, kp, 20,
                                      N.ptr(X), ms, N.C.byref(fused), N.ptr(ws), ws.numel(),
                                      N.stream_handle()))
    res.append(list(ms))
r = np.array(res)
for k, name in enumerate(["spmm", "update_r", "update_xp"]):
    print(f"{name}: min {r[:, k].min():.3f} median {np.median(r[:, k]):.3f} max {r[:, k].max():.3f} ms")
tot = r.sum(axis=1)
print("round per 20-round block:", " ".join(f"{t:.3f}" for t in tot))
