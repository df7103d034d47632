"""Does a cheap per-column proxy predict PCG iteration counts (so long columns could
be handed out first)?  C3 (MEG) columns: iterations vs the Rayleigh quotient
b'Ab / b'Db and vs ||b||_2 / ||b||_inf.  Diagnostics only."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_07717_b200 import meg, synthetic  # noqa: E402
from paper_1811_07717_b200.device import PcgOperator  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig, solve_block  # noqa: E402


def spearman(a, b):
    ra, rb = np.argsort(np.argsort(a)), np.argsort(np.argsort(b))
    return float(np.corrcoef(ra, rb)[0, 1])


prob = synthetic.eeg_problem("c2", device=True, with_G=False)
eng = meg.MegEngine(prob.mesh, meg.helmet_306(), prob.sources, PcgConfig(1e-8))
A = eng.assemble()
S = eng.rhs()
op = PcgOperator(A, "ldp")
T, info = solve_block(op, S, eng.cfg)
its = info.iterations.astype(float)
At = torch.sparse_csr_tensor(A.indptr.long(), A.indices.long(), A.val, size=A.shape)
AS = (At @ S)
num = (S * AS).sum(0)
den = (S * S * op.d[:, None]).sum(0)
rq = (num / den).cpu().numpy()
nrm = (S.norm(dim=0) / S.abs().max(dim=0).values).cpu().numpy()
print("iterations", its.min(), its.max(), "by sensor type (mag, grad1, grad2):",
      [float(its[k::3].mean()) for k in range(3)])
print("spearman(iters, rayleigh)", spearman(its, rq), " spearman(iters, l2/linf)", spearman(its, nrm))
order = np.argsort(rq)
print("first columns by rayleigh:", its[order[:10]], " last:", its[order[-10:]])
