"""Diagnostic: PCG batch time with fixed vs shifted buffer addresses."""
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
A = eng.assemble()
op = PcgOperator(A, "ldp")
n, kp = op.n, 64
dev = A.val.device
big = torch.empty(int(6.0e9), dtype=torch.uint8, device=dev)  # one arena: place buffers by hand
wsb = N.lib.hf_pcg_workspace_bytes(n, kp, op.Ac.nnz)
nb = n * kp * 8


def run(shift_x, shift_ws):
    base = big.data_ptr()
    off_b = 0
    off_x = ((nb + 4096 + shift_x) // 256) * 256
    off_ws = off_x + ((nb + 4096 + shift_ws) // 256) * 256
    Bb = big[off_b:off_b + nb].view(torch.float64).view(n, kp)
    Bb.zero_()
    Bb[:, :64] = eng.Bd[:, :64]
    X = big[off_x:off_x + nb].view(torch.float64).view(n, kp)
    ws = big[off_ws:off_ws + wsb]
    it = np.zeros(kp, np.int32); st = np.zeros(kp, np.int32); bi = np.zeros(kp, np.int32)
    tr = np.zeros(kp); br = np.zeros(kp)
    P = N.C.c_void_p
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    N.check("pcg", N.lib.hf_pcg_multi(N.C.byref(op.Ac.struct), N.ptr(op.d), N.ptr(Bb), n, kp, 1e-8,
                                      6002, None, N.ptr(X), P(it.ctypes.data), P(st.ctypes.data),
                                      P(tr.ctypes.data), P(br.ctypes.data), P(bi.ctypes.data),
                                      N.ptr(ws), ws.numel(), N.stream_handle()))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), int(it.max())


for sx, sw in [(0, 0)] * 4 + [(4096, 0), (0, 4096), (65536, 65536), (1 << 20, 0), (0, 1 << 21),
                              (3 << 20, 5 << 20), (0, 0), (0, 0)]:
    ms, its = run(sx, sw)
    print(f"shift_x {sx:>8d} shift_ws {sw:>8d}: {ms:7.1f} ms  ({its} iterations, {ms / its:.3f} ms/round)",
          flush=True)
