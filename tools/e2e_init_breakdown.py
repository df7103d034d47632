"""Timers around each step of EegEngine.__init__ from host arrays (the e2e leg's
fixed cost on top of the device build)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import torch  # noqa: E402

from paper_1811_07717_b200 import model, synthetic  # noqa: E402
from paper_1811_07717_b200.device import DeviceCsr  # noqa: E402
from paper_1811_07717_b200.fem import DeviceMesh  # noqa: E402
from paper_1811_07717_b200.solver import rhs_block  # noqa: E402
from paper_1811_07717_b200.topology import assemble_Gt_device  # noqa: E402

prob = synthetic.eeg_problem("c2", device=True)
mesh, el, B, C = prob.mesh, prob.electrodes, prob.B, prob.C
dev = torch.device("cuda", 0)
for rep in range(3):
    ts = []

    def mark(name):
        torch.cuda.synchronize()
        ts.append((name, time.perf_counter()))

    mark("start")
    t32 = np.array(mesh.tetra, dtype=np.int32, order="C")
    mark("tetra->int32 (host)")
    dm = DeviceMesh(mesh.nodes, mesh.tetra, dev)
    mark("DeviceMesh (convert+H2D)")
    sig = torch.from_numpy(np.array(mesh.sigma, dtype=np.float64, order="C")).to(dev)
    mark("sigma H2D")
    g = model.ground_node(mesh, el)
    mark("ground_node")
    tri, coef = model.electrode_contacts(el)
    mark("electrode_contacts")
    Bd = rhs_block(sp.csc_matrix(B)[:, 0:B.shape[1]], dev=dev)
    mark("rhs_block")
    Bt = DeviceCsr.from_scipy(sp.csr_matrix(sp.csr_matrix(B).T), dev)
    mark("B' CSR")
    Gt = assemble_Gt_device(mesh, prob.sources)
    mark("G' device")
    print(" | ".join(f"{n} {1e3 * (t - ts[i][1]):.1f}" for i, (n, t) in enumerate(ts[1:])), flush=True)
