"""Time hf_eit_sens alone (CUDA events) at C4 size: C2 mesh, 5,000 DOFs over the two
inner compartments, L = 64 electrode columns, P = 32 patterns (random T and U:
the kernel's cost does not depend on the values).  ncu target.

    python tools/eit_sens_probe.py [--reps 5]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_07717_b200 import _native as N, synthetic  # noqa: E402
from paper_1811_07717_b200.fem import DeviceMesh  # noqa: E402
from paper_1811_07717_b200.leadfield import build_dof_map  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--P", type=int, default=32)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    mesh = synthetic.sphere_mesh(synthetic.C2_RADII, synthetic.C2_COND, 0.0015)
    dofs = build_dof_map(mesh, [0, 1], 5000, seed=2)
    dm = DeviceMesh.of(mesh)
    elems = np.concatenate(dofs.element_sets).astype(np.int32)
    ptr = np.cumsum([0] + [len(e) for e in dofs.element_sets]).astype(np.int32)
    de, dp = torch.from_numpy(elems).cuda(), torch.from_numpy(ptr).cuda()
    g = torch.Generator(device="cuda").manual_seed(1)
    T = torch.randn((mesh.n_nodes, a.L), dtype=torch.float64, device="cuda", generator=g)
    U = torch.randn((mesh.n_nodes, a.P), dtype=torch.float64, device="cuda", generator=g)
    nd = dofs.n_dofs
    Q = torch.empty((a.P, nd, a.L), dtype=torch.float64, device="cuda")
    ws = torch.empty(N.lib.hf_eit_sens_workspace_bytes(len(elems)), dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    times = []
    for r in range(a.reps):
        ev[0].record()
        N.check("hf_eit_sens", N.lib.hf_eit_sens(
            N.ptr(dm.nodes), N.ptr(dm.tetra), N.ptr(de), N.ptr(dp), nd, 0, N.ptr(T), T.stride(0), a.L,
            N.ptr(U), U.stride(0), a.P, N.ptr(Q), N.ptr(ws), ws.numel(), N.stream_handle()))
        ev[1].record()
        torch.cuda.synchronize()
        times.append(ev[0].elapsed_time(ev[1]))
    E = len(elems)
    flops = 2.0 * a.P * a.L * 4 * E + 2.0 * 16 * a.P * E
    t = float(np.median(times))
    print(f"hf_eit_sens: {E} DOF elements, L={a.L}, P={a.P}: {t:.2f} ms median of {times} "
          f"({flops / t / 1e9:.2f} TFLOP/s DMMA-shaped work)")


if __name__ == "__main__":
    main()
