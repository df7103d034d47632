"""SpMM/PCG round time at C2 under different node orderings (experiment).

The SpMM's bytes through L1 depend on how many of a row's 7 gathered p rows a
tile already touched.  This permutes the C2 matrix symmetrically (P A P') by a
few orderings of the grid nodes and times one PCG round per kernel with
hf_pcg_profile (CUDA events), kp = 64/32/16.
"""
import json
import sys
import time

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1811_07717_b200 import _native as N, synthetic  # noqa: E402
from paper_1811_07717_b200.device import DeviceCsr, PcgOperator  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402


def part1by2(v):
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
    return v


def grid_index(nodes, h):
    lo = nodes.min(axis=0)
    return np.rint((nodes - lo) / h).astype(np.int64)


def orders(nodes, h):
    g = grid_index(nodes, h)
    out = {"identity": np.arange(len(nodes))}
    m = part1by2(g[:, 0]) | (part1by2(g[:, 1]) << np.uint64(1)) | (part1by2(g[:, 2]) << np.uint64(2))
    out["morton"] = np.argsort(m, kind="stable")
    for bx, by, bz in ((4, 4, 2), (8, 4, 1), (8, 2, 2), (4, 4, 4), (16, 2, 1)):
        key = ((g[:, 2] // bz) * 10**12 + (g[:, 1] // by) * 10**8 + (g[:, 0] // bx)) * 10**6 \
            + (g[:, 2] % bz) * 10**4 + (g[:, 1] % by) * 10**2 + (g[:, 0] % bx)
        out[f"brick{bx}x{by}x{bz}"] = np.argsort(key, kind="stable")
    # bricks in x-fastest order of brick columns but brick-major in y-z slabs
    return out


def main():
    torch.cuda.set_device(0)
    prob = synthetic.eeg_problem("c2", device=True)
    eng = EegEngine(prob.mesh, prob.electrodes, prob.G, B=prob.B, C=prob.C, R=prob.R)
    A = eng.assemble().to_scipy()
    nodes = prob.mesh.nodes
    B = eng.Bd
    res = {}
    for name, perm in orders(nodes, 0.0015).items():
        Ap = A[perm][:, perm].tocsr()
        Ap.sort_indices()
        dA = DeviceCsr.from_scipy(Ap)
        op = PcgOperator(dA, "ldp")
        row = {}
        for kp in (64, 32, 16):
            Bb = torch.zeros((op.n, kp), dtype=torch.float64, device="cuda")
            Bb[:, :] = B[torch.from_numpy(perm).cuda()][:, :kp]
            X = torch.empty_like(Bb)
            ws = torch.empty(N.lib.hf_pcg_workspace_bytes(op.n, kp, op.Ac.nnz), dtype=torch.uint8, device="cuda")
            best = None
            for rep in range(3):
                ms = (N.C.c_float * 3)()
                f = N.C.c_int32(0)
                N.check("prof", N.lib.hf_pcg_profile(N.C.byref(op.Ac.struct), N.ptr(op.d), N.ptr(Bb), op.n, kp, 24,
                                                     N.ptr(X), ms, N.C.byref(f), N.ptr(ws), ws.numel(),
                                                     N.stream_handle()))
                t = [round(float(v), 4) for v in ms]
                if best is None or sum(t) < sum(best):
                    best = t
            row[kp] = best
            del ws, X, Bb
        res[name] = row
        print(name, json.dumps(row), flush=True)
    with open("gpurun_out/order_experiment.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
