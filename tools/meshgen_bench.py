"""generate_mesh on the device at the bench's head-model sizes.

The 4-shell sphere segmentation of experiments.py:64-66 (icosphere
subdivisions 3, 1280 triangles per shell) meshed at h = 1.5 mm (C2, ~1.0M
nodes) and at coarser h.  CUDA-event time of generate_mesh_device (grid,
two hf_locate passes, compaction, priorities) plus the host TetMesh copy,
and a CPU figure: the oracle's vectorised numpy locate (the reference's own
algorithm, geometry.py:186-249) on a bounded sample of the same centroids,
one thread, extrapolated per point.  Prints one JSON line per h.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_07717_b200 import meshgen  # noqa: E402
from paper_1811_07717_b200.geometry import layered_sphere_segmentation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--h", type=float, nargs="+", default=[0.004, 0.0015])
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--cpu-sample", type=int, default=4000)
args = ap.parse_args()

seg = layered_sphere_segmentation((0.079, 0.082, 0.087, 0.092), (0.33, 1.79, 0.0064, 0.43),
                                  (2, 1, 0, 3), (0,), 3)
for h in args.h:
    g = meshgen.generate_mesh_device(seg, h)  # warm-up (tables, allocator)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g = meshgen.generate_mesh_device(seg, h)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t0 = time.perf_counter()
    mesh = g.to_mesh()
    host_ms = (time.perf_counter() - t0) * 1e3
    # locate-only device time on all candidate centroids of the grid
    lo, hi = seg.bounding_box()
    nx, ny, nz = (int(v) for v in np.maximum(1, np.ceil((hi - lo) / h - 1e-12).astype(int)))
    out = {"h": h, "grid": [nx, ny, nz], "candidates": 6 * nx * ny * nz, "n_nodes": mesh.n_nodes,
           "n_elements": mesh.n_elements, "device_ms": round(float(np.median(ts)), 2),
           "steps_ms": [round(t, 2) for t in ts], "host_tetmesh_ms": round(host_ms, 1)}
    if args.cpu_sample:
        import oracle.meshgen as OM
        from threadpoolctl import threadpool_limits

        parts = [([(s.nodes, s.triangles) for s in c.surfaces], c.conductivity, c.priority)
                 for c in seg.compartments]
        rng = np.random.default_rng(0)
        pts = mesh.centroids()[rng.choice(mesh.n_elements, args.cpu_sample, replace=False)]
        with threadpool_limits(1):
            t0 = time.perf_counter()
            OM.locate(parts, pts)
            dt = time.perf_counter() - t0
        per_pt = dt / args.cpu_sample
        # generate_mesh locates every candidate centroid and every used node
        est = per_pt * (out["candidates"] + mesh.n_nodes)
        out["cpu_locate"] = {"kind": "port", "cores": 1, "sample_points": args.cpu_sample,
                             "us_per_point": round(per_pt * 1e6, 2), "est_generate_mesh_s": round(est, 1)}
    print(json.dumps(out), flush=True)
