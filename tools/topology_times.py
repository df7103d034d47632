"""Times of the device topology builders at C2 (vs the host numpy mirrors)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1811_07717_b200 import model, synthetic  # noqa: E402
from paper_1811_07717_b200.fem import DeviceMesh  # noqa: E402
from paper_1811_07717_b200.topology import assemble_Gt_device, boundary_triangles_device  # noqa: E402

mesh = synthetic.sphere_mesh(synthetic.C2_RADII, synthetic.C2_COND, 0.0015)
DeviceMesh.of(mesh)
src = model.place_sources(mesh, [0], 10_000, seed=1)
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    f, o = boundary_triangles_device(mesh)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    Gt = assemble_Gt_device(mesh, src)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"device: boundary_triangles {1e3 * (t1 - t):.1f} ms ({len(f)} faces), "
          f"assemble_G {1e3 * (t2 - t1):.1f} ms (G' {Gt.shape}, nnz {Gt.nnz})", flush=True)
t = time.perf_counter()
mesh._boundary = None
mesh.boundary_triangles()
t1 = time.perf_counter()
model.assemble_G(mesh, src)
t2 = time.perf_counter()
print(f"host numpy mirror: boundary_triangles {t1 - t:.2f} s, assemble_G {t2 - t1:.2f} s")
