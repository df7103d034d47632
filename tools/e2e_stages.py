"""Stage times of the e2e-from-raw-arrays leg (bench.py e2e_from_arrays): mesh
view, device boundary faces, electrodes, engine construction (mesh upload, B/C/R,
ground, G'), build, LF to host.  Wall clock with synchronize; diagnostics only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_07717_b200 import model, synthetic  # noqa: E402
from paper_1811_07717_b200.device import to_host  # noqa: E402
from paper_1811_07717_b200.engine import EegEngine  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402

prob = synthetic.eeg_problem("c2", device=True)
nodes, tetra, sigma = prob.mesh.nodes, prob.mesh.tetra, prob.mesh.sigma
tri_ids, imp = prob.electrodes.triangle_ids, prob.electrodes.impedances
src_ids = np.asarray(prob.sources.element_ids)
cfg = PcgConfig(1e-8)


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for rep in range(3):
    mesh, a = t(lambda: model.MeshArrays(nodes, tetra, sigma))
    _, b = t(mesh.boundary_triangles)
    el, c = t(lambda: model.ElectrodeSet(mesh, tri_ids, imp))
    src = model.SourceSpace(positions=np.empty((len(src_ids), 3)), orientations=None, element_ids=src_ids,
                            mode="unconstrained")
    eng, d = t(lambda: EegEngine(mesh, el, src, cfg))
    LF, e = t(lambda: eng.build())
    _, f = t(lambda: to_host(LF.contiguous()))
    print(f"view {a:.1f}  boundary(+mesh upload) {b:.1f}  electrodes {c:.1f}  engine {d:.1f}  build {e:.1f}  "
          f"LF->host {f:.1f}  total {a + b + c + d + e + f:.1f} ms", flush=True)
