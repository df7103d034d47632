"""Where the drop-in e2e leg's host time goes: headfem.leadfield.eeg_leadfield(sys)
after install(headfem) at C2, under cProfile (diagnostics only; needs baseline/_ref)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_07717_b200 import synthetic  # noqa: E402
from paper_1811_07717_b200.solver import PcgConfig  # noqa: E402


class A:
    steps = 1


prob = synthetic.eeg_problem("c2", device=True)
cfg = PcgConfig(1e-8)
r = bench.e2e_dropin(A, prob, cfg, 128)
print("drop-in ms/step", r["ms_per_step"], flush=True)
hf = bench._import_reference()
import paper_1811_07717_b200 as eng  # noqa: E402

# rebuild the reference system once more and profile one call
eng.install(hf)
import scipy.sparse as sp  # noqa: E402

from paper_1811_07717_b200 import model  # noqa: E402
from paper_1811_07717_b200.topology import assemble_Gt_device  # noqa: E402

m = prob.mesh
rmesh = hf.meshgen.TetMesh(m.nodes, m.tetra, m.labels, m.sigma)
rmesh._boundary = m.boundary_triangles()
rel = hf.fem.ElectrodeSet(rmesh, list(prob.electrodes.triangle_ids), prob.electrodes.impedances)
Am = hf.fem.assemble_A(rmesh, rel)
B, C, R = hf.fem.assemble_B_C_R(rmesh, rel)
G = sp.csr_matrix(assemble_Gt_device(m, prob.sources).to_scipy().T)
sysm = hf.fem.CemSystem(mesh=rmesh, electrodes=rel, A=Am, B=B, C=C, R=R,
                        ground=model.ground_node(m, prob.electrodes), G=G, source_space=prob.sources)
rcfg = hf.solver.PcgConfig(tolerance=1e-8)
hf.leadfield.eeg_leadfield(sysm, rcfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
hf.leadfield.eeg_leadfield(sysm, rcfg)
torch.cuda.synchronize()
pr.disable()
print("profiled call ms", (time.perf_counter() - t0) * 1e3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
