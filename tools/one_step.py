"""One bench step (C2 LF build, or C3 / C4) between cudaProfilerStart/Stop, after a
warm-up step: the target of the ncu launch list (`--profile-from-start off`)
whose per-kernel shares go to profiles/ (tools/launch_shares.py).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \\
        --csv --log-file gpurun_out/launches.csv python tools/one_step.py [--config c2|c3|c4|c5]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    from paper_1811_07717_b200 import synthetic
    from paper_1811_07717_b200.solver import PcgConfig

    cfg = PcgConfig(1e-8)
    if a.config in ("c2", "c5"):
        from paper_1811_07717_b200.engine import EegEngine

        prob = synthetic.eeg_problem(a.config, device=True)
        eng = EegEngine(prob.mesh, prob.electrodes, prob.G, cfg, prob.B, prob.C, prob.R)
        step = eng.build
    elif a.config == "c3":
        from paper_1811_07717_b200 import meg

        prob = synthetic.eeg_problem("c2", device=True, with_G=False)
        eng = meg.MegEngine(prob.mesh, meg.helmet_306(), prob.sources, cfg)
        step = eng.build
    else:  # c4: EIT lead field on the C2 mesh
        from paper_1811_07717_b200 import model
        from paper_1811_07717_b200.fem import assemble_A
        from paper_1811_07717_b200.leadfield import adjacent_pair_patterns, build_dof_map, eit_leadfield
        from paper_1811_07717_b200.topology import electrodes_from_centers

        mesh = synthetic.sphere_mesh(synthetic.C2_RADII, synthetic.C2_COND, 0.0015)
        el = electrodes_from_centers(mesh, synthetic.fibonacci_sphere_points(64, 0.092), 0.012, 1e3)
        dofs = build_dof_map(mesh, [0, 1], 5000, seed=2)
        B, C, R = model.assemble_B_C_R(mesh, el)
        sysm = model.CemSystem(mesh=mesh, electrodes=el, A=assemble_A(mesh, el), B=B, C=C, R=R,
                               ground=model.ground_node(mesh, el))
        I = adjacent_pair_patterns(64)[:, :32]

        def step():
            return eit_leadfield(sysm, dofs, I, cfg)
    step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    out = step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    m = out.matrix if hasattr(out, "matrix") else out
    print("step done", tuple(m.shape), bool(np.isfinite(np.asarray(m.cpu() if torch.is_tensor(m) else m)).all()))


if __name__ == "__main__":
    main()
