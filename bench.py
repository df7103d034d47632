#!/usr/bin/env python
"""bench.py — the BASELINE.json metric on config C2.

Workload ("c2"): 1,001,184-node 4-compartment concentric-sphere Kuhn mesh
(h = 1.5 mm, radii 79/82/87/92 mm), 128 electrodes, 10k unconstrained dipole
sources (G: n x 30,000), PCG tolerance 1e-8, max_iter = 5 sqrt(n) + 1000.
One step = one EEG lead-field build on the device from resident mesh arrays:
P1 assembly -> LDP preconditioner -> multi-RHS PCG for all 128 electrodes ->
M = C - B'T -> W = -R M^-1 -> LF = W (G'T)'.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric: RHS-solves/s (electrode transfer columns per second of LF build,
whole job), with the LF build time as ms_per_step and the SpMM/PCG kernels'
achieved HBM GB/s against the measured copy peak.  For N > 1 (torchrun) the
electrode columns are sharded over ranks (strong scaling: the problem is
fixed) and the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "LF build time & PCG RHS-solves/sec on 1M-node mesh; SpMM HBM GB/s vs peak"
UNIT = "RHS-solves/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload_config(prob, cfg):
    return eeg_config(prob.name, prob.mesh.n_nodes, prob.mesh.n_elements, len(np.unique(prob.mesh.labels)),
                      prob.electrodes.count, prob.sources.n_sources, cfg.tolerance)


def eeg_config(name, n_nodes, n_elements, ncomp, L, S, tol):
    """The `config` object of an EEG line; both arms print the same one."""
    return {"workload": f"{name}: {n_nodes:,}-node {ncomp}-compartment sphere Kuhn mesh, "
                        f"{L}-electrode EEG lead field, {S:,} dipole sources",
            "config": name, "n_nodes": int(n_nodes), "n_elements": int(n_elements), "electrodes": int(L),
            "sources": int(S), "lf_shape": [int(L), 3 * int(S)], "tolerance": tol, "precision": "fp64",
            "l2_policy": "inputs larger than L2 (n x 64 fp64 vector blocks = 512 MB each)"}


# sources of the EEG configs (synthetic.eeg_problem)
SOURCES = {"c1": 1000, "c2": 10_000, "c5": 50_000}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples (200 ms) during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = str(index)
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8 or parts[0] != self.index:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- our arm
def _nnz(A):
    return int(A.nnz) if hasattr(A, "nnz") else int(A.indices.numel())


def survey_round(n, nnz_stored, kp, round_ms, peak):
    """bytes_per_rhs_iter(k) = 80 n + (12 nnz + 4 (n+1) + 16 n) / k."""
    per = 80 * n + (12 * nnz_stored + 4 * (n + 1) + 16 * n) / kp
    gbs = per * kp / (round_ms * 1e-3) / 1e9
    return {"bytes_per_rhs_iter": round(per, 1), "nnz_stored": nnz_stored, "equivalent_gbs": round(gbs, 1),
            "equivalent_frac": round(gbs / peak, 4),
            "note": "the model's bytes / the measured round time; above 1 because the round moves fewer bytes "
                    "(x deferred over 8 rounds, explicit zeros pruned): see pcg_round.frac for the bytes moved"}


def kernel_roofline(Bd, A, rounds=24, config="c2"):
    """Per-kernel CUDA-event timing of a PCG round at the bench's batch width,
    algorithmic bytes per launch, fraction of the HBM peak."""
    import torch

    from paper_1811_07717_b200 import _native as N
    from paper_1811_07717_b200.device import PcgOperator, width_for
    from paper_1811_07717_b200.solver import MAX_BATCH

    op = PcgOperator(A, "ldp")
    n = op.n
    kp = width_for(op.batch_width(Bd.shape[1], MAX_BATCH))  # the solver's own batch width
    Bb = torch.zeros((n, kp), dtype=torch.float64, device=Bd.device)
    k = min(kp, Bd.shape[1])
    Bb[:, :k] = Bd[:, :k]
    X = torch.empty_like(Bb)
    ws = torch.empty(N.lib.hf_pcg_workspace_bytes(n, kp, op.Ac.nnz), dtype=torch.uint8, device=Bb.device)
    flags = N.C.c_int32(0)
    reps = []
    for _ in range(3):  # three profiles of `rounds` rounds each: the median per kernel
        ms3 = (N.C.c_float * 3)()
        N.check("hf_pcg_profile", N.lib.hf_pcg_profile(
            N.C.byref(op.Ac.struct), N.ptr(op.d), N.ptr(Bb), n, kp, rounds, N.ptr(X), ms3,
            N.C.byref(flags), N.ptr(ws), ws.numel(), N.stream_handle()))
        reps.append([float(v) for v in ms3])
    ms = np.median(np.array(reps), axis=0)
    nnz = op.Ac.nnz
    xd = max(1, flags.value >> 8)
    # SURVEY.md §8d per launch: the SpMM reads p and the CSR (8 B value + 4 B index
    # per entry, row pointers) and writes q; the r update reads r, q, dd and writes r;
    # the p update reads p, r, dd and writes p, except every xd-th round, which also
    # reads and writes x and reads the xd ring slots (averaged per round)
    algo = {"k_spmm": 16 * n * kp + 12 * nnz + 4 * (n + 1),
            "k_update_r": 24 * n * kp + 16 * n,
            "k_update_pxring": ((xd - 1) * 24 + 32 + 8 * xd) * n * kp // xd + 16 * n}
    times = dict(zip(algo, [float(ms[0]), float(ms[1]), float(ms[2])]))
    peak, peak_kind = peaks()
    kern = {name: {"ms": times[name], "bytes": algo[name],
                   "gbs": algo[name] / (times[name] * 1e-3) / 1e9} for name in algo}
    total_ms = sum(times.values())
    total_bytes = sum(algo.values())
    dominant = max(times, key=times.get)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as f:
                traffic = json.load(f).get(config, {}).get(f"{dominant}<{kp}>")
        except Exception:
            traffic = None
    ach = kern[dominant]["gbs"]
    return {"bound": "hbm", "kernel": f"{dominant}<{kp}>", "achieved": round(ach, 1),
            "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(ach / peak, 4),
            "traffic": traffic,
            "traffic_source": "profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per launch from "
                              "one ncu --set full capture of these kernels (tools/refresh_profiles.sh ncu)",
            "algorithmic_bytes_per_launch": algo[dominant],
            "launch_ms": round(times[dominant], 4),
            "share_of_round": round(times[dominant] / total_ms, 3),
            "pcg_round": {"kp": kp, "n": n, "nnz_spmm": nnz, "x_deferral": xd,
                          "ms": round(total_ms, 4),
                          "bytes": total_bytes,
                          "gbs": round(total_bytes / (total_ms * 1e-3) / 1e9, 1),
                          "frac": round(total_bytes / (total_ms * 1e-3) / 1e9 / peak, 4),
                          "bytes_per_rhs_iter": total_bytes / kp,
                          # SURVEY.md §8(d)'s model of the reference recurrence (x, p, r, q
                          # streamed every round; stored CSR incl. explicit zeros), for comparison
                          "survey_model": survey_round(n, _nnz(A), kp, total_ms, peak)},
            "kernels": {k2: {kk: (round(v, 4) if isinstance(v, float) else v) for kk, v in d.items()}
                        for k2, d in kern.items()}}


def cpu_baseline(A, b, iters_per_col, sample_iters=200):
    """The reference's own pcg_solve (baseline/_ref, unmodified; solver.py:64-111)
    on one host core for a bounded sample of one C2 column (max_iterations =
    sample_iters; the ConvergenceError it then raises ends the sample), RHS-solves/s
    extrapolated to the measured iterations per column.  Falls back to the
    oracle's restatement (kind "port") only if baseline/_ref is missing."""
    from threadpoolctl import threadpool_limits

    try:
        _import_reference()
        from headfem.errors import ConvergenceError
        from headfem.solver import PcgConfig, pcg_solve

        def run(k):
            try:
                pcg_solve(A, b, PcgConfig(tolerance=1e-8, max_iterations=k))
            except ConvergenceError:
                pass
        kind, what = "reference", "headfem.solver.pcg_solve (baseline/_ref)"
    except Exception:
        import oracle

        def run(k):
            oracle.pcg_solve(A, b, oracle.PcgSettings(), iterations_cap=k)
        kind, what = "port", "the oracle's pcg_solve restatement"
    with threadpool_limits(1):
        run(3)
        t0 = time.perf_counter()
        run(sample_iters)
        dt = time.perf_counter() - t0
    t_iter = dt / sample_iters
    return {"value": 1.0 / (t_iter * iters_per_col), "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{sample_iters} PCG iterations of electrode column 0 on the bench system through "
                      f"{what} ({t_iter * 1e3:.1f} ms/iteration, 1 thread), extrapolated to "
                      f"{iters_per_col:.0f} iterations per column",
            "ms_per_iteration": round(t_iter * 1e3, 3)}


def e2e_from_arrays(args, prob, cfg, blocks, rank, world, dev, L):
    """The engine's public API from raw host arrays, every step: nodes, tetra and
    sigma, the electrodes' boundary-triangle ids and impedances, the sources'
    element ids.  Inside the timed step: the mesh upload, boundary faces on the
    device, electrodes, ground node, B/C/R, G' on the device, assembly, PCG,
    response, the lead field back to host memory.  Nothing is cached across
    steps (a fresh MeshArrays each step)."""
    import torch
    import torch.distributed as dist

    from paper_1811_07717_b200 import model
    from paper_1811_07717_b200.device import to_host
    from paper_1811_07717_b200.distributed import sharded_leadfield
    from paper_1811_07717_b200.engine import EegEngine

    nodes, tetra, sigma = prob.mesh.nodes, prob.mesh.tetra, prob.mesh.sigma
    tri_ids, imp = prob.electrodes.triangle_ids, prob.electrodes.impedances
    src_ids = np.asarray(prob.sources.element_ids)
    h2d = d2h = 0
    if world > 1:
        dist.barrier(device_ids=[dev.index])
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        mesh = model.MeshArrays(nodes, tetra, sigma)
        el = model.ElectrodeSet(mesh, tri_ids, imp)
        src = model.SourceSpace(positions=np.empty((len(src_ids), 3)), orientations=None,
                                element_ids=src_ids, mode="unconstrained")
        eng = EegEngine(mesh, el, src, cfg, columns=blocks[rank], dev=dev)
        if world == 1:
            lf_host = eng.build(to_host=True)
        else:
            lf_dev = sharded_leadfield(eng, world, rank)
            lf_host = None if lf_dev is None else to_host(lf_dev.contiguous())
        h2d += eng.h2d_bytes
        d2h += 4 * len(mesh.boundary_triangles()[1]) + 8 * L * L
        if lf_host is not None:
            d2h += lf_host.nbytes
        del eng, mesh
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    tt = torch.tensor([wall, h2d, d2h], dtype=torch.float64, device=dev)
    if world > 1:
        mx = tt[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        tt[0] = mx[0]
    wall, h2d, d2h = (float(v) for v in tt.tolist())
    return {"value": L * args.steps / wall, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
            "ms_per_step": round(wall * 1e3 / args.steps, 2),
            "api": "EegEngine(MeshArrays(nodes, tetra, sigma), ElectrodeSet(triangle ids), "
                   "SourceSpace(element ids)).build(to_host=True): mesh upload, device boundary faces, "
                   "B/C/R, device G', assembly, PCG and LF inside every step"}


def e2e_dropin(args, prob, cfg, L):
    """The drop-in: the reference's own entry point headfem.leadfield.eeg_leadfield(sys)
    (leadfield.py:122-134) after install(headfem), on the unmodified reference
    installed in baseline/_ref.  sys is the reference's CemSystem with host scipy
    A, B, C, G (built once, outside the timed region, from the same arrays); every
    timed call moves them to the device, solves, and returns the LeadField in host
    memory."""
    import torch

    try:
        hf = _import_reference()
    except Exception as exc:  # baseline/_ref missing
        log(f"[e2e] drop-in leg skipped: {exc}")
        return None
    import scipy.sparse as sp

    import paper_1811_07717_b200 as eng
    from paper_1811_07717_b200 import model
    from paper_1811_07717_b200.topology import assemble_Gt_device

    eng.install(hf)
    try:
        m = prob.mesh
        rmesh = hf.meshgen.TetMesh(m.nodes, m.tetra, m.labels, m.sigma)
        rmesh._boundary = m.boundary_triangles()  # device faces, bit-exact with meshgen.py:114-130
        rel = hf.fem.ElectrodeSet(rmesh, list(prob.electrodes.triangle_ids), prob.electrodes.impedances)
        A = hf.fem.assemble_A(rmesh, rel)         # the engine (installed)
        B, C, R = hf.fem.assemble_B_C_R(rmesh, rel)
        G = sp.csr_matrix(assemble_Gt_device(m, prob.sources).to_scipy().T)
        sysm = hf.fem.CemSystem(mesh=rmesh, electrodes=rel, A=A, B=B, C=C, R=R,
                                ground=model.ground_node(m, prob.electrodes), G=G,
                                source_space=prob.sources)
        rcfg = hf.solver.PcgConfig(tolerance=cfg.tolerance)
        hf.leadfield.eeg_leadfield(sysm, rcfg)   # warm-up
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            lf = hf.leadfield.eeg_leadfield(sysm, rcfg)
        wall = time.perf_counter() - w0
        assert isinstance(lf.matrix, np.ndarray) and lf.matrix.shape == (L, G.shape[1])
    finally:
        eng.uninstall()
    h2d = (4 * (A.shape[0] + 1) + 12 * A.nnz + 20 * B.nnz + 12 * B.nnz + 4 * (L + 1)
           + 8 * L + 4 * (G.shape[1] + 1) + 12 * G.nnz + 8 * L * L)
    d2h = lf.matrix.nbytes + 8 * L * L
    return {"value": L * args.steps / wall, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(wall * 1e3 / args.steps, 2),
            "api": "headfem.leadfield.eeg_leadfield(sys) after paper_1811_07717_b200.install(headfem) "
                   "(baseline/_ref, unmodified reference); host scipy CemSystem in, LeadField in host "
                   "memory out"}


def run_meg(args):
    """C3 (BASELINE.json configs[2]): the 306-sensor MEG lead field on the C2 mesh
    (paper_1811_07717_b200.meg; parity unpinned, the reference has no MEG).  One
    step = assembly -> S' (hf_meg_rhs) -> 306 PCG solves -> primary field + T'G."""
    import torch

    from paper_1811_07717_b200 import _native as N
    from paper_1811_07717_b200 import meg, model, synthetic
    from paper_1811_07717_b200.solver import PcgConfig

    torch.cuda.set_device(0)
    cfg = PcgConfig(tolerance=1e-8)
    prob = synthetic.eeg_problem("c2", device=True, with_G=False)
    sensors = meg.helmet_306()
    eng = meg.MegEngine(prob.mesh, sensors, prob.sources, cfg)
    for _ in range(args.warmup):
        eng.build()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = N.lib.hf_launch_count()
    with ClockSampler(0) as clocks:
        e0.record()
        for _ in range(args.steps):
            Lf = eng.build()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = N.lib.hf_launch_count() - launches0
    ns = sensors.n_sensors
    roof = kernel_roofline(eng.rhs(), eng.assemble(), config="c3")
    # end to end from host arrays: fresh mesh object, sensors and source ids every step
    w0 = time.perf_counter()
    for _ in range(args.steps):
        mesh = model.MeshArrays(prob.mesh.nodes, prob.mesh.tetra, prob.mesh.sigma)
        e2 = meg.MegEngine(mesh, sensors, prob.sources, cfg)
        lf_host = e2.build(to_host=True)
    wall = (time.perf_counter() - w0) / args.steps
    h2d = prob.mesh.nodes.nbytes + 4 * prob.mesh.tetra.size + prob.mesh.sigma.nbytes + \
        sensors.coils.nbytes + 4 * len(sensors.coil_ptr) + 4 * len(prob.sources.element_ids) + \
        prob.sources.positions.nbytes
    info = eng.last_info
    out = {"metric": METRIC, "value": round(ns / (ms * 1e-3), 3), "unit": UNIT, "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (C2 mesh; Elekta-like 102-site helmet: 102 magnetometers + 204 planar "
                   "gradiometers; volume-weighted random sources)",
           "config": {"workload": f"c3: {prob.mesh.n_nodes:,}-node 4-compartment sphere mesh, {ns}-sensor MEG "
                                  f"lead field, {prob.sources.n_sources:,} dipole sources (parity unpinned: "
                                  "the reference has no MEG, SPEC.md:8)", "config": "c3",
                      "n_nodes": int(prob.mesh.n_nodes), "sensors": ns, "sources": int(prob.sources.n_sources),
                      "lf_shape": list(Lf.shape), "tolerance": cfg.tolerance, "precision": "fp64",
                      "parallelism": "sensor-columns x1"},
           "pcg_iterations": {"min": int(info.iterations.min()), "max": int(info.iterations.max()),
                              "mean": float(np.mean(info.iterations))},
           "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": None,
           "e2e": {"value": ns / wall, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(lf_host.nbytes), "ms_per_step": round(wall * 1e3, 2),
                   "api": "MegEngine(MeshArrays(nodes, tetra, sigma), helmet_306(), sources).build(to_host=True)"},
           "clocks": clocks.summary()}
    print(json.dumps(out), flush=True)


def run_eit(args):
    """C4 (BASELINE.json configs[3]): the linearised EIT lead field on the C2 mesh,
    64 electrodes, 32 adjacent-pair patterns, 5,000 conductivity DOFs.  One step =
    eit_leadfield (leadfield.py:210-237): 64 transfer solves, 32 pattern solves, the
    DMMA sensitivities and the 2,048 x 5,000 Jacobian; RHS-solves/s counts both
    kinds of solves (96 per step)."""
    import torch

    from paper_1811_07717_b200 import _native as N
    from paper_1811_07717_b200 import model, synthetic
    from paper_1811_07717_b200.fem import assemble_A
    from paper_1811_07717_b200.leadfield import adjacent_pair_patterns, build_dof_map, eit_leadfield
    from paper_1811_07717_b200.solver import PcgConfig
    from paper_1811_07717_b200.topology import electrodes_from_centers

    torch.cuda.set_device(0)
    cfg = PcgConfig(tolerance=1e-8)
    mesh = synthetic.sphere_mesh(synthetic.C2_RADII, synthetic.C2_COND, 0.0015)
    el = electrodes_from_centers(mesh, synthetic.fibonacci_sphere_points(64, 0.092), 0.012, 1e3)
    t0 = time.perf_counter()
    dofs = build_dof_map(mesh, [0, 1], 5000, seed=2)
    t_dof = time.perf_counter() - t0
    B, C, R = model.assemble_B_C_R(mesh, el)
    sysm = model.CemSystem(mesh=mesh, electrodes=el, A=assemble_A(mesh, el), B=B, C=C, R=R,
                           ground=model.ground_node(mesh, el))
    I = adjacent_pair_patterns(64)[:, :32]
    for _ in range(args.warmup):
        eit_leadfield(sysm, dofs, I, cfg)
    torch.cuda.synchronize()
    launches0 = N.lib.hf_launch_count()
    with ClockSampler(0) as clocks:
        w0 = time.perf_counter()
        for _ in range(args.steps):
            lf = eit_leadfield(sysm, dofs, I, cfg)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) / args.steps
    launches = N.lib.hf_launch_count() - launches0
    solves = 64 + 32
    out = {"metric": METRIC, "value": round(solves / wall, 3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(wall * 1e3, 2), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (C2 mesh, 64 fibonacci electrodes r = 12 mm, adjacent-pair patterns, "
                   "volume-weighted DOF centres, seed 2)",
           "config": {"workload": "c4: linearised EIT lead field on the 1,001,184-node C2 mesh, 64 electrodes, "
                                  "32 injection patterns, 5,000 conductivity DOFs (4,105,824 DOF elements)",
                      "config": "c4", "lf_shape": list(lf.matrix.shape), "tolerance": cfg.tolerance,
                      "precision": "fp64", "parallelism": "columns x1"},
           "e2e": {"value": round(solves / wall, 3), "unit": UNIT,
                   "h2d_bytes_per_step": int(12 * sysm.A.nnz + 4 * (sysm.A.shape[0] + 1) + 20 * B.nnz),
                   "d2h_bytes_per_step": int(lf.matrix.nbytes),
                   "api": "eit_leadfield(sys, dofs, currents) with host scipy A/B (the drop-in signature)"},
           "build_dof_map_s": round(t_dof, 3), "gpu_launches": int(launches), "clocks": clocks.summary()}
    print(json.dumps(out), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1811_07717_b200 import _native as N
    from paper_1811_07717_b200 import synthetic
    from paper_1811_07717_b200.distributed import init_from_env, sharded_leadfield
    from paper_1811_07717_b200.device import to_host
    from paper_1811_07717_b200.engine import EegEngine, column_blocks
    from paper_1811_07717_b200.solver import PcgConfig

    rank, world, local = init_from_env("nccl")
    dev = torch.device("cuda", local)
    cfg = PcgConfig(tolerance=1e-8)
    t0 = time.time()
    prob = synthetic.eeg_problem(args.config, device=True)  # boundary faces + G' on the device
    log(f"[rank {rank}] problem {prob.mesh} built in {time.time() - t0:.1f}s")
    blocks = column_blocks(prob.electrodes.count, world)

    def make_engine(sources=None):
        return EegEngine(prob.mesh, prob.electrodes, sources if sources is not None else prob.G,
                         cfg, prob.B, prob.C, prob.R, columns=blocks[rank], dev=dev)

    engine = make_engine()

    def step():
        if world == 1:
            return engine.build()
        return sharded_leadfield(engine, world, rank)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    L = prob.electrodes.count
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = N.lib.hf_launch_count()
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            LF = step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = N.lib.hf_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    info = engine.last_info
    value = L * args.steps / (ms * 1e-3)

    # per-kernel roofline right after the timed region (same GPU state), clocks sampled
    roof = None
    A = None
    if rank == 0:
        A = engine.assemble()
        with ClockSampler(local) as rclk:
            roof = kernel_roofline(engine.Bd, A, config=args.config)
        roof["clocks"] = rclk.summary()

    # end to end from host buffers, two ways; the headline `e2e` is the drop-in
    e2e_engine = None if args.no_e2e else e2e_from_arrays(args, prob, cfg, blocks, rank, world, dev, L)
    e2e = None
    if not args.no_e2e and world == 1:
        e2e = e2e_dropin(args, prob, cfg, L)
    if e2e is None:
        e2e = e2e_engine

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Ah = A.to_scipy()
        b = prob.B[:, 0].toarray().ravel()
        cpu = cpu_baseline(Ah, b, float(np.mean(info.iterations)))
    clk = clocks.summary()
    if rank == 0:
        lf_ok = LF is not None and bool(torch.isfinite(LF).all().item())
        out = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 2),
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (analytic-label Kuhn sphere mesh; fibonacci electrodes; "
                       "volume-weighted random sources)",
               "config": {**workload_config(prob, cfg), "parallelism": f"electrode-columns x{world}"},
               "lf_build_ms": round(ms / args.steps, 2),
               "pcg_iterations": {"min": int(info.iterations.min()), "max": int(info.iterations.max()),
                                  "mean": float(np.mean(info.iterations))} if info is not None else None,
               "lf_finite": lf_ok, "gpu_launches": int(launches), "roofline": roof,
               "cpu_baseline": cpu, "e2e": e2e, "e2e_engine": e2e_engine, "clocks": clk}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_REF = {}


def _import_reference():
    """The unmodified reference package installed in baseline/_ref
    (tools/install_reference.sh); nothing of this repo's engine is imported."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import headfem

    if not os.path.abspath(headfem.__file__).startswith(REF_DIR):
        raise RuntimeError(f"headfem resolved to {headfem.__file__}, not baseline/_ref")
    return headfem


def reference_problem(name):
    """The bench workload built with the reference's own API: SURVEY.md App. A.4's
    analytic-label Kuhn sphere (the reference's Kuhn table, corner offsets and
    TetMesh), fibonacci electrodes through ElectrodeSet.from_centers, and the
    stiffness/electrode matrices through assemble_A / assemble_B_C_R.  The arrays
    are the ones paper_1811_07717_b200.synthetic builds for our arm
    (tests/golden/make_fullsize_golden.py checks them array-equal)."""
    _import_reference()
    from headfem.fem import ElectrodeSet, assemble_A, assemble_B_C_R
    from headfem.meshgen import _CORNER_OFFSETS, _KUHN_TETS, TetMesh
    from headfem.simulate import fibonacci_sphere_points

    radii, cond = (0.079, 0.082, 0.087, 0.092), (0.33, 1.79, 0.0064, 0.43)
    h, L, erad = {"c2": (0.0015, 128, 0.01), "c5": (0.00088, 256, 0.006),
                  "c1": (0.004, 32, 0.014)}[name]
    if name == "c1":
        radii, cond = (0.079, 0.086, 0.092), (0.33, 0.0064, 0.43)
    R = radii[-1]
    nx = int(np.ceil(2 * R / h - 1e-12))
    xs = -R + h * np.arange(nx + 1)
    gz, gy, gx = np.meshgrid(xs, xs, xs, indexing="ij")
    grid = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    cz, cy, cx = np.meshgrid(*(np.arange(nx),) * 3, indexing="ij")
    base = (cx + (nx + 1) * (cy + (nx + 1) * cz)).ravel()
    off = _CORNER_OFFSETS[:, 0] + (nx + 1) * (_CORNER_OFFSETS[:, 1] + (nx + 1) * _CORNER_OFFSETS[:, 2])
    tetra = (base[:, None] + off[None, :])[:, _KUHN_TETS].reshape(-1, 4)
    r = np.linalg.norm(grid[tetra].mean(1), axis=1)
    lab = np.full(len(r), -1)
    for k in reversed(range(len(radii))):
        lab[r <= radii[k]] = k
    keep = lab >= 0
    used, tet = np.unique(tetra[keep], return_inverse=True)
    mesh = TetMesh(grid[used], tet.reshape(-1, 4), lab[keep], np.asarray(cond)[lab[keep]])
    el = ElectrodeSet.from_centers(mesh, fibonacci_sphere_points(L, R), radius=erad, impedances=1e3)
    A = assemble_A(mesh, el)
    B, _, _ = assemble_B_C_R(mesh, el)
    return mesh, el, A, B.tocsc()


def _ref_column(job):
    """One electrode column through the reference's pcg_solve (solver.py:64-111),
    unmodified, on one core.  max_iterations=None: a whole solve."""
    col, max_it = job
    from threadpoolctl import threadpool_limits
    from headfem.errors import ConvergenceError
    from headfem.solver import PcgConfig, pcg_solve

    A, B = _REF["A"], _REF["B"]
    b = B[:, [col]].toarray().ravel()
    with threadpool_limits(1):
        t0 = time.perf_counter()
        try:
            _, it, _ = pcg_solve(A, b, PcgConfig(tolerance=1e-8, max_iterations=max_it))
        except ConvergenceError as exc:  # bounded warm-up sample
            it = exc.iterations
        return time.perf_counter() - t0, int(it)


def run_reference(args):
    """The reference itself (baseline/_ref, numpy/scipy, unmodified) on the box's
    host cores.  The timed region solves one WHOLE electrode column per core, in
    parallel processes through headfem.solver.pcg_solve (solver.py:64-111), and is
    reported as K equal steps: ms_per_step = measured wall / K, RHS-solves/s =
    columns solved / measured wall — nothing extrapolated, and the run ends in
    about a minute plus setup for any K (a whole column takes ~33 s on one core;
    K steps of whole columns would take K times that).  Warm-up steps are bounded
    10-iteration samples (page-in and import only).  Rank 0 alone runs under
    torchrun; the line's config is the GPU arm's."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.config == "c3":
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no MEG lead field (SPEC.md:8)"}))
        return
    if args.config == "c4":
        print(json.dumps({"impl": "reference", "unavailable": "C4's build_dof_map needs a 459 GiB array in the "
                                                              "reference (leadfield.py:98)"}))
        return
    import multiprocessing as mp

    hf = _import_reference()
    t0 = time.time()
    mesh, el, A, B = reference_problem(args.config)
    t_setup = time.time() - t0
    log(f"[reference] {hf.__file__}: mesh {mesh.n_nodes} nodes, assemble_A nnz {A.nnz} in {t_setup:.1f}s")
    _REF["A"], _REF["B"] = A, B
    L = B.shape[1]
    # every host core (16 on this pool's boxes), capped at 32 processes (past ~32 the
    # shared memory bandwidth makes the columns slower without more columns per second)
    cores = int(args.ref_cores or min(os.cpu_count() or 1, 32))
    cores = max(1, min(cores, L))
    ctx = mp.get_context("fork")
    # the cores' columns spread over the electrode set
    cols = sorted({(c * L) // cores for c in range(cores)})
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            pool.map(_ref_column, [(c, 10) for c in cols])
        w0 = time.perf_counter()
        res = pool.map(_ref_column, [(c, None) for c in cols])
        wall = time.perf_counter() - w0
    its = [r[1] for r in res]
    log(f"[reference] {len(cols)} whole columns in {wall:.1f}s (iterations {min(its)}-{max(its)})")
    value = len(cols) / wall
    sample = (f"{len(cols)} whole electrode columns (of {L}), one per process, through headfem.solver.pcg_solve "
              f"from baseline/_ref (tol 1e-8, 1 BLAS thread per process), {min(its)}-{max(its)} iterations; "
              f"the measured wall time of that solve is the timed region, reported as {args.steps} equal steps")
    ncomp = len(np.unique(np.asarray(mesh.labels)))
    out = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": int(args.gpus),
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(wall * 1e3 / args.steps, 1), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (same inputs as the GPU arm)",
           "config": {**eeg_config(args.config, mesh.n_nodes, len(mesh.tetra), ncomp, L, SOURCES[args.config],
                                   1e-8),
                      "parallelism": f"electrode-columns x{int(args.gpus)}"},
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": len(cols), "kind": "reference",
                            "sample": sample},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "reference_setup_s": round(t_setup, 1),
           "timed_region_s": round(wall, 2),
           "lf_build_s_extrapolated": round(L / value, 1)}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c1", "c2", "c3", "c4", "c5"], default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-cores", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("note: fewer than 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c3":
        run_meg(args)
    elif args.config == "c4":
        run_eit(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
