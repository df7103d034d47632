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
    ncomp = len(np.unique(prob.mesh.labels))
    return {"workload": f"{prob.name}: {prob.mesh.n_nodes:,}-node {ncomp}-compartment sphere Kuhn mesh, "
                        f"{prob.electrodes.count}-electrode EEG lead field, "
                        f"{prob.sources.n_sources:,} dipole sources",
            "config": prob.name, "n_nodes": int(prob.mesh.n_nodes),
            "n_elements": int(prob.mesh.n_elements), "electrodes": int(prob.electrodes.count),
            "sources": int(prob.sources.n_sources), "lf_shape": [int(prob.electrodes.count),
                                                                 3 * int(prob.sources.n_sources)],
            "tolerance": cfg.tolerance, "precision": "fp64",
            "l2_policy": "inputs larger than L2 (n x 64 fp64 vector blocks = 512 MB each)"}


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
def kernel_roofline(engine, A, rounds=24, config="c2"):
    """Per-kernel CUDA-event timing of a PCG round at the bench's batch width,
    algorithmic bytes per launch, fraction of the HBM peak."""
    import torch

    from paper_1811_07717_b200 import _native as N
    from paper_1811_07717_b200.device import PcgOperator, width_for
    from paper_1811_07717_b200.solver import MAX_BATCH

    op = PcgOperator(A, "ldp")
    n = op.n
    kp = width_for(op.batch_width(engine.Bd.shape[1], MAX_BATCH))  # the solver's own batch width
    Bb = torch.zeros((n, kp), dtype=torch.float64, device=engine.Bd.device)
    k = min(kp, engine.Bd.shape[1])
    Bb[:, :k] = engine.Bd[:, :k]
    X = torch.empty_like(Bb)
    ws = torch.empty(N.lib.hf_pcg_workspace_bytes(n, kp, op.Ac.nnz), dtype=torch.uint8, device=Bb.device)
    ms = (N.C.c_float * 3)()
    fused = N.C.c_int32(0)
    N.check("hf_pcg_profile", N.lib.hf_pcg_profile(
        N.C.byref(op.Ac.struct), N.ptr(op.d), N.ptr(Bb), n, kp, rounds, N.ptr(X), ms,
        N.C.byref(fused), N.ptr(ws), ws.numel(), N.stream_handle()))
    nnz = op.Ac.nnz
    spmm = ("k_spmm_ell2" if fused.value & 4 else "k_spmm_ell") if fused.value & 2 else "k_spmm_pq"
    if fused.value & 1:
        # k_xs: x/p update (read x, p, r, dd; write x, p) + next SpMM (write q; CSR);
        # the p rows it gathers were just written and are not re-read from DRAM
        algo = {"k_xs": 48 * n * kp + 12 * nnz + 4 * (n + 1) + 16 * n,
                "k_update_r": 24 * n * kp + 16 * n}
        times = dict(zip(algo, [float(ms[0]), float(ms[1])]))
    else:
        # the SpMM's algorithmic bytes count the CSR (the ELL copy reads 12 B x 8 slots per row)
        xd = fused.value >> 8
        if xd > 1:
            # x deferred over a ring of xd p blocks: xd-1 p-only rounds (read p, r;
            # write p) and one x round (x read+write, xd p reads, r read, p write),
            # averaged per round; dd (16 B/row) read in every round
            upd = ("k_update_pxring", ((xd - 1) * 24 + 32 + 8 * xd) * n * kp // xd + 16 * n)
        else:
            upd = ("k_update_xp", 40 * n * kp + 16 * n)
        algo = {spmm: 16 * n * kp + 12 * nnz + 4 * (n + 1),
                "k_update_r": 24 * n * kp + 16 * n,
                upd[0]: upd[1]}
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
            "traffic": traffic, "algorithmic_bytes_per_launch": algo[dominant],
            "launch_ms": round(times[dominant], 4),
            "share_of_round": round(times[dominant] / total_ms, 3),
            "pcg_round": {"kp": kp, "n": n, "nnz_spmm": nnz, "fused": bool(fused.value & 1),
                          "x_deferral": max(1, fused.value >> 8),
                          "ms": round(total_ms, 4),
                          "bytes": total_bytes,
                          "gbs": round(total_bytes / (total_ms * 1e-3) / 1e9, 1),
                          "frac": round(total_bytes / (total_ms * 1e-3) / 1e9 / peak, 4),
                          "bytes_per_rhs_iter": total_bytes / kp},
            "kernels": {k2: {kk: (round(v, 4) if isinstance(v, float) else v) for kk, v in d.items()}
                        for k2, d in kern.items()}}


def cpu_baseline_port(A, b, iters_per_col, sample_iters=150):
    """The oracle's numpy PCG (solver.py:64-111 restated) on one host core, for a
    bounded number of iterations of one C2 column; RHS-solves/s extrapolated."""
    import oracle
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        oracle.pcg_solve(A, b, oracle.PcgSettings(), iterations_cap=3)
        t0 = time.perf_counter()
        oracle.pcg_solve(A, b, oracle.PcgSettings(), iterations_cap=sample_iters)
        dt = time.perf_counter() - t0
    t_iter = dt / sample_iters
    return {"value": 1.0 / (t_iter * iters_per_col), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{sample_iters} PCG iterations of electrode column 0 on the bench system "
                      f"({t_iter * 1e3:.1f} ms/iteration, 1 thread), extrapolated to "
                      f"{iters_per_col:.0f} iterations per column",
            "ms_per_iteration": round(t_iter * 1e3, 3)}


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

    # end to end through the public API: host mesh/electrodes/G in, host LF out
    e2e = None
    if not args.no_e2e:
        h2d = d2h = 0
        barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            # B, C, R and G' (on the device) assembled inside the timed call
            eng2 = EegEngine(prob.mesh, prob.electrodes, prob.sources, cfg, columns=blocks[rank], dev=dev)
            if world == 1:
                lf_host = eng2.build(to_host=True)
            else:
                lf_dev = sharded_leadfield(eng2, world, rank)
                lf_host = None if lf_dev is None else to_host(lf_dev.contiguous())
            h2d += eng2.h2d_bytes
            if lf_host is not None:
                d2h += lf_host.nbytes + 8 * L * L
            del eng2
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - w0
        tt = torch.tensor([wall, h2d, d2h], dtype=torch.float64, device=dev)
        if world > 1:
            mx = tt[:1].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(tt, op=dist.ReduceOp.SUM)
            tt[0] = mx[0]
        wall, h2d, d2h = (float(v) for v in tt.tolist())
        e2e = {"value": L * args.steps / wall, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
               "ms_per_step": round(wall * 1e3 / args.steps, 2),
               "api": "engine.EegEngine(mesh, electrodes, sources).build(to_host=True) -> LF on host "
                      "(B, C, R and, on the device, G' assembled inside the step)"}

    roof = None
    A = None
    if rank == 0:
        A = engine.assemble()
        roof = kernel_roofline(engine, A, config=args.config)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Ah = A.to_scipy()
        b = prob.B[:, 0].toarray().ravel()
        cpu = cpu_baseline_port(Ah, b, float(np.mean(info.iterations)))
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
               "cpu_baseline": cpu, "e2e": e2e, "clocks": clk}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm
_REF = {}


def _ref_worker(args):
    col, iters = args
    import oracle
    from threadpoolctl import threadpool_limits

    A, B = _REF["A"], _REF["B"]
    b = B[:, col].toarray().ravel()
    with threadpool_limits(1):
        t0 = time.perf_counter()
        oracle.pcg_solve(A, b, oracle.PcgSettings(), iterations_cap=iters)
        return time.perf_counter() - t0


def run_reference(args):
    """The reference's CPU algorithm (oracle port of headfem, numpy/scipy) on the
    box's host cores: every step runs one bounded PCG sample per core in parallel
    (one electrode column each); RHS-solves/s is extrapolated with the column
    iteration count measured by one full reference solve."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    import oracle
    from paper_1811_07717_b200 import synthetic
    from paper_1811_07717_b200.solver import PcgConfig

    cfg = PcgConfig(tolerance=1e-8)
    t0 = time.time()
    prob = synthetic.eeg_problem(args.config, with_G=False)
    tris = [t for t in prob.electrodes.triangles]
    A, g = oracle.assemble_A(prob.mesh.nodes, prob.mesh.tetra, prob.mesh.sigma, tris,
                             prob.electrodes.triangle_areas, prob.electrodes.impedances,
                             prob.electrodes.areas)
    t_asm = time.time() - t0
    log(f"[reference] problem + oracle assembly in {t_asm:.1f}s")
    _REF["A"], _REF["B"] = A, prob.B.tocsc()
    b0 = prob.B[:, 0].toarray().ravel()
    t1 = time.time()
    if args.ref_full_column:
        _, iters, _ = oracle.pcg_solve(A, b0, oracle.PcgSettings())
    else:
        iters = None
    t_full = time.time() - t1
    cores = int(args.ref_cores or os.cpu_count() or 1)
    sample = args.ref_sample_iters
    L = prob.electrodes.count
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        jobs = [((c % L), sample) for c in range(cores)]
        for _ in range(args.warmup):
            pool.map(_ref_worker, jobs)
        walls = []
        for _ in range(args.steps):
            w0 = time.perf_counter()
            pool.map(_ref_worker, jobs)
            walls.append(time.perf_counter() - w0)
    wall = float(np.mean(walls))
    t_iter_eff = wall / (cores * sample)              # seconds per column-iteration, all cores
    if iters is None:
        iters = float(args.ref_iters_hint)
    value = 1.0 / (t_iter_eff * iters)
    sample_desc = (f"{cores} processes x {sample} PCG iterations (one electrode column each) of the "
                   f"{prob.name.upper()} system per step, {t_iter_eff * cores * 1e3:.1f} ms/iteration/process; "
                   f"extrapolated with {iters} iterations per column "
                   f"({'measured by one full reference solve' if args.ref_full_column else 'hint'})")
    out = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": int(args.gpus),
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(L / value * 1e3, 1), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (same inputs as the GPU arm)",
           "config": {**workload_config(prob, cfg), "parallelism": f"{cores} host processes"},
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "port",
                            "sample": sample_desc},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "reference_setup_s": {"problem_and_assembly": round(t_asm, 1), "full_column": round(t_full, 1)},
           "lf_build_s_extrapolated": round(L / value + t_asm, 1)}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c1", "c2", "c5"], default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-cores", type=int, default=0)
    ap.add_argument("--ref-sample-iters", type=int, default=40)
    ap.add_argument("--ref-full-column", type=int, default=1)
    ap.add_argument("--ref-iters-hint", type=float, default=828)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("note: fewer than 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
