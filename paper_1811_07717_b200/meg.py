"""MEG lead field on the EEG path's FEM system (BASELINE.json configs[2], C3).

The reference has no MEG (SPEC.md:8 puts it out of scope), so this config is
throughput-only with parity unpinned: the standard FEM reciprocity
formulation (csrc/meg.cu) on the same grounded stiffness matrix, the same
multi-RHS LDP-PCG (one right-hand side per sensor instead of per electrode)
and the same gather + DMMA tail as the EEG lead field:

    S'     = hf_meg_rhs(mesh, sensors)           n x n_sensors
    T_meg  = A^-1 S'                              hf_pcg_multi (solver.solve_block)
    L      = L_primary - T_meg' G                 hf_meg_primary + hf_lf_tail (W = -I)

The minus sign: the reference's source matrix enters with the potential
u = -A^-1 G q (its EEG lead field is L = -R M^-1 T'G, leadfield.py:129).

A is assembled without electrode contact terms and grounded at the lowest
boundary node (the reference's ground_node rule with no electrodes,
fem.py:188-194).  A sensor is a weighted set of point coils: `helmet_306`
builds an Elekta-like array of 102 sites with one radial magnetometer and two
planar gradiometers (coil pairs 16.8 mm apart) each.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .device import device
from .device import to_host as host_copy
from .fem import DeviceMesh, assemble_device, blocks_device
from .leadfield import LeadField, lf_tail_device
from .solver import PcgConfig, _raise_failed, solve_block
from .device import PcgOperator


@dataclass(frozen=True)
class SensorArray:
    coils: np.ndarray      # (n_coils, 8): position (3), normal (3), weight, pad
    coil_ptr: np.ndarray   # (n_sensors + 1,) coils of sensor s: coil_ptr[s]:coil_ptr[s+1]
    kinds: tuple           # 'mag' | 'grad1' | 'grad2' per sensor

    @property
    def n_sensors(self):
        return len(self.coil_ptr) - 1


def helmet_306(radius=0.12, n_sites=102, baseline=0.0168, z_min=-0.02):
    """102 sites on a spherical cap (golden-angle spiral, z >= z_min), each with a
    radial magnetometer and two orthogonal planar gradiometers: 306 sensors."""
    pts = []
    k = 0
    while len(pts) < n_sites:  # spiral on the whole sphere, keep the cap
        m = 4 * n_sites
        i = k + 0.5
        phi = np.arccos(1.0 - 2.0 * i / m)
        theta = np.pi * (1.0 + 5.0 ** 0.5) * i
        p = np.array([np.sin(phi) * np.cos(theta), np.sin(phi) * np.sin(theta), np.cos(phi)])
        if radius * p[2] >= z_min:
            pts.append(p)
        k += 1
    coils, ptr, kinds = [], [0], []
    for p in pts:
        nrm = p / np.linalg.norm(p)
        a = np.cross(nrm, [0.0, 0.0, 1.0] if abs(nrm[2]) < 0.9 else [1.0, 0.0, 0.0])
        e1 = a / np.linalg.norm(a)
        e2 = np.cross(nrm, e1)
        r0 = radius * nrm
        coils.append([*r0, *nrm, 1.0, 0.0])
        ptr.append(len(coils))
        kinds.append("mag")
        for e, name in ((e1, "grad1"), (e2, "grad2")):
            w = 1.0 / baseline
            coils.append([*(r0 + 0.5 * baseline * e), *nrm, w, 0.0])
            coils.append([*(r0 - 0.5 * baseline * e), *nrm, -w, 0.0])
            ptr.append(len(coils))
            kinds.append(name)
    return SensorArray(np.array(coils, dtype=np.float64), np.array(ptr, dtype=np.int32), tuple(kinds))


def _ground(mesh):
    """Lowest boundary node (fem.py:188-194 with no electrode)."""
    return int(mesh.boundary_nodes()[0])


class MegEngine:
    """C3 lead field with the mesh, sensors and source matrix resident in HBM."""

    def __init__(self, mesh, sensors, sources, cfg=PcgConfig(), dev=None):
        from .topology import assemble_Gt_device

        dev = dev or device()
        self.cfg = cfg
        self.mesh = mesh
        self.dmesh = DeviceMesh.of(mesh)
        self.sigma = torch.from_numpy(np.array(mesh.sigma, dtype=np.float64)).to(dev)
        if self.sigma.dim() != 1:
            raise ValueError("the MEG right-hand side needs scalar conductivities")
        self.ground = _ground(mesh)
        self.sensors = sensors
        self.coils = torch.from_numpy(np.ascontiguousarray(sensors.coils)).to(dev)
        self.coil_ptr = torch.from_numpy(np.ascontiguousarray(sensors.coil_ptr, dtype=np.int32)).to(dev)
        self.Gt = assemble_Gt_device(mesh, sources) if hasattr(sources, "element_ids") else sources
        self.positions = torch.from_numpy(np.ascontiguousarray(sources.positions, dtype=np.float64)).to(dev)
        self.n_sources = len(sources.positions)
        self.last_info = None

    def assemble(self):
        blocks = blocks_device(self.dmesh, self.sigma, 0.0)
        return assemble_device(self.dmesh, blocks, self.dmesh.n, None, None, self.ground)

    def rhs(self):
        """S' (n x n_sensors) on the device."""
        dm, ns = self.dmesh, self.sensors.n_sensors
        out = torch.empty((dm.n, ns), dtype=torch.float64, device=self.sigma.device)
        ws = torch.empty(N.lib.hf_meg_workspace_bytes(dm.n, dm.m), dtype=torch.uint8, device=out.device)
        N.check("hf_meg_rhs", N.lib.hf_meg_rhs(
            N.ptr(dm.nodes), N.ptr(dm.tetra), N.ptr(self.sigma), dm.n, dm.m, self.ground,
            N.ptr(self.coils), N.ptr(self.coil_ptr), ns, N.ptr(out), ns, N.ptr(ws), ws.numel(),
            N.stream_handle()))
        return out

    def primary(self):
        ns = self.sensors.n_sensors
        Lp = torch.empty((ns, 3 * self.n_sources), dtype=torch.float64, device=self.sigma.device)
        N.check("hf_meg_primary", N.lib.hf_meg_primary(
            N.ptr(self.coils), N.ptr(self.coil_ptr), ns, N.ptr(self.positions), self.n_sources,
            N.ptr(Lp), N.stream_handle()))
        return Lp

    def build(self, to_host=False):
        A = self.assemble()
        S = self.rhs()
        op = PcgOperator(A, self.cfg.preconditioner)
        T, info = solve_block(op, S, self.cfg)
        _raise_failed(info, T, self.cfg, column_tag=True)
        self.last_info = info
        ns = self.sensors.n_sensors
        L = self.primary() + lf_tail_device(T, self.Gt, -np.eye(ns))  # u = -A^-1 G q
        return host_copy(L.contiguous()) if to_host else L


def meg_leadfield(mesh, sensors, sources, cfg=PcgConfig()):
    """(n_sensors x 3 S) MEG lead field as a LeadField (modality 'meg')."""
    eng = MegEngine(mesh, sensors, sources, cfg)
    L = eng.build(to_host=True)
    return LeadField(matrix=L, positions=sources.positions, orientations=None, modality="meg")


__all__ = ["SensorArray", "helmet_306", "MegEngine", "meg_leadfield"]
