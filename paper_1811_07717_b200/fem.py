"""P1 stiffness assembly on the B200: drop-in for the hot part of headfem/fem.py.

  stiffness_blocks   fem.py:70-93   -> hf_p1_blocks
  volume_stiffness   fem.py:105-109 -> hf_p1_blocks + hf_p1_assemble_{prepare,fill}
  assemble_A         fem.py:197-224 -> the same, with electrode contact terms and grounding

The CSR pattern is scipy's (sorted columns, explicit zeros kept, grounded
row/column deleted except the diagonal); values are summed in a fixed order,
so the matrix is bit-reproducible run to run.  The non-hot input builders
(electrodes, B/C/R, G) live in `model.py`.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .device import DeviceCsr, device, to_device
from .errors import AssemblyError
from .model import electrode_contacts


def _sigma_arg(mesh, sigma, elements):
    """(array or None, scalar) following stiffness_blocks' sigma rules (fem.py:84-93)."""
    if sigma is None:
        s = mesh.sigma if elements is None else np.asarray(mesh.sigma)[elements]
        return np.asarray(s, dtype=float), 0.0
    if np.isscalar(sigma):
        return None, float(sigma)
    s = np.asarray(sigma, dtype=float)
    return s, 0.0


class DeviceMesh:
    """Mesh arrays resident in HBM: nodes (n,3) f64, tetra (m,4) int32."""

    def __init__(self, nodes, tetra, dev=None):
        dev = dev or device()
        self.n = int(len(nodes))
        self.m = int(len(tetra))
        self.nodes = to_device(nodes, np.float64, dev, slot=0)
        self.tetra = to_device(tetra, np.int32, dev, slot=1)

    @classmethod
    def of(cls, mesh):
        dm = getattr(mesh, "_hfb200_device", None)
        if dm is None or dm.nodes.device != device():
            dm = cls(mesh.nodes, mesh.tetra)
            try:
                object.__setattr__(mesh, "_hfb200_device", dm)
            except (AttributeError, TypeError):
                pass
        return dm


def blocks_device(dmesh, sigma_arr, sigma_scalar, elements=None):
    """(m_sub*16 + 1) device buffer of 4x4 blocks (+ flag slot) and host flags."""
    dev = dmesh.nodes.device
    m_sub = dmesh.m if elements is None else len(elements)
    el = None
    if elements is not None:
        el = torch.from_numpy(np.ascontiguousarray(elements, dtype=np.int32)).to(dev)
    sg, cols = None, 0
    if torch.is_tensor(sigma_arr):  # already resident (engine.EegEngine)
        sg, cols = sigma_arr, (1 if sigma_arr.dim() == 1 else 6)
    elif sigma_arr is not None:
        sg = torch.from_numpy(np.array(sigma_arr, dtype=np.float64, order="C")).to(dev)
        cols = 1 if sigma_arr.ndim == 1 else 6
    blocks = torch.empty(m_sub * 16 + 1, dtype=torch.float64, device=dev)
    flags = N.C.c_int32(0)
    N.check("hf_p1_blocks", N.lib.hf_p1_blocks(
        N.ptr(dmesh.nodes), N.ptr(dmesh.tetra), dmesh.m, N.ptr(el), m_sub, N.ptr(sg), cols,
        float(sigma_scalar), N.ptr(blocks), None, N.C.byref(flags), N.stream_handle()))
    f = int(flags.value)
    if f & 1:
        raise AssemblyError("non-positive element volume")
    if f & 2:
        raise AssemblyError("negative scalar conductivity")
    if f & 4:
        raise AssemblyError("conductivity tensor row is not positive definite")
    return blocks


def stiffness_blocks(mesh, sigma=None, elements=None):
    """Per-element 4x4 blocks V grad_i . sigma grad_j, shape (m, 4, 4) (fem.py:70-93)."""
    dm = DeviceMesh.of(mesh)
    s, sc = _sigma_arg(mesh, sigma, elements)
    el = None if elements is None else np.asarray(elements, dtype=np.int64)
    blocks = blocks_device(dm, s, sc, el)
    m_sub = dm.m if el is None else len(el)
    return blocks[: m_sub * 16].view(m_sub, 4, 4).cpu().numpy()


def assemble_device(dmesh, blocks, n, etri=None, ecoef=None, ground=-1, tetra=None):
    """CSR of the summed element blocks (+ contact terms, grounding) in HBM."""
    dev = dmesh.nodes.device
    tet = dmesh.tetra if tetra is None else tetra
    m = int(tet.shape[0])
    nt = 0 if etri is None else int(etri.shape[0])
    et = None if nt == 0 else etri
    ec = None if nt == 0 else ecoef
    ws = torch.empty(N.lib.hf_p1_assemble_workspace_bytes(n, m, nt), dtype=torch.uint8, device=dev)
    indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    nnz = N.C.c_int64(0)
    st = N.stream_handle()
    N.check("hf_p1_assemble_prepare", N.lib.hf_p1_assemble_prepare(
        N.ptr(tet), n, m, N.ptr(et), nt, int(ground), N.ptr(indptr), N.C.byref(nnz), N.ptr(ws),
        ws.numel(), st))
    k = int(nnz.value)
    indices = torch.empty(max(k, 1), dtype=torch.int32, device=dev)[:k]
    val = torch.empty(max(k, 1), dtype=torch.float64, device=dev)[:k]
    N.check("hf_p1_assemble_fill", N.lib.hf_p1_assemble_fill(
        N.ptr(tet), n, m, N.ptr(blocks), N.ptr(et), N.ptr(ec), nt, int(ground), N.ptr(indptr),
        N.ptr(indices), N.ptr(val), N.ptr(ws), ws.numel(), st))
    return DeviceCsr(indptr, indices, val, (n, n))


def volume_stiffness_device(mesh, sigma=None, elements=None):
    dm = DeviceMesh.of(mesh)
    s, sc = _sigma_arg(mesh, sigma, elements)
    if elements is None:
        blocks = blocks_device(dm, s, sc)
        return assemble_device(dm, blocks, dm.n)
    el = np.asarray(elements, dtype=np.int64)
    blocks = blocks_device(dm, s, sc, el)
    sub = dm.tetra[torch.from_numpy(el).to(dm.tetra.device)].contiguous()
    return assemble_device(dm, blocks, dm.n, tetra=sub)


def _sorted(M):
    """The assembled CSR has sorted column indices (scipy's COO -> CSR pattern, bit-exact):
    record it so callers that check (`has_sorted_indices`, an O(nnz) scan) need not."""
    M.has_sorted_indices = True
    return M


def volume_stiffness(mesh, sigma=None, elements=None):
    """Conductivity stiffness without electrode or grounding terms (fem.py:105-109)."""
    return _sorted(volume_stiffness_device(mesh, sigma, elements).to_scipy())


def assemble_A_device(mesh, electrodes, ground=True):
    """(DeviceCsr A, ground index or None) — fem.py:197-224 without leaving HBM."""
    dm = DeviceMesh.of(mesh)
    s, sc = _sigma_arg(mesh, None, None)
    blocks = blocks_device(dm, s, sc)
    tri, coef = electrode_contacts(electrodes)
    g = -1
    if ground and electrodes.count:
        from .topology import ground_node_device

        g = ground_node_device(mesh, electrodes)
    dev = dm.nodes.device
    et = torch.from_numpy(np.ascontiguousarray(tri, dtype=np.int32)).to(dev) if len(tri) else None
    ec = torch.from_numpy(np.ascontiguousarray(coef, dtype=np.float64)).to(dev) if len(tri) else None
    A = assemble_device(dm, blocks, dm.n, et, ec, g)
    return A, (None if g < 0 else g)


def assemble_A(mesh, electrodes, ground=True):
    """Grounded CEM stiffness matrix as scipy CSR (fem.py:197-224)."""
    return _sorted(assemble_A_device(mesh, electrodes, ground)[0].to_scipy())


__all__ = ["stiffness_blocks", "volume_stiffness", "assemble_A", "assemble_A_device",
           "volume_stiffness_device", "DeviceMesh"]
