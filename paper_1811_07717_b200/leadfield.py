"""EEG and linearised EIT lead fields on the B200: drop-in for headfem/leadfield.py.

  LeadField, EitDofMap      leadfield.py:32-77
  build_dof_map             leadfield.py:80-101 (chunked nearest-centre search:
                            identical draws and argmin ties, no E x m x 3 array)
  electrode_response        leadfield.py:104-109
  eeg_leadfield             leadfield.py:122-134
  check_current_patterns,
  adjacent_pair_patterns    leadfield.py:137-162
  eit_forward               leadfield.py:165-176
  eit_leadfield             leadfield.py:210-237

Device pipeline of eeg_leadfield (T never leaves HBM):
  hf_pcg_multi (T = A^-1 B, all electrodes at once)
  -> hf_response_matrix (M = C - B'T, symmetrised)
  -> W = -R M^-1  (L x L, host LAPACK exactly as _solve_response)
  -> hf_lf_tail (LF = W (G'T)', gather + fp64 DMMA)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import torch

from . import _native as N
from .device import DeviceCsr, to_host
from .errors import CurrentPatternError, DofError, SingularSystemError
from .fem import DeviceMesh
from .solver import PcgConfig, _raise_failed, operator, rhs_block, solve_block, transfer_device


@dataclass(frozen=True)
class LeadField:
    """Dense measurement-per-DOF matrix with its DOF geometry (leadfield.py:32-56)."""

    matrix: np.ndarray
    positions: np.ndarray
    orientations: np.ndarray | None
    modality: str
    n_patterns: int = 1
    background_sigma: np.ndarray | None = None
    background_data: np.ndarray | None = None

    @property
    def n_electrodes(self):
        return self.matrix.shape[0] // self.n_patterns

    @property
    def n_dofs(self):
        return self.matrix.shape[1]


@dataclass(frozen=True)
class EitDofMap:
    """Disjoint element sets with centres (leadfield.py:59-77)."""

    element_sets: tuple
    centers: np.ndarray

    def __post_init__(self):
        for k, es in enumerate(self.element_sets):
            if len(es) == 0:
                raise DofError(f"DOF {k} has an empty element set")

    @property
    def n_dofs(self):
        return len(self.element_sets)


def nearest_center_device(cc, centers):
    """owner = argmin_j ||cc_i - centers_j|| on the GPU (hf_nearest_center):
    the reference's rounding and first-index ties, every pair evaluated."""
    dev = torch.device("cuda", torch.cuda.current_device())
    P = torch.from_numpy(np.ascontiguousarray(cc, dtype=np.float64)).to(dev)
    Cc = torch.from_numpy(np.ascontiguousarray(centers, dtype=np.float64)).to(dev)
    owner = torch.empty(max(len(cc), 1), dtype=torch.int32, device=dev)
    N.check("hf_nearest_center", N.lib.hf_nearest_center(
        N.ptr(P), len(cc), N.ptr(Cc), len(centers), N.ptr(owner), None, N.stream_handle()))
    return owner[: len(cc)].cpu().numpy().astype(np.int64)


def build_dof_map(mesh, compartments, n_dofs, seed=0):
    """Nearest-centre partition of the perturbable elements (leadfield.py:80-101).

    The reference's centre draw (rng.choice, the one host step), then on the
    device: element centroids with numpy's rounding, the nearest centre for every
    (element, centre) pair with the reference's distance arithmetic and first-index
    argmin, and the partition into sets.  C4 has 4.1M elements x 5,000 DOFs, where
    the reference needs a 459 GiB array.  Needs a CUDA device (no CPU fallback)."""
    N.require_cuda()
    cand = np.flatnonzero(np.isin(mesh.labels, np.asarray(compartments)))
    if cand.size == 0:
        raise DofError("no mesh elements in the perturbable compartments")
    n_dofs = int(n_dofs)
    if not (1 <= n_dofs <= cand.size):
        raise DofError(f"need 1 <= n_dofs <= {cand.size}, got {n_dofs}")
    rng = np.random.default_rng(seed)
    vols = mesh.volumes[cand]
    chosen = rng.choice(cand, size=n_dofs, replace=False, p=vols / vols.sum())
    return _dof_map_device(mesh, cand, chosen)


def _dof_map_device(mesh, cand, chosen):
    """Centroids (hf_tet_centroids), nearest centre (hf_nearest_center) and the
    partition into sets (hf_dof_partition) on the device; only the reference's
    random draw and the final split into per-DOF views run on the host.  The
    device arrays stay attached to the map for dof_sensitivities_device."""
    from .fem import DeviceMesh

    dm = DeviceMesh.of(mesh)
    dev = dm.nodes.device
    st = N.stream_handle()
    n_dofs = len(chosen)
    cand_d = torch.from_numpy(cand.astype(np.int32)).to(dev)
    cc = torch.empty((len(cand), 3), dtype=torch.float64, device=dev)
    N.check("hf_tet_centroids", N.lib.hf_tet_centroids(N.ptr(dm.nodes), N.ptr(dm.tetra), N.ptr(cand_d),
                                                       len(cand), N.ptr(cc), st))
    chosen_d = torch.from_numpy(np.asarray(chosen, dtype=np.int32)).to(dev)
    ctr = torch.empty((n_dofs, 3), dtype=torch.float64, device=dev)
    N.check("hf_tet_centroids", N.lib.hf_tet_centroids(N.ptr(dm.nodes), N.ptr(dm.tetra), N.ptr(chosen_d),
                                                       n_dofs, N.ptr(ctr), st))
    owner = torch.empty(max(len(cand), 1), dtype=torch.int32, device=dev)
    N.check("hf_nearest_center", N.lib.hf_nearest_center(N.ptr(cc), len(cand), N.ptr(ctr), n_dofs,
                                                         N.ptr(owner), None, st))
    sorted_d = torch.empty_like(cand_d)
    ptr_d = torch.empty(n_dofs + 1, dtype=torch.int32, device=dev)
    ws = torch.empty(N.lib.hf_dof_partition_workspace_bytes(len(cand)), dtype=torch.uint8, device=dev)
    N.check("hf_dof_partition", N.lib.hf_dof_partition(N.ptr(cand_d), N.ptr(owner), len(cand), n_dofs,
                                                       N.ptr(sorted_d), N.ptr(ptr_d), N.ptr(ws),
                                                       ws.numel(), st))
    elems = sorted_d.cpu().numpy().astype(np.int64)
    ptr = ptr_d.cpu().numpy().astype(np.int64)
    sets = tuple(np.split(elems, ptr[1:-1]))
    dmap = EitDofMap(element_sets=sets, centers=ctr.cpu().numpy())
    object.__setattr__(dmap, "_device", (sorted_d, ptr_d))
    return dmap


# ---------------------------------------------------------------- device system

class DeviceSystem:
    """The blocks of a CemSystem staged in HBM once per system."""

    def __init__(self, sys, cfg):
        self.sys = sys
        self.n = sys.A.shape[0] if not isinstance(sys.A, DeviceCsr) else sys.A.shape[0]
        self.L = sys.B.shape[1]
        self.op = operator(sys.A, cfg)
        dev = self.op.A.val.device
        self.Bd = rhs_block(sys.B, dev=dev)                        # n x L dense RHS block
        self.Bt = DeviceCsr.from_scipy(sp.csr_matrix(sp.csr_matrix(sys.B).T), dev)
        self.Cdiag = torch.from_numpy(np.ascontiguousarray(sys.C.diagonal(), dtype=np.float64)).to(dev)


def response_block_device(Bt, T, L, Cdiag, col0=0):
    """Raw response block (C - B'T)[:, col0:col0+k] (device L x k) for the k
    transfer columns held in T (leadfield.py:107)."""
    k = T.shape[1]
    Mraw = torch.empty((L, k), dtype=torch.float64, device=T.device)
    N.check("hf_response_matrix", N.lib.hf_response_matrix(
        N.C.byref(Bt.struct), N.ptr(T), T.stride(0), L, int(col0), k, N.ptr(Cdiag), N.ptr(Mraw),
        N.stream_handle()))
    return Mraw


def symmetrize(Mraw):
    """M = (M + M')/2, the exact-symmetry step of leadfield.py:108."""
    return 0.5 * (Mraw + Mraw.T)


def response_matrix_device(dsys, T):
    """M = C - B'T, symmetrised (leadfield.py:107-108), as a host array."""
    return symmetrize(response_block_device(dsys.Bt, T, dsys.L, dsys.Cdiag).cpu().numpy())


_BLAS = None


def _one_blas_thread():
    """A context that runs BLAS/LAPACK single-threaded: for an L x L (L <= 256)
    factorisation a multi-threaded OpenBLAS spends 5-200 ms synchronising its
    threads against well under 1 ms of work (measured on the GPU box and here)."""
    global _BLAS
    if _BLAS is None:
        from threadpoolctl import ThreadpoolController

        _BLAS = ThreadpoolController()
    return _BLAS.limit(limits=1, user_api="blas")


def _solve_response(M, rhs):
    """lu_factor / lu_solve with the reference's singularity rule (leadfield.py:112-119)."""
    with _one_blas_thread():
        try:
            lu, piv = sla.lu_factor(M)
        except (ValueError, sla.LinAlgError) as exc:
            raise SingularSystemError(f"electrode response factorization failed: {exc}")
        if np.any(np.abs(np.diag(lu)) < 1e-300):
            raise SingularSystemError("electrode response matrix is singular")
        return sla.lu_solve((lu, piv), rhs)


def _electrode_response_device(sys, cfg):
    dsys = DeviceSystem(sys, cfg)
    T, info = transfer_device(dsys.op, dsys.Bd, cfg)
    M = response_matrix_device(dsys, T)
    return dsys, T, M, info


def electrode_response(sys, cfg=PcgConfig(), threads=1):
    """Transfer matrix T = A^-1 B and the symmetric response M = C - B'T (leadfield.py:104-109)."""
    _, T, M, _ = _electrode_response_device(sys, cfg)
    return to_host(T.contiguous()), M


def lf_tail_device(T, Gt, W):
    """LF (L x ncols, device) = W (G'T)' by hf_lf_tail; T holds K columns and W
    is L x K (the whole response operator, or one rank's column block of it)."""
    dev = T.device
    K = T.shape[1]
    Wh = np.ascontiguousarray(W, dtype=np.float64)
    L = Wh.shape[0]
    if Wh.shape[1] != K:
        raise ValueError(f"W has {Wh.shape[1]} columns, T has {K}")
    ncols = Gt.shape[0]
    LF = torch.empty((L, ncols), dtype=torch.float64, device=dev)
    Wd = torch.from_numpy(Wh).to(dev)
    N.check("hf_lf_tail", N.lib.hf_lf_tail(N.ptr(T), T.stride(0), K, N.C.byref(Gt.struct),
                                           N.ptr(Wd), L, K, N.ptr(LF), N.stream_handle()))
    return LF


def response_operator(M, R):
    """W = -R M^-1 (L x L) with the reference's LU (leadfield.py:112-119, 129)."""
    L = M.shape[0]
    X = _solve_response(M, np.eye(L))
    with _one_blas_thread():
        return -(R @ X)


def eeg_leadfield(sys, cfg=PcgConfig(), threads=1):
    """EEG lead field L = -R M^-1 (T'G); columns are zero-mean (leadfield.py:122-134)."""
    if sys.G is None or sys.G.shape[1] == 0:
        raise SingularSystemError("system has no source matrix G")
    dsys, T, M, _ = _electrode_response_device(sys, cfg)
    W = response_operator(M, sys.R)
    G = sys.G if sp.issparse(sys.G) else sp.csr_matrix(np.asarray(sys.G, dtype=float))
    Gt = DeviceCsr.from_scipy(sp.csr_matrix(G.T), T.device)
    LF = to_host(lf_tail_device(T, Gt, W))
    src = sys.source_space
    return LeadField(matrix=LF, positions=src.positions if src is not None else None,
                     orientations=src.orientations if src is not None else None, modality="eeg")


def check_current_patterns(currents, n_electrodes):
    """Zero-sum injection patterns, shape (L,) or (L, P) (leadfield.py:137-152)."""
    I = np.asarray(currents, dtype=float)
    if I.ndim == 1:
        I = I[:, None]
    if I.shape[0] != n_electrodes:
        raise CurrentPatternError(f"pattern length {I.shape[0]} != electrode count {n_electrodes}")
    norms = np.linalg.norm(I, axis=0)
    if np.any(norms == 0):
        return I
    bad = np.abs(I.sum(axis=0)) > 1e-12 * np.maximum(norms, 1e-300)
    if np.any(bad):
        raise CurrentPatternError(f"current pattern(s) {np.flatnonzero(bad).tolist()} do not sum to zero")
    return I


def adjacent_pair_patterns(n_electrodes, amplitude=1.0):
    """+amplitude on electrode k, -amplitude on k+1 (leadfield.py:155-162)."""
    I = np.zeros((n_electrodes, n_electrodes - 1))
    for k in range(n_electrodes - 1):
        I[k, k] = amplitude
        I[k + 1, k] = -amplitude
    return I


def eit_forward(sys, currents, cfg=PcgConfig(), tm=None, threads=1):
    """Electrode voltages y = R M^-1 I (leadfield.py:165-176)."""
    I = check_current_patterns(currents, sys.n_electrodes)
    if tm is None:
        tm = electrode_response(sys, cfg, threads=threads)
    _, M = tm
    y = sys.R @ _solve_response(M, I)
    return y[:, 0] if np.asarray(currents).ndim == 1 else y


def dof_sensitivities_device(mesh, dofs, ground, T, U, L, P):
    """Q (P x m_dofs x L, device) = T' K_m u_p for every DOF and pattern."""
    dm = DeviceMesh.of(mesh)
    dev = T.device
    cached = getattr(dofs, "_device", None)
    if cached is not None and cached[0].device == dev:  # built by _dof_map_device
        de, dp = cached
    else:
        elems = np.concatenate([np.asarray(e, dtype=np.int64) for e in dofs.element_sets])
        ptr = np.cumsum([0] + [len(e) for e in dofs.element_sets])
        de = torch.from_numpy(elems.astype(np.int32)).to(dev)
        dp = torch.from_numpy(ptr.astype(np.int32)).to(dev)
    nd = dofs.n_dofs
    Q = torch.empty((P, nd, L), dtype=torch.float64, device=dev)
    ws = torch.empty(N.lib.hf_eit_sens_workspace_bytes(de.numel()), dtype=torch.uint8, device=dev)
    N.check("hf_eit_sens", N.lib.hf_eit_sens(
        N.ptr(dm.nodes), N.ptr(dm.tetra), N.ptr(de), N.ptr(dp), nd, int(ground), N.ptr(T),
        T.stride(0), L, N.ptr(U), U.stride(0), P, N.ptr(Q), N.ptr(ws), ws.numel(), N.stream_handle()))
    return Q


def eit_columns_device(mesh, dofs, ground, T, U, W, c0=0):
    """EIT Jacobian columns cols[p*L:(p+1)*L] = W[:, c0:c0+k] Q[p]' (leadfield.py:230-237)
    with Q = T' K_m u_p for the k transfer columns in T (electrodes c0..c0+k-1).
    With every electrode (k = L) this is the lead field; on a rank holding an
    electrode block it is that block's share of the sum over electrodes."""
    L, k, P = W.shape[0], T.shape[1], U.shape[1]
    dev = T.device
    Q = dof_sensitivities_device(mesh, dofs, ground, T, U, k, P)      # P x nd x k
    Wd = torch.from_numpy(np.ascontiguousarray(W)).to(dev)
    nd = dofs.n_dofs
    cols = torch.empty((P * L, nd), dtype=torch.float64, device=dev)
    for p in range(P):
        N.check("hf_dense_lf", N.lib.hf_dense_lf(
            N.ptr(Q[p]), nd, k, N.ptr(Wd[:, c0:]), L, L, N.ptr(cols[p * L:(p + 1) * L]), nd,
            N.stream_handle()))
    return cols


def eit_leadfield(sys, dofs, currents, cfg=PcgConfig(), threads=1):
    """Linearised EIT lead field around the mesh conductivity (leadfield.py:210-237)."""
    I = check_current_patterns(currents, sys.n_electrodes)
    dsys, T, M, _ = _electrode_response_device(sys, cfg)
    V = _solve_response(M, I)                     # M^-1 I, (L, P)
    y_bg = sys.R @ V
    L, P = dsys.L, I.shape[1]
    dev = T.device
    Vd = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    Bcsr = DeviceCsr.from_scipy(sp.csr_matrix(sys.B), dev)
    BV = torch.empty((dsys.n, P), dtype=torch.float64, device=dev)  # n x P right-hand sides u_p
    N.check("hf_csr_dense", N.lib.hf_csr_dense(N.C.byref(Bcsr.struct), N.ptr(Vd), P, P, N.ptr(BV), P,
                                               N.stream_handle()))
    U, info = solve_block(dsys.op, BV, cfg)
    _raise_failed(info, U, cfg, column_tag=False)  # pcg_solve semantics: no column tag
    cols = eit_columns_device(sys.mesh, dofs, sys.ground, T, U, response_operator(M, sys.R))
    return LeadField(matrix=to_host(cols.contiguous()), positions=dofs.centers, orientations=None,
                     modality="eit", n_patterns=P,
                     background_sigma=np.array(sys.mesh.sigma, copy=True),
                     background_data=y_bg.T.ravel())


__all__ = ["LeadField", "EitDofMap", "build_dof_map", "electrode_response", "eeg_leadfield",
           "check_current_patterns", "adjacent_pair_patterns", "eit_forward", "eit_leadfield",
           "DeviceSystem", "lf_tail_device", "eit_columns_device", "response_operator", "response_block_device",
           "symmetrize"]
