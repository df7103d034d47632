"""Device-resident EEG lead-field build (the BASELINE.json hot path end to end).

`EegEngine` stages one problem in HBM once — mesh (nodes, int32 tetra,
sigma), electrode contact triangles, the RHS block of this rank's electrode
columns, B' and G' as CSR — and then every `build()` runs the whole path
without host round trips of n-sized data:

  hf_p1_blocks + hf_p1_assemble_*   A (fem.py:197-224)
  hf_ldp, hf_csr_prune_*            preconditioner, zero-free SpMM copy
  hf_pcg_multi                      T[:, block] = A^-1 B[:, block] (solver.py:114-141)
  hf_response_matrix                (C - B'T)[:, block]            (leadfield.py:107)
  host (L x L)                      M = (M + M')/2, W = -R M^-1    (leadfield.py:108-119)
  hf_lf_tail                        LF (partial over the block) = W[:, block] (G'T_block)'

With one rank the block is every electrode.  `distributed.eeg_leadfield_sharded`
splits the electrode columns over ranks and exchanges the two small results
(M blocks, LF partial sums) with NCCL.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch

from . import model
from .device import DeviceCsr, PcgOperator, device, to_device
from .device import to_host as _to_host
from .fem import DeviceMesh, assemble_device, blocks_device
from .leadfield import lf_tail_device, response_block_device, response_operator, symmetrize
from .solver import PcgConfig, _raise_failed, rhs_block, solve_block


def column_blocks(L, world):
    """Contiguous electrode blocks, sizes differing by at most one."""
    base, extra = divmod(L, world)
    out, c = [], 0
    for r in range(world):
        k = base + (1 if r < extra else 0)
        out.append((c, c + k))
        c += k
    return out


class EegEngine:
    """One rank's share of an EEG lead-field build with inputs resident in HBM."""

    def __init__(self, mesh, electrodes, G, cfg=PcgConfig(), B=None, C=None, R=None,
                 columns=None, dev=None):
        """G: n x ncols (scipy / ndarray), G' already in HBM (DeviceCsr, ncols x n), or a
        SourceSpace, in which case G' is assembled on the device (fem.py:391-422)."""
        dev = dev or device()
        self.cfg = cfg
        self.h2d_bytes = 0
        self.dmesh = DeviceMesh.of(mesh)  # once per mesh object (G' assembly reuses it)
        self.h2d_bytes += self.dmesh.nodes.numel() * 8 + self.dmesh.tetra.numel() * 4
        self.sigma = to_device(mesh.sigma, np.float64, dev, slot=2)
        self.h2d_bytes += self.sigma.numel() * 8
        if B is None or C is None or R is None:
            B, C, R = model.assemble_B_C_R(mesh, electrodes)
        self.L = B.shape[1]
        self.n = mesh.n_nodes if hasattr(mesh, "n_nodes") else len(mesh.nodes)
        from .topology import ground_node_device

        self.ground = ground_node_device(mesh, electrodes)
        tri, coef = model.electrode_contacts(electrodes)
        self.etri = torch.from_numpy(np.ascontiguousarray(tri, dtype=np.int32)).to(dev)
        self.ecoef = torch.from_numpy(np.ascontiguousarray(coef, dtype=np.float64)).to(dev)
        self.h2d_bytes += tri.size * 4 + coef.nbytes
        self.c0, self.c1 = columns if columns is not None else (0, self.L)
        Bc = sp.csc_matrix(B)[:, self.c0:self.c1]
        self.Bd = rhs_block(Bc, dev=dev)
        self.Bt = DeviceCsr.from_scipy(sp.csr_matrix(sp.csr_matrix(B).T), dev)
        self.Cdiag = torch.from_numpy(np.ascontiguousarray(C.diagonal(), dtype=np.float64)).to(dev)
        self.R = np.asarray(R, dtype=np.float64)
        if G is None:  # EIT: no source matrix
            self.Gt, self.ncols = None, 0
        elif isinstance(G, DeviceCsr):  # already G' in HBM (topology.assemble_Gt_device)
            self.Gt = G
            self.ncols = G.shape[0]
        elif hasattr(G, "element_ids"):  # a SourceSpace: assemble G' on the device
            from .topology import assemble_Gt_device

            self.Gt = assemble_Gt_device(mesh, G)
            self.ncols = self.Gt.shape[0]
            self.h2d_bytes += 4 * len(G.element_ids)
        else:
            Gs = G if sp.issparse(G) else sp.csr_matrix(np.asarray(G, dtype=float))
            self.Gt = DeviceCsr.from_scipy(sp.csr_matrix(Gs.T), dev)
            self.ncols = Gs.shape[1]
        self.mesh = mesh
        self.B = sp.csr_matrix(B)
        self._op = None
        gnnz = self.Gt.nnz if self.Gt is not None else 0
        self.h2d_bytes += (Bc.nnz * 20 + self.Bt.nnz * 12 + gnnz * 12 + 8 * self.L
                           + 4 * (self.n + 1) + 4 * (self.ncols + 1) + 4 * (self.L + 1))
        self.last_info = None

    # ---- stages -------------------------------------------------------------
    def assemble(self):
        blocks = blocks_device(self.dmesh, self.sigma, 0.0)
        return assemble_device(self.dmesh, blocks, self.n, self.etri, self.ecoef, self.ground)

    def operator(self, A):
        if self._op is None or self._op.A is not A:
            op = PcgOperator(A, self.cfg.preconditioner)
            if op.n_zero_rows:
                from .errors import SingularPreconditionerError
                raise SingularPreconditionerError(f"{op.n_zero_rows} zero row(s) in the operator")
            self._op = op
        return self._op

    def solve(self, A):
        T, info = solve_block(self.operator(A), self.Bd, self.cfg)
        self.last_info = info
        try:
            _raise_failed(info, T, self.cfg, column_tag=True)
        except Exception as exc:  # the global electrode index, as transfer_matrix reports it
            if hasattr(exc, "column"):
                exc.column = self.c0 + exc.column
            raise
        return T

    def solve_rhs(self, A, rhs):
        """A^-1 rhs for a host n x k block with pcg_solve semantics (no column tag):
        the EIT pattern solves u_p = A^-1 B M^-1 I_p (leadfield.py:223-227)."""
        Rd = rhs_block(np.asarray(rhs, dtype=np.float64), dev=self.Bd.device)
        U, info = solve_block(self.operator(A), Rd, self.cfg)
        _raise_failed(info, U, self.cfg, column_tag=False)
        return U

    def eit_partial(self, dofs, T, U, W):
        """This rank's share of the EIT Jacobian: W[:, block] Q_block[p]' stacked over
        patterns (P*L x n_dofs), Q_block = T_block' K_m u_p (leadfield.py:179-207, 230-237)."""
        from .leadfield import eit_columns_device

        return eit_columns_device(self.mesh, dofs, self.ground, T, U, W, self.c0)

    def response_block(self, T):
        return response_block_device(self.Bt, T, self.L, self.Cdiag, self.c0)

    def lf_partial(self, T, W):
        if self.Gt is None:
            from .errors import SingularSystemError
            raise SingularSystemError("no source matrix G on this engine")
        return lf_tail_device(T, self.Gt, np.ascontiguousarray(W[:, self.c0:self.c1]))

    # ---- single-rank build --------------------------------------------------
    def build(self, to_host=False):
        """Whole LF build on this device (requires every column: columns=(0, L))."""
        if (self.c0, self.c1) != (0, self.L):
            raise ValueError("build() needs all electrode columns; use distributed.eeg_leadfield_sharded")
        A = self.assemble()
        T = self.solve(A)
        M = symmetrize(self.response_block(T).cpu().numpy())
        W = response_operator(M, self.R)
        LF = self.lf_partial(T, W)
        return _to_host(LF.contiguous()) if to_host else LF


def eeg_leadfield_from_mesh(mesh, electrodes, sources, cfg=PcgConfig()):
    """Host mesh, electrodes and sources (a SourceSpace, or G itself) in, host
    lead field (L x ncols) out: assemble_cem_system + eeg_leadfield in one call."""
    return EegEngine(mesh, electrodes, sources, cfg).build(to_host=True)
