"""Device-resident sparse matrices and the prepared PCG operator.

Buffers are torch CUDA tensors (PyTorch is only the allocator/stream layer);
all arithmetic runs in libhfb200.so.  HBM layout:

* CSR as scipy stores it: int32 indptr (n+1), int32 indices (nnz, sorted per
  row), float64 values.  The parity copy keeps scipy's explicit zeros; the
  SpMM runs on a zero-free copy (`PcgOperator.Ac`).
* n-vector blocks are n x kp row-major float64 (kp columns of one node
  contiguous), kp in {2,...,64}.
"""
from __future__ import annotations

import threading

import numpy as np
import scipy.sparse as sp
import torch

from . import _native as N


def device():
    N.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


# Host -> device staging.  A pageable torch copy runs at 3-10 GB/s on the GPU
# box and the int64 -> int32 narrowing of a mesh's tetra is a single-threaded
# numpy pass; instead the host array is converted in parallel slices straight
# into a grow-only pinned buffer (numpy releases the GIL in copyto) and moved
# with one DMA.  The buffer is reused across calls; each copy is synchronous,
# so reuse never races a transfer in flight.
_PINNED = {}
_LOCK = threading.Lock()
_POOL = None
_WORKERS = 1


def _pool():
    global _POOL, _WORKERS
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor

        _WORKERS = max(1, min(8, os.cpu_count() or 1))
        _POOL = ThreadPoolExecutor(max_workers=_WORKERS)
    return _POOL


def _pinned(slot, nbytes):
    buf = _PINNED.get(slot)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        _PINNED[slot] = buf
    return buf


def to_host(t, slot=7):
    """Copy a device tensor to a new host numpy array through pinned staging
    (one DMA at full PCIe rate instead of a pageable copy)."""
    nbytes = t.numel() * t.element_size()
    if nbytes < (4 << 20):
        return t.cpu().numpy()
    with _LOCK:
        buf = _pinned(slot, nbytes)
        stage = torch.from_numpy(buf[:nbytes].numpy().view(np.dtype(str(t.dtype).replace("torch.", ""))))
        stage = stage.view(t.shape)
        stage.copy_(t)  # synchronous device -> pinned copy
        src = stage.numpy()
        out = np.empty(src.shape, dtype=src.dtype)
        flat_src, flat_dst = src.reshape(-1), out.reshape(-1)
        pool = _pool()
        step = -(-flat_src.size // (4 * _WORKERS))
        futs = [pool.submit(np.copyto, flat_dst[i:i + step], flat_src[i:i + step])
                for i in range(0, flat_src.size, step)]
        for f in futs:
            f.result()
        return out


def to_device(arr, dtype, dev=None, slot=0):
    """Copy a host array to a new device tensor of numpy dtype `dtype` via pinned staging."""
    dev = dev or device()
    a = np.asarray(arr)
    dt = np.dtype(dtype)
    nbytes = a.size * dt.itemsize
    if nbytes < (4 << 20):  # small: the plain path is cheaper than the pool
        return torch.from_numpy(np.array(a, dtype=dt, order="C")).to(dev)
    with _LOCK:  # one staging buffer per slot: concurrent callers take turns
        buf = _pinned(slot, nbytes)
        view = buf[:nbytes].numpy().view(dt).reshape(a.shape)
        flat_src, flat_dst = a.reshape(-1), view.reshape(-1)
        pool = _pool()
        step = -(-flat_src.size // (4 * _WORKERS))
        futs = [pool.submit(np.copyto, flat_dst[i:i + step], flat_src[i:i + step], casting="unsafe")
                for i in range(0, flat_src.size, step)]
        for f in futs:
            f.result()
        out = torch.empty(a.shape, dtype=torch.from_numpy(view[:0]).dtype, device=dev)
        out.copy_(torch.from_numpy(view))  # synchronous: the buffer is free again on return
    return out


class DeviceCsr:
    """A CSR matrix in HBM (int32 indptr/indices, float64 values)."""

    def __init__(self, indptr, indices, val, shape):
        self.indptr, self.indices, self.val = indptr, indices, val
        self.shape = (int(shape[0]), int(shape[1]))
        self._s = N.csr_struct(self.shape[0], self.shape[1], indptr, indices, val)

    @property
    def nnz(self):
        return int(self.indices.numel())

    @property
    def struct(self):
        return self._s

    @classmethod
    def from_scipy(cls, M, dev=None):
        dev = dev or device()
        M = sp.csr_matrix(M)
        if not M.has_sorted_indices:
            M = M.copy()
            M.sort_indices()
        # pinned staging (one DMA per array at full PCIe rate): the drop-in entry
        # points move the caller's scipy matrices on every call
        ip = to_device(M.indptr, np.int32, dev, slot=3)
        ix = to_device(M.indices, np.int32, dev, slot=4)
        vv = to_device(M.data, np.float64, dev, slot=5)
        return cls(ip, ix, vv, M.shape)

    def to_scipy(self):
        return sp.csr_matrix((self.val.cpu().numpy(), self.indices.cpu().numpy(),
                              self.indptr.cpu().numpy()), shape=self.shape)

    def pruned(self):
        """Zero-free copy (explicit zeros contribute +0*x, an exact no-op)."""
        n = self.shape[0]
        ws = torch.empty(N.lib.hf_csr_prune_workspace_bytes(n), dtype=torch.uint8, device=self.val.device)
        nnz = N.C.c_int64(0)
        st = N.stream_handle()
        N.check("hf_csr_prune_count",
                N.lib.hf_csr_prune_count(N.C.byref(self._s), N.ptr(ws), ws.numel(), N.C.byref(nnz), st))
        k = int(nnz.value)
        ip = torch.empty(n + 1, dtype=torch.int32, device=self.val.device)
        ix = torch.empty(max(k, 1), dtype=torch.int32, device=self.val.device)[:k]
        vv = torch.empty(max(k, 1), dtype=torch.float64, device=self.val.device)[:k]
        N.check("hf_csr_prune_fill",
                N.lib.hf_csr_prune_fill(N.C.byref(self._s), N.ptr(ws), ws.numel(), N.ptr(ip),
                                        N.ptr(ix), N.ptr(vv), st))
        return DeviceCsr(ip, ix, vv, self.shape)

    def transpose_scipy(self):
        return sp.csr_matrix(self.to_scipy().T)


def ldp_device(A: DeviceCsr):
    """(d, n_zero_rows) for d_i = sum_j |a_ij| (solver.py:50-61)."""
    n = A.shape[0]
    d = torch.empty(max(n, 1), dtype=torch.float64, device=A.val.device)[:n]
    scratch = torch.empty(1, dtype=torch.int32, device=A.val.device)
    nz = N.C.c_int32(0)
    N.check("hf_ldp", N.lib.hf_ldp(N.C.byref(A.struct), N.ptr(d), N.ptr(scratch), N.C.byref(nz),
                                   N.stream_handle()))
    return d, int(nz.value)


# bytes of the 126 MB L2 the SpMM's two-plane reuse window may take
L2_WINDOW = 48 << 20


class PcgOperator:
    """A prepared for the multi-RHS solver: parity CSR, zero-free SpMM copy and
    the preconditioner diagonal (computed once, not once per column as
    solver.py:77 does)."""

    def __init__(self, A: DeviceCsr, preconditioner="ldp"):
        if A.shape[0] != A.shape[1]:
            raise ValueError("matrix must be square")
        self.A = A
        self.n = A.shape[0]
        if preconditioner == "ldp":
            self.d, self.n_zero_rows = ldp_device(A)
        else:
            self.d = torch.ones(self.n, dtype=torch.float64, device=A.val.device)
            self.n_zero_rows = 0
        self.Ac = A.pruned()
        scratch = torch.empty(1, dtype=torch.int32, device=A.val.device)
        bw = N.C.c_int32(0)
        N.check("hf_csr_bandwidth", N.lib.hf_csr_bandwidth(N.C.byref(self.Ac.struct), N.ptr(scratch),
                                                           N.C.byref(bw), N.stream_handle()))
        self.bandwidth = int(bw.value)

    def batch_width(self, k, cap):
        """RHS columns per multi-RHS solve: `cap`, halved (not below 16) while the
        p and q rows one sweep reaches twice (about 2 x bandwidth rows each, kp
        doubles per row) would fill more than L2_WINDOW bytes of the 126 MB L2.
        C2 (bandwidth ~15k rows) keeps 64; the 5M-node C5 mesh (~35k) runs at 32,
        3% faster per column than 64 (its q/p window at 64 is 72 MB and its
        SpMM re-reads p from DRAM)."""
        w = cap
        while w > 16 and 4 * self.bandwidth * w * 8 > L2_WINDOW:
            w //= 2
        return min(w, k) if k > 0 else w


def width_for(k):
    for w in N.PCG_WIDTHS:
        if w >= k:
            return w
    return N.PCG_WIDTHS[-1]
