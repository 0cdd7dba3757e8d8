"""Slab decomposition and exchange schedule for grids too large for one B200
(2048x2048x64 across 2/4/8 GPUs of one box).

One rank per GPU. Rank r owns the z-slab [z0, z1) of M and H (y-slabs when nz < P) and, in
Fourier space, the kx column range [k0, k1) of the half spectrum. One step of the sharded
pipeline is:

    KX  on the local rows            -> S_local[kx][c][z in slab][y]     (all Xh columns)
    transpose_forward  (all-to-all)  -> S_cols[kx in range][c][z][y]     (all nz planes)
    KYZ on the local kx columns      (y/z FFTs, tensor MAC, inverse: no communication)
    transpose_backward (all-to-all)  -> S_local
    KXI on the local rows            -> H_demag slab
    halo_exchange of M (one plane per neighbour), then K6 on the slab

The exchanges go through torch.distributed (NCCL over NVLink on GPUs; gloo in the CPU tests).
This module holds only the partition and the communication; the per-rank compute is the
same kernels as the single-GPU path, applied to a sub-grid.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple


def _split(n: int, p: int) -> List[Tuple[int, int]]:
    """Contiguous near-equal ranges covering [0, n)."""
    base, extra = divmod(n, p)
    out, s = [], 0
    for r in range(p):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


def padded_len(n: int) -> int:
    if n == 1:
        return 1
    L = 1
    while L < 2 * n - 1:
        L <<= 1
    return L


@dataclass
class SlabPlan:
    nx: int
    ny: int
    nz: int
    world: int
    slabs: List[Tuple[int, int]]     # z (or y) range per rank
    cols: List[Tuple[int, int]]      # kx range per rank
    axis: str                        # "z" or "y"

    @property
    def xh(self) -> int:
        lx = padded_len(self.nx)
        return 1 if lx == 1 else lx // 2 + 1

    def slab(self, r: int) -> Tuple[int, int]:
        return self.slabs[r]

    def nslab(self, r: int) -> int:
        a, b = self.slabs[r]
        return b - a

    def ncols(self, r: int) -> int:
        a, b = self.cols[r]
        return b - a

    def rows_per_plane(self) -> int:
        """Complex values of one (kx, c, plane) row in the spectrum scratch."""
        return self.ny if self.axis == "z" else self.nz

    # all-to-all element counts (complex values) for the forward transpose of rank r
    def send_counts_forward(self, r: int) -> List[int]:
        return [self.ncols(q) * 3 * self.nslab(r) * self.rows_per_plane() for q in range(self.world)]

    def recv_counts_forward(self, r: int) -> List[int]:
        return [self.ncols(r) * 3 * self.nslab(q) * self.rows_per_plane() for q in range(self.world)]

    def halo_neighbours(self, r: int) -> Tuple[int, int]:
        """Ranks owning the plane below / above the slab (-1 at the open boundary)."""
        lo = r - 1 if r > 0 and self.nslab(r - 1) > 0 else -1
        hi = r + 1 if r + 1 < self.world and self.nslab(r + 1) > 0 else -1
        return lo, hi

    def bytes_per_step(self, w: int) -> dict:
        """Per-rank NVLink bytes per step: two transposes and the M halo."""
        r = 0
        a2a = sum(c for q, c in enumerate(self.send_counts_forward(r)) if q != r) * 2 * w
        plane = self.nx * (self.ny if self.axis == "z" else self.nz) * 3 * w
        return {"transpose_each_way": a2a, "transposes": 2 * a2a, "halo": 2 * plane}


def plan(nx: int, ny: int, nz: int, world: int) -> SlabPlan:
    if world < 1:
        raise ValueError("world size must be >= 1")
    axis = "z" if nz >= world else "y"
    slabs = _split(nz if axis == "z" else ny, world)
    lx = padded_len(nx)
    xh = 1 if lx == 1 else lx // 2 + 1
    cols = _split(xh, world)
    return SlabPlan(nx, ny, nz, world, slabs, cols, axis)


# ------------------------------------------------------------------ communication
def transpose_forward(p: SlabPlan, rank: int, s_local, group=None):
    """s_local: complex tensor [Xh, 3, nslab, R] (R = ny for z-slabs) in kx-major order.
    Returns the rank's kx columns with all planes: [ncols, 3, nplanes_total, R]."""
    import torch
    import torch.distributed as dist
    xh, R = p.xh, p.rows_per_plane()
    assert tuple(s_local.shape) == (xh, 3, p.nslab(rank), R), s_local.shape
    parts = [s_local[a:b].reshape(-1) for a, b in p.cols]
    send = torch.view_as_real(torch.cat(parts)).reshape(-1)
    recv_counts = p.recv_counts_forward(rank)
    recv = torch.empty(2 * sum(recv_counts), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, [2 * c for c in recv_counts],
                           [2 * c for c in p.send_counts_forward(rank)], group=group)
    recv = torch.view_as_complex(recv.reshape(-1, 2))
    ncols = p.ncols(rank)
    nplanes = p.nz if p.axis == "z" else p.ny
    out = torch.empty((ncols, 3, nplanes, R), dtype=recv.dtype, device=recv.device)
    off = 0
    for q in range(p.world):
        a, b = p.slabs[q]
        cnt = recv_counts[q]
        out[:, :, a:b, :] = recv[off:off + cnt].reshape(ncols, 3, b - a, R)
        off += cnt
    return out


def transpose_backward(p: SlabPlan, rank: int, s_cols, group=None):
    """Inverse of transpose_forward: [ncols, 3, nplanes, R] -> [Xh, 3, nslab, R]."""
    import torch
    import torch.distributed as dist
    R = p.rows_per_plane()
    parts = [s_cols[:, :, a:b, :].reshape(-1) for a, b in p.slabs]
    send = torch.view_as_real(torch.cat(parts)).reshape(-1)
    send_counts = p.recv_counts_forward(rank)   # mirror of the forward exchange
    recv_counts = p.send_counts_forward(rank)
    recv = torch.empty(2 * sum(recv_counts), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, [2 * c for c in recv_counts], [2 * c for c in send_counts],
                           group=group)
    recv = torch.view_as_complex(recv.reshape(-1, 2))
    out = torch.empty((p.xh, 3, p.nslab(rank), R), dtype=recv.dtype, device=recv.device)
    off = 0
    for q, (a, b) in enumerate(p.cols):
        cnt = recv_counts[q]
        out[a:b] = recv[off:off + cnt].reshape(b - a, 3, p.nslab(rank), R)
        off += cnt
    return out


# ------------------------------------------------------------------ chunked zero-copy exchange
# Mirror of csrc/shard.cu's default exchange (ShardSolver::exchange_chunk / chunk_rows): each
# rank's kx columns are split into `nch` chunks; in chunk j every rank sends each peer q the
# contiguous S_local range of q's chunk-j columns and receives each peer's planes of its own
# chunk-j columns into that peer's receive block [ncols][3][nslab_q][R] (no packing, no
# placement); the y/z kernels read and write rows in place through the row map below.
def column_chunks(p: SlabPlan, nch: int) -> List[List[Tuple[int, int]]]:
    """[rank][chunk] local column range; ranks with fewer columns than chunks get empty tails."""
    out = []
    for q in range(p.world):
        nc = p.ncols(q)
        ch = _split(nc, min(nch, nc)) if nc else []
        out.append(ch + [(nc, nc)] * (nch - len(ch)))
    return out


def recv_offsets(p: SlabPlan, r: int) -> List[int]:
    """Start (complex elements) of peer q's block in rank r's receive buffer (q != r)."""
    off, out = 0, []
    for q in range(p.world):
        out.append(off)
        if q != r:
            off += p.ncols(r) * 3 * p.nslab(q) * p.rows_per_plane()
    return out


def chunk_exchange_ops(p: SlabPlan, r: int, j: int, nch: int):
    """Rank r's point-to-point operations of chunk j's forward exchange: per peer q,
    (q, (start, count) in r's S_local sent to q, (start, count) in r's receive buffer filled by
    q). The backward exchange sends the second range and receives into the first."""
    ch = column_chunks(p, nch)
    R = p.rows_per_plane()
    roff = recv_offsets(p, r)
    a, b = ch[r][j]
    ops = []
    for q in range(p.world):
        if q == r:
            continue
        qa, qb = ch[q][j]
        send = ((p.cols[q][0] + qa) * 3 * p.nslab(r) * R, (qb - qa) * 3 * p.nslab(r) * R)
        recv = (roff[q] + a * 3 * p.nslab(q) * R, (b - a) * 3 * p.nslab(q) * R)
        ops.append((q, send, recv))
    return ops


def chunk_row(p: SlabPlan, r: int, j: int, nch: int, kx: int, c: int, z: int) -> Tuple[str, int]:
    """Where row (kx, c, z) of rank r's chunk-j launch lives (RowMap::row of chunk_rows):
    ("s_local", offset) for r's own planes, ("recv", offset) for a peer's."""
    a = column_chunks(p, nch)[r][j][0]
    q = 0
    while z >= p.slabs[q][1]:
        q += 1
    z0, R = p.slabs[q][0], p.rows_per_plane()
    if q == r:
        return "s_local", ((p.cols[r][0] + a + kx) * 3 + c) * p.nslab(r) * R + (z - z0) * R
    return "recv", recv_offsets(p, r)[q] + (((a + kx) * 3 + c) * p.nslab(q) + (z - z0)) * R


# ------------------------------------------------------------------ peer-memory mode
def peer_row(p: SlabPlan, rank: int, kx_local: int, c: int, z: int) -> Tuple[int, int]:
    """Where row (kx_local, c, z) of rank `rank`'s columns lives in peer mode (MMB_SHARD_PEER,
    csrc/fast.hpp RowMap::row): (owning rank q, complex-element offset into q's flat
    S_local [Xh][3][nslab_q][R])."""
    q = 0
    while z >= p.slabs[q][1]:
        q += 1
    z0 = p.slabs[q][0]
    k = p.cols[rank][0] + kx_local
    return q, ((k * 3 + c) * p.nslab(q) + (z - z0)) * p.rows_per_plane()


def gather_columns_from_peers(p: SlabPlan, rank: int, s_locals):
    """The [ncols, 3, nplanes, R] column block of `rank` read row by row from every rank's
    S_local (s_locals[q], flat or [Xh, 3, nslab_q, R]): what the peer-mode y/z kernels load
    instead of the transpose_forward output."""
    import torch
    flat = [s.reshape(-1) for s in s_locals]
    R = p.rows_per_plane()
    nplanes = p.nz if p.axis == "z" else p.ny
    out = torch.empty((p.ncols(rank), 3, nplanes, R), dtype=flat[0].dtype)
    for k in range(p.ncols(rank)):
        for c in range(3):
            for z in range(nplanes):
                q, off = peer_row(p, rank, k, c, z)
                out[k, c, z] = flat[q][off:off + R]
    return out


def scatter_columns_to_peers(p: SlabPlan, rank: int, s_cols, s_locals):
    """Write `rank`'s processed column rows back into every rank's S_local in place (the
    peer-mode y/z kernels' stores, replacing transpose_backward)."""
    flat = [s.reshape(-1) for s in s_locals]
    R = p.rows_per_plane()
    for k in range(s_cols.shape[0]):
        for c in range(3):
            for z in range(s_cols.shape[2]):
                q, off = peer_row(p, rank, k, c, z)
                flat[q][off:off + R] = s_cols[k, c, z]


def halo_exchange(p: SlabPlan, rank: int, m_slab, group=None):
    """m_slab: [3, nslab, ...] (slab axis second). Returns (plane_below, plane_above): the
    neighbours' boundary planes of M (None at the open boundary), for the exchange stencil's
    z (or y) neighbours with Neumann boundaries at the global ends."""
    import torch
    import torch.distributed as dist
    lo, hi = p.halo_neighbours(rank)
    ops, below, above = [], None, None
    if lo >= 0:
        below = torch.empty_like(m_slab[:, 0])
        ops.append(dist.P2POp(dist.isend, m_slab[:, 0].contiguous(), lo, group=group))
        ops.append(dist.P2POp(dist.irecv, below, lo, group=group))
    if hi >= 0:
        above = torch.empty_like(m_slab[:, -1])
        ops.append(dist.P2POp(dist.isend, m_slab[:, -1].contiguous(), hi, group=group))
        ops.append(dist.P2POp(dist.irecv, above, hi, group=group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return below, above
