"""Multi-rank host path on CPU: world_size-2 (and 3) gloo runs of the slab-decomposed demag
convolution (paper_1501_07293_b200/shard.py: partition, forward/backward all-to-all transpose,
halo exchange) with NumPy FFTs standing in for the per-rank kernels; the gathered field must
equal the single-process oracle (the reference's DemagSolver restated) to FFT round-off."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mmsim_oracle as O
from paper_1501_07293_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _wrapped_tensor_spectrum(g, lx, ly, lz):
    oz = np.arange(-(g.nz - 1), g.nz)
    oy = np.arange(-(g.ny - 1), g.ny)
    ox = np.arange(-(g.nx - 1), g.nx)
    K, J, I = np.meshgrid(oz, oy, ox, indexing="ij")
    comps = O.tensor_entry(I, J, K, g.delta)
    out = []
    for c in range(6):
        t = np.zeros((lz, ly, lx))
        t[K % lz, J % ly, I % lx] = comps[c]
        out.append(np.fft.rfftn(t))
    return np.stack(out)  # [6, lz, ly, xh]


def _rank_main(rank, world, port, nx, ny, nz, delta, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = O.Grid(nx, ny, nz, delta)
        p = shard.plan(nx, ny, nz, world)
        assert p.axis == "z"
        lx, ly, lz = shard.padded_len(nx), shard.padded_len(ny), shard.padded_len(nz)
        rng = np.random.default_rng(7)
        m = rng.uniform(-800, 800, (3, nz, ny, nx))
        z0, z1 = p.slab(rank)
        m_slab = m[:, z0:z1]
        # KX stand-in: r2c along x on the local rows, kx-major [Xh, 3, nslab, ny]
        s_local = np.fft.rfft(m_slab, n=lx, axis=-1).transpose(3, 0, 1, 2).copy()
        cols = shard.transpose_forward(p, rank, torch.from_numpy(s_local)).numpy()
        k0, k1 = p.cols[rank]
        spec = _wrapped_tensor_spectrum(g, lx, ly, lz)[:, :, :, k0:k1]  # [6, lz, ly, ncols]
        # KYZ stand-in: y/z FFTs of the live planes, MAC, inverse, crop
        a = np.fft.fftn(cols, s=(lz, ly), axes=(2, 3))  # [ncols, 3, lz, ly]
        kk = spec.transpose(0, 3, 1, 2)                   # [6, ncols, lz, ly]
        rows = ((0, 1, 2), (1, 3, 4), (2, 4, 5))
        h = np.stack([sum(kk[rows[c][j]] * a[:, j] for j in range(3)) for c in range(3)], axis=1)
        h = np.fft.ifftn(h, axes=(2, 3))[:, :, :nz, :ny]
        back = shard.transpose_backward(p, rank, torch.from_numpy(np.ascontiguousarray(h))).numpy()
        # KXI stand-in
        h_slab = np.fft.irfft(back.transpose(1, 2, 3, 0), n=lx, axis=-1)[..., :nx]
        # halo exchange of M
        below, above = shard.halo_exchange(p, rank, torch.from_numpy(np.ascontiguousarray(m_slab)))
        ok_halo = True
        if below is not None:
            ok_halo &= np.array_equal(below.numpy(), m[:, z0 - 1])
        if above is not None:
            ok_halo &= np.array_equal(above.numpy(), m[:, z1])
        full = [torch.zeros(1) for _ in range(world)]
        dist.all_gather_object(full, (z0, z1, h_slab, ok_halo))
        if rank == 0:
            hh = np.zeros((3, nz, ny, nx))
            halos = True
            for a_, b_, hs, okh in full:
                hh[:, a_:b_] = hs
                halos &= okh
            want = O.demag_field_fft(m, g)
            q.put((O.max_relative_error(hh, want), halos, p.bytes_per_step(4)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (12, 10, 6)), (3, (9, 7, 7)), (2, (16, 8, 2))])
def test_sharded_demag_equals_single_process(world, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, *shape, 2.0, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    err, halos, nbytes = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert err <= 1e-12
    assert halos
    assert nbytes["transposes"] > 0


def test_plan_partitions_and_counts():
    p = shard.plan(2048, 2048, 64, 8)
    assert p.axis == "z" and [b - a for a, b in p.slabs] == [8] * 8
    assert sum(p.ncols(r) for r in range(8)) == 2049
    for r in range(8):
        assert sum(p.send_counts_forward(r)) == p.xh * 3 * p.nslab(r) * 2048
        assert sum(p.recv_counts_forward(r)) == p.ncols(r) * 3 * 64 * 2048
    # nz < P falls back to y-slabs
    assert shard.plan(64, 64, 2, 4).axis == "y"
    b = p.bytes_per_step(4)
    # f32: each rank ships 7/8 of its 1/8 share of the 6.4 GB half spectrum each way
    assert abs(b["transpose_each_way"] - 2049 * 3 * 8 * 2048 * 8 * 7 / 8) < 2049 * 3 * 8 * 2048 * 8


def _peer_rank_main(rank, world, port, nx, ny, nz, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = shard.plan(nx, ny, nz, world)
        gen = torch.Generator().manual_seed(7 + rank)
        mine = torch.complex(torch.randn(p.xh, 3, p.nslab(rank), ny, generator=gen, dtype=torch.float64),
                             torch.randn(p.xh, 3, p.nslab(rank), ny, generator=gen, dtype=torch.float64))
        # every rank's S_local, as the IPC-mapped peer views would show them
        sizes = [p.xh * 3 * p.nslab(r) * ny for r in range(world)]
        flat = torch.view_as_real(mine.reshape(-1)).reshape(-1)
        padded = [torch.empty(2 * max(sizes), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(padded, torch.nn.functional.pad(flat, (0, 2 * max(sizes) - flat.numel())))
        locals_ = [torch.view_as_complex(padded[r][:2 * sizes[r]].reshape(-1, 2)).clone() for r in range(world)]
        cols_t = shard.transpose_forward(p, rank, mine)
        cols_p = shard.gather_columns_from_peers(p, rank, locals_)
        ok_fwd = torch.equal(cols_t, cols_p)
        # write back a transformed block both ways
        new_cols = cols_t * (2.0 - 1.0j) + 0.5
        back_t = shard.transpose_backward(p, rank, new_cols)
        # each rank scatters its own columns into copies of all slabs; gather rank's slab back
        copies = [l.clone() for l in locals_]
        obj = [None] * world
        dist.all_gather_object(obj, new_cols)
        for r in range(world):
            shard.scatter_columns_to_peers(p, r, obj[r], copies)
        ok_bwd = torch.equal(copies[rank].reshape(back_t.shape), back_t)
        q.put((rank, ok_fwd, ok_bwd))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (12, 6, 5)), (3, (9, 4, 7))])
def test_peer_rows_equal_the_transposes(world, shape):
    """Peer mode (MMB_SHARD_PEER): the rows the y/z kernels read from / write to the peers'
    slab spectra (RowMap) are exactly the all-to-all transposes' blocks, on world 2 and 3
    gloo ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_rank_main, args=(r, world, port, *shape, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(ok_f and ok_b for _, ok_f, ok_b in res), res


def _chunk_rank_main(rank, world, port, nx, ny, nz, nch, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = shard.plan(nx, ny, nz, world)
        gen = torch.Generator().manual_seed(11 + rank)
        mine = torch.complex(torch.randn(p.xh, 3, p.nslab(rank), ny, generator=gen, dtype=torch.float64),
                             torch.randn(p.xh, 3, p.nslab(rank), ny, generator=gen, dtype=torch.float64))
        s_local = mine.reshape(-1).clone()
        roff = shard.recv_offsets(p, rank)
        nrecv = sum(p.ncols(rank) * 3 * p.nslab(qq) * ny for qq in range(world) if qq != rank)
        recv = torch.zeros(max(nrecv, 1), dtype=torch.complex128)
        want_cols = shard.transpose_forward(p, rank, mine)          # [ncols, 3, nz, ny]
        new_cols = want_cols * (2.0 - 1.0j) + 0.5
        want_back = shard.transpose_backward(p, rank, new_cols)
        chunks = shard.column_chunks(p, nch)
        ok_fwd = True

        def exchange(j, backward):
            ops = []
            for peer, (ss, sc), (rs, rc) in shard.chunk_exchange_ops(p, rank, j, nch):
                src, dst = (s_local[ss:ss + sc], recv[rs:rs + rc]) if not backward else \
                    (recv[rs:rs + rc], s_local[ss:ss + sc])
                if src.numel():
                    ops.append(dist.P2POp(dist.isend, torch.view_as_real(src.contiguous()), peer))
                bufs = torch.view_as_real(torch.empty_like(dst)) if dst.numel() else None
                if bufs is not None:
                    ops.append(dist.P2POp(dist.irecv, bufs, peer))
                    ops_dst.append((dst, bufs))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()

        for j in range(nch):
            ops_dst = []
            exchange(j, False)
            for dst, buf in ops_dst:
                dst.copy_(torch.view_as_complex(buf))
            a, b = chunks[rank][j]
            # the y/z stand-in: gather the chunk's rows through the row map, compare, transform,
            # write back in place
            for kx in range(b - a):
                for c in range(3):
                    for z in range(nz):
                        where, off = shard.chunk_row(p, rank, j, nch, kx, c, z)
                        buf = s_local if where == "s_local" else recv
                        row = buf[off:off + ny]
                        ok_fwd &= torch.equal(row, want_cols[a + kx, c, z])
                        buf[off:off + ny] = new_cols[a + kx, c, z]
        for j in range(nch):
            ops_dst = []
            exchange(j, True)
            for dst, buf in ops_dst:
                dst.copy_(torch.view_as_complex(buf))
        ok_bwd = torch.equal(s_local.reshape(want_back.shape), want_back)
        q.put((rank, bool(ok_fwd), bool(ok_bwd)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,nch", [(2, (12, 6, 5), 1), (2, (12, 6, 5), 3), (3, (9, 4, 7), 4),
                                             (3, (5, 4, 7), 7)])
def test_chunked_exchange_rows_equal_the_transposes(world, shape, nch):
    """The default sharded exchange (csrc/shard.cu exchange_chunk + chunk_rows, mirrored in
    shard.py): per column chunk, contiguous S_local ranges to each peer and one receive block
    per peer, rows addressed in place by the row map. On world 2 and 3 gloo ranks, the rows the
    y/z stage sees are the all-to-all transpose's, and the in-place results sent back are the
    backward transpose's, for 1..7 chunks (more chunks than a rank's columns included)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_rank_main, args=(r, world, port, *shape, nch, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(ok_f and ok_b for _, ok_f, ok_b in res), res
