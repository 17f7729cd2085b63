"""Multi-process exchange geometry of distributed.solve_partitioned, on CPU (gloo).

The GPU path packs with a kernel and moves blocks with NCCL all_to_all_single;
here the same split sizes and block layout run through gloo on CPU tensors
(packing with distributed.pack_blocks_reference), checked against the
reference's transpose oracle (test_solver.py:133-138): rank p's y-slab must be
values[:, y-range(p), :], and the inverse exchange must restore the z-slabs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_1912_03565_b200 as hb

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shape, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_1912_03565_b200 as hb
    from paper_1912_03565_b200 import distributed as hd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nz, ny, nx = shape
        values = torch.from_numpy(np.random.default_rng(5).standard_normal(shape))
        grid = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
        ex = hb.make_exchange_plan(grid, world)
        z0, z1 = ex.partition.z_ranges[rank]
        y0, y1 = ex.partition.y_ranges[rank]
        send = hd.pack_blocks_reference(values[z0:z1].contiguous(), ex)
        y_slab = hd.exchange_forward_collective(send, ex, rank)
        ok_fwd = torch.equal(y_slab, values[:, y0:y1, :])
        recv = hd.exchange_inverse_collective(y_slab.contiguous(), ex, rank)
        back = hd.unpack_blocks_reference(recv, ex, rank)
        ok_inv = torch.equal(back, values[z0:z1])
        s, r = hd.split_sizes(ex, rank)
        ok_vol = sum(s) == (z1 - z0) * ny * nx and sum(r) == nz * (y1 - y0) * nx
        out_q.put((rank, bool(ok_fwd), bool(ok_inv), bool(ok_vol)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (9, 7, 5)), (3, (10, 11, 4)), (2, (31, 31, 31))])
def test_alltoall_exchange_matches_transpose_oracle(world, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results = sorted(q.get(timeout=10) for _ in range(world))
    assert all(fwd and inv and vol for _, fwd, inv, vol in results), results


def test_split_sizes_match_exchange_plan_blocks():
    import paper_1912_03565_b200 as hb
    from paper_1912_03565_b200 import distributed as hd
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 1023, 1023, 1023)
    ex = hb.make_exchange_plan(g, 8)
    for rank in range(8):
        s, r = hd.split_sizes(ex, rank)
        assert s == [int(np.prod(ex.block_extents(rank, q))) for q in range(8)]
        assert r == [int(np.prod(ex.block_extents(p, rank))) for p in range(8)]
    assert list(hd.y_starts(ex)) == [0, 128, 256, 384, 512, 640, 768, 896, 1023]


def test_fused_block_geometry_predicate():
    """distributed.fused_blocks: the block transforms (no pack / unpack pass) apply
    exactly to the uniform exchange geometry — kp = (n_y + 1) / parts for every
    part, a multiple of 16, FFT-engine line lengths — which covers every BASELINE
    config at 2, 4 and 8 ranks; everything else keeps the pack kernels. The block
    sizes of mode_split_sizes are then parts equal blocks of kpz * n_x * kp."""
    from paper_1912_03565_b200 import distributed as hd
    mk = lambda nx, ny, nz: hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
    for n in (511, 1023, 2047):
        for parts in (2, 4, 8):
            ex = hb.make_exchange_plan(mk(n, n, n), parts)
            assert hd.fused_blocks(ex), (n, parts)
            kp = (n + 1) // parts
            for r in range(parts):
                z0, z1 = ex.partition.z_ranges[r]
                assert hd.mode_split_sizes(ex, r)[0] == [(z1 - z0) * n * kp] * parts
    assert not hd.fused_blocks(hb.make_exchange_plan(mk(1023, 1023, 1023), 3))   # ragged
    assert hd.fused_blocks(hb.make_exchange_plan(mk(1023, 1023, 1023), 1))       # one part
    assert not hd.fused_blocks(hb.make_exchange_plan(mk(1023, 100, 64), 4))      # not 2^p
    assert not hd.fused_blocks(hb.make_exchange_plan(mk(31, 31, 31), 2))         # DMMA sizes
    assert not hd.fused_blocks(hb.make_exchange_plan(mk(1023, 127, 64), 16))     # kp = 8
    assert hd.fused_blocks(hb.make_exchange_plan(mk(63, 255, 64), 16))           # kp = 16


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_mode_split_sizes_consistent(parts):
    """Mode-space exchange: what p sends to q is what q expects from p, blocks
    cover every (l, n, m) once (plus one pad column for odd y-counts)."""
    from paper_1912_03565_b200 import distributed as hd
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 37, 61, 29)
    ex = hb.make_exchange_plan(g, parts)
    sends = [hd.mode_split_sizes(ex, r)[0] for r in range(parts)]
    recvs = [hd.mode_split_sizes(ex, r)[1] for r in range(parts)]
    for p in range(parts):
        for q in range(parts):
            assert sends[p][q] == recvs[q][p]
    kp = [((y1 - y0) + 1) & ~1 for y0, y1 in ex.partition.y_ranges]
    assert sum(map(sum, sends)) == g.n_z * g.n_x * sum(kp)
    assert sum(kp) - g.n_y == sum((y1 - y0) & 1 for y0, y1 in ex.partition.y_ranges)


@pytest.mark.parametrize("parts,chunks", [(1, 4), (2, 4), (3, 3), (8, 4), (5, 2)])
def test_chunk_layout_is_a_permutation(parts, chunks):
    from paper_1912_03565_b200 import distributed as hd
    g = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), 31, 47, 61)
    ex = hb.make_exchange_plan(g, parts)
    ranges, lp = hd.chunk_layout(ex, chunks)
    assert sorted(lp.tolist()) == list(range(g.n_z))
    for r, (z0, z1) in enumerate(ex.partition.z_ranges):
        assert ranges[r][0][0] == 0 and ranges[r][-1][1] == z1 - z0
    # per-chunk splits are consistent across ranks and add up to the unchunked ones
    for c in range(chunks):
        for p in range(parts):
            for q in range(parts):
                assert hd.chunk_split_sizes(ex, ranges, p, c)[0][q] == \
                    hd.chunk_split_sizes(ex, ranges, q, c)[1][p]
    for r in range(parts):
        tot = [sum(hd.chunk_split_sizes(ex, ranges, r, c)[0][q] for c in range(chunks))
               for q in range(parts)]
        assert tot == hd.mode_split_sizes(ex, r)[0]


# ------------------------------------------- transpose-free carry protocol
def _slab_sweep(w, table, cx, cy, z0, nz, recv_fwd, send_fwd, recv_bwd, send_bwd, blocks):
    """One rank's share of the distributed z-solve on its slab w (levels
    z0 .. z0 + len(w) - 1 of nz) with the carry protocol of
    csrc/thomas_carry.cu: forward (x', cp) at z0 - 1 arrives per column block
    from the previous rank and the slab's last level leaves per block to the
    next; the backward W at z1 arrives from the next rank and W at z0 leaves to
    the previous one. Same expression order as oracle.thomas_sweep."""
    A, B, C, D = table
    nzl = w.shape[0]
    cyc, cxr = cy[:, None], cx[None, :]

    def lam(l, k):
        return 4.0 * A[l, k] * (cyc * cxr) + 2.0 * B[l, k] * cxr + 2.0 * C[l, k] * cyc + D[l, k]

    cp = np.empty_like(w)
    c_in = np.zeros_like(w[0])
    for b0, b1 in blocks:  # forward, block by block
        cols = slice(b0, b1)
        if z0 > 0:
            x_prev, c_prev = recv_fwd(b1 - b0, w.shape[1])
            c_in[:, cols] = c_prev
        for i in range(nzl):
            l = z0 + i
            lo = lam(l, 0)[:, cols]
            if l == 0:
                r = 1.0 / lam(l, 1)[:, cols]
                w[i, :, cols] = w[i, :, cols] * r
            else:
                cprev = c_prev if i == 0 else cp[i - 1, :, cols]
                r = 1.0 / (lam(l, 1)[:, cols] - lo * cprev)
                xp = x_prev if i == 0 else w[i - 1, :, cols]
                w[i, :, cols] = (w[i, :, cols] - lo * xp) * r
            if l < nz - 1:
                cp[i, :, cols] = lam(l, 2)[:, cols] * r
        if z0 + nzl < nz:
            send_fwd(w[nzl - 1, :, cols], cp[nzl - 1, :, cols])
    for b0, b1 in blocks:  # backward
        cols = slice(b0, b1)
        top = nzl - 1
        if z0 + nzl < nz:
            w_next = recv_bwd(b1 - b0, w.shape[1])
            w[top, :, cols] -= cp[top, :, cols] * w_next
        for i in range(top - 1, -1, -1):
            w[i, :, cols] -= cp[i, :, cols] * w[i + 1, :, cols]
        if z0 > 0:
            send_bwd(w[0, :, cols])
    return w


def _carry_worker(rank, world, port, shape, nblocks, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_1912_03565_b200 as hb
    from oracle import helm_oracle as orc
    from paper_1912_03565_b200 import distributed as hd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nz, ny, nx = shape
        grid = hb.make_grid(hb.Domain(0, 1, 0, 1, 0, 1), nx, ny, nz)
        k2 = -30.0 * (1 + 0.5 * np.sin(np.pi * np.linspace(0, 1, nz + 2)))
        table = orc.weight_table("4", k2, np.zeros(nz + 2), np.zeros(nz + 2), 0.0,
                                 (grid.h_x, grid.h_y, grid.h_z), nz)
        cx, cy = orc.mode_cosines(nx, ny)
        F = np.random.default_rng(9).standard_normal(shape)
        ex = hb.make_exchange_plan(grid, world)
        z0, z1 = ex.partition.z_ranges[rank]
        prev, nxt = hd.carry_neighbours(rank, world)
        cuts = [round(b * nx / nblocks) for b in range(nblocks + 1)]
        blocks = [(cuts[b], cuts[b + 1]) for b in range(nblocks) if cuts[b + 1] > cuts[b]]

        def recv_fwd(cols, rows):
            t = torch.empty((2, rows, cols), dtype=torch.float64)
            dist.recv(t, src=prev)
            return t[0].numpy(), t[1].numpy()

        def send_fwd(x, c):
            dist.send(torch.from_numpy(np.stack([x, c])), dst=nxt)

        def recv_bwd(cols, rows):
            t = torch.empty((rows, cols), dtype=torch.float64)
            dist.recv(t, src=nxt)
            return t.numpy()

        def send_bwd(wv):
            dist.send(torch.from_numpy(np.ascontiguousarray(wv)), dst=prev)

        mine = _slab_sweep(F[z0:z1].copy(), table, cx, cy, z0, nz, recv_fwd, send_fwd,
                           recv_bwd, send_bwd, blocks)
        ref = orc.thomas_sweep(F.copy(), table, cx, cy)[z0:z1]
        out_q.put((rank, bool(np.array_equal(mine, ref)), (prev, nxt)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,nblocks", [(2, (12, 7, 9), 3), (3, (10, 5, 16), 4),
                                                 (4, (9, 6, 6), 2)])
def test_carry_protocol_matches_global_thomas(world, shape, nblocks):
    """The transpose-free distributed z-solve's protocol on CPU ranks (gloo):
    every rank sweeps only its z-slab, the (x', cp) / W carries move per column
    block between neighbours, and the result equals the single-process Thomas
    sweep of the oracle bit for bit (tridiag.py:126-167 arithmetic)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_carry_worker, args=(r, world, port, shape, nblocks, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok, _ in res)
    assert [nb for _, _, nb in res] == [((r - 1) if r else None, (r + 1) if r + 1 < world else None)
                                        for r in range(world)]
