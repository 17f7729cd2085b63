"""Multi-GPU partitioned solve: one process per GPU, NCCL all-to-all over NVLink.

The reference's Partitioned mode (solver.py:319-399) gives each part a z-slab
for the transforms and a y-slab (n_z, kpy, n_x) for the z-solves, with two
block transposes in between (exchange_forward / exchange_inverse,
solver.py:146-201). Here each part is a rank (``torch.distributed``, backend
"nccl" on GPUs, "gloo" in the CPU tests of the exchange geometry):

  1. 2D DST-I of the local z-slab (kpz planes)              [sm_100a kernels]
  2. pack z_slab[:, y-range(q), :] blocks, ascending q      [pack kernel]
  3. all_to_all_single with the reference's uneven splits   [NCCL]
     -> the received buffer IS the y-slab (blocks land contiguously at
        y_slab[z-range(p)], solver.py:173)
  4. per-mode Thomas on the y-slab, mode offset y0          [sm_100a kernel]
  5. inverse all_to_all (send y_slab[z-range(q)], contiguous)
  6. unpack into the z-slab, inverse 2D DST-I               [kernels]

Ranges come from the reference's plan_partition (larger chunks first), so
block extents are exactly (n_x, kpy(q), kpz(p)) as in ExchangePlan.
"""

import ctypes

import numpy as np

from ._native import check, get_plan, ptr
from .solver import make_exchange_plan
from .tridiag import device_coefficients


def split_sizes(ex, rank):
    """(send_splits_fwd, recv_splits_fwd) element counts for rank's forward exchange."""
    zr, yr = ex.partition.z_ranges, ex.partition.y_ranges
    kpz = zr[rank][1] - zr[rank][0]
    kpy = yr[rank][1] - yr[rank][0]
    send = [kpz * (y1 - y0) * ex.n_x for y0, y1 in yr]
    recv = [(z1 - z0) * kpy * ex.n_x for z0, z1 in zr]
    return send, recv


def y_starts(ex):
    return np.array([r[0] for r in ex.partition.y_ranges] + [ex.n_y], dtype=np.int32)


def pack_blocks_reference(z_slab, ex):
    """torch slicing version of the pack kernel (CPU tests / cross-check)."""
    import torch
    return torch.cat([z_slab[:, y0:y1, :].reshape(-1) for y0, y1 in ex.partition.y_ranges])


def unpack_blocks_reference(recv, ex, rank):
    """torch slicing version of the unpack kernel: recv blocks (kpz, kpy(q), n_x) -> z-slab."""
    import torch
    z0, z1 = ex.partition.z_ranges[rank]
    kpz = z1 - z0
    out = torch.empty((kpz, ex.n_y, ex.n_x), dtype=recv.dtype, device=recv.device)
    off = 0
    for y0, y1 in ex.partition.y_ranges:
        n = kpz * (y1 - y0) * ex.n_x
        out[:, y0:y1, :] = recv[off:off + n].view(kpz, y1 - y0, ex.n_x)
        off += n
    return out


def exchange_forward_collective(send, ex, rank, group=None):
    """Forward all-to-all; returns the y-slab (n_z, kpy, n_x)."""
    import torch
    import torch.distributed as dist
    s, r = split_sizes(ex, rank)
    y0, y1 = ex.partition.y_ranges[rank]
    recv = torch.empty(sum(r), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=r, input_split_sizes=s, group=group)
    return recv.view(ex.n_z, y1 - y0, ex.n_x)


def exchange_inverse_collective(y_slab, ex, rank, group=None):
    """Inverse all-to-all; returns the flat receive buffer of (kpz, kpy(q), n_x) blocks."""
    import torch
    import torch.distributed as dist
    s_fwd, r_fwd = split_sizes(ex, rank)
    recv = torch.empty(sum(s_fwd), dtype=y_slab.dtype, device=y_slab.device)
    dist.all_to_all_single(recv, y_slab.reshape(-1), output_split_sizes=s_fwd,
                           input_split_sizes=r_fwd, group=group)
    return recv


def solve_partitioned(z_slab, scheme, profile, grid, group=None, timings=None):
    """Solve with the grid split over the ranks of `group`; z_slab is this rank's
    (kpz, n_y, n_x) CUDA float64 part of the folded RHS. Returns the solution slab
    (a new tensor). Raises SingularSystemError on every rank if any rank hit a
    vanishing pivot."""
    import torch
    import torch.distributed as dist
    rank, parts = dist.get_rank(group), dist.get_world_size(group)
    ex = make_exchange_plan(grid, parts)
    z0, z1 = ex.partition.z_ranges[rank]
    y0, y1 = ex.partition.y_ranges[rank]
    kpz = z1 - z0
    if tuple(z_slab.shape) != (kpz, grid.n_y, grid.n_x):
        raise ValueError(f"z-slab shape {tuple(z_slab.shape)} != {(kpz, grid.n_y, grid.n_x)}")
    dev = z_slab.device
    tplan = get_plan(grid.n_x, grid.n_y, kpz, dev)
    zplan = get_plan(grid.n_x, grid.n_y, grid.n_z, dev)
    ys = y_starts(ex)
    ys_c = ys.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
    local = z_slab.contiguous().clone()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if timings is not None else None

    def mark(i):
        if ev is not None:
            ev[i].record()

    with tplan.lock, zplan.lock:
        device_coefficients(zplan, scheme, profile, grid)
        st = tplan.stream()
        wk = tplan.workspace(1)
        mark(0)
        check(tplan.lib.hfb_transform_stack(tplan.handle, ptr(local), 0, kpz, ptr(wk), st),
              "transform")
        send = torch.empty(local.numel(), dtype=local.dtype, device=dev)
        check(tplan.lib.hfb_pack_yblocks(tplan.handle, ptr(local), ptr(send), kpz, ys_c, parts,
                                         st), "pack")
        mark(1)
        y_slab = exchange_forward_collective(send, ex, rank, group).contiguous()
        mark(2)
        cpw = torch.empty_like(y_slab)
        check(zplan.lib.hfb_solve_slab(zplan.handle, ptr(y_slab), y1 - y0, y0, ptr(cpw),
                                       zplan.stream()), "solve_slab")
        mark(3)
        recv = exchange_inverse_collective(y_slab, ex, rank, group)
        mark(4)
        check(tplan.lib.hfb_unpack_yblocks(tplan.handle, ptr(recv), ptr(local), kpz, ys_c, parts,
                                           st), "unpack")
        check(tplan.lib.hfb_transform_stack(tplan.handle, ptr(local), 0, kpz, ptr(wk), st),
              "transform")
        mark(5)
        # agree on the first failing pivot across ranks
        flag = torch.zeros(1, dtype=torch.int64, device=dev)
        try:
            zplan.fetch_status()
        except Exception:
            flag.fill_(1)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        if int(flag.item()):
            from .errors import SingularSystemError
            raise SingularSystemError("vanishing pivot on at least one rank")
    if timings is not None:
        torch.cuda.synchronize(dev)
        timings.update(transform_s=(ev[0].elapsed_time(ev[1]) + ev[4].elapsed_time(ev[5])) / 1e3,
                       exchange_s=(ev[1].elapsed_time(ev[2]) + ev[3].elapsed_time(ev[4])) / 1e3,
                       tridiag_s=ev[2].elapsed_time(ev[3]) / 1e3)
    return local
