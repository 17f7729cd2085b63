"""Multi-GPU partitioned solve: one process per GPU, NCCL all-to-all over NVLink.

The reference's Partitioned mode (solver.py:319-399) gives each part a z-slab
for the transforms and a y-slab (n_z, kpy, n_x) for the z-solves, with two
block transposes in between (exchange_forward / exchange_inverse,
solver.py:146-201). Here each part is a rank (``torch.distributed``, backend
"nccl" on GPUs, "gloo" in the CPU tests of the exchange geometry):

  1. 2D DST-I of the local z-slab (kpz planes) into padded mode rows
     (l, n, m), then pack blocks (kpz, n_x, kp(q)), ascending q  [sm_100a kernels]
  2. all_to_all_single with the reference's uneven z/y splits   [NCCL]
     -> the received buffer IS the y-slab of mode rows (n_z, n_x, kp)
        (blocks land contiguously by sender z-range, as solver.py:173)
  3. TMA-streamed Thomas on the y-slab, mode offset y0          [sm_100a kernel]
  4. inverse all_to_all (the y-slab goes back as it came)
  5. unpack into the mode rows, inverse 2D DST-I                 [kernels]

(The reference's natural-layout blocks (kpz, kpy(q), n_x) are kept by
split_sizes / exchange_*_collective for the gloo tests of the geometry.)

solve_partitioned_carry is the transpose-free alternative:
the z-slab stays on its rank for the whole solve and the z-solve itself is
swept across the ranks, forward then backward, with O(n_x n_y) carries per
rank boundary moving through peer memory (csrc/thomas_carry.cu). It needs
no all-to-all, so it is not bound by the 2 (P-1) N^3 8 / P^2 bytes per GPU of
the exchange.

Ranges come from the reference's plan_partition (larger chunks first), so
block extents are exactly (n_x, kpy(q), kpz(p)) as in ExchangePlan.
"""

import ctypes
import os

import numpy as np

from ._native import HFB_ERR_EXCHANGE, check, get_plan, ptr
from ._native import check as _check  # for functions whose `check` argument shadows it
from .errors import ExchangeError
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


# The transforms write / read the exchange blocks themselves (hfb_forward_blocks,
# hfb_inverse_blocks: no pack / unpack pass) whenever the exchange geometry is
# uniform; False keeps the pack / unpack kernels everywhere (A/B and tests).
FUSED_BLOCKS = os.environ.get("HFB_FUSED_BLOCKS", "1") != "0"


def fused_blocks(ex):
    """True when the block transforms apply: every part owns kp = (n_y + 1) / parts
    y-modes (the last one kp - 1 plus the padding column), kp a multiple of 16, and
    both line lengths run on the FFT engine (n + 1 >= 64)."""
    if not FUSED_BLOCKS:
        return False
    kp, rem = divmod(ex.n_y + 1, ex.n_parts)
    if rem or kp % 16 or ex.n_x + 1 < 64 or ex.n_y + 1 < 64:
        return False
    return all(y0 == q * kp for q, (y0, _) in enumerate(ex.partition.y_ranges))


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


def mode_split_sizes(ex, rank):
    """(send, recv) element counts of the mode-space exchange (forward direction):
    the block from rank p to rank q is (kpz(p), n_x, kp(q)), kp(q) = the y-mode
    count of q rounded up to even (16-byte aligned mode rows)."""
    zr, yr = ex.partition.z_ranges, ex.partition.y_ranges
    kp = [((y1 - y0) + 1) & ~1 for y0, y1 in yr]
    kpz = zr[rank][1] - zr[rank][0]
    send = [kpz * ex.n_x * k for k in kp]
    recv = [(z1 - z0) * ex.n_x * kp[rank] for z0, z1 in zr]
    return send, recv


def forward_to_blocks(z_slab, grid, ex, rank):
    """Stage 1 (per rank): forward 2D DST of the z-slab into padded mode rows
    and pack the exchange blocks. Returns (send, modes)."""
    import torch
    z0, z1 = ex.partition.z_ranges[rank]
    kpz = z1 - z0
    dev = z_slab.device
    tplan = get_plan(grid.n_x, grid.n_y, kpz, dev)
    st = tplan.stream()
    ldm = int(tplan.lib.hfb_modes_ld(tplan.handle))
    modes = torch.empty(kpz * grid.n_x * ldm, dtype=torch.float64, device=dev)
    with tplan.lock:
        work = tplan.workspace(5)
        send = torch.empty(sum(mode_split_sizes(ex, rank)[0]), dtype=torch.float64, device=dev)
        ys = y_starts(ex)
        ysp = ys.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
        if fused_blocks(ex):  # `modes` stays scratch for the way back
            check(tplan.lib.hfb_forward_blocks(tplan.handle, ptr(z_slab), ptr(send), ptr(work),
                                               ysp, ex.n_parts, st), "forward_blocks")
        else:
            check(tplan.lib.hfb_forward_modes(tplan.handle, ptr(z_slab), ptr(modes), ptr(work),
                                              st), "forward_modes")
            check(tplan.lib.hfb_pack_modes(tplan.handle, ptr(modes), ptr(send), ysp, ex.n_parts,
                                           st), "pack_modes")
    return send, modes


def solve_received(recv, scheme, profile, grid, ex, rank):
    """Stage 2 (per rank): z-solve of the received y-slab of mode rows
    (n_z, n_x, kp) in place; the pivot latch stays in the full-grid plan.
    scheme None: the full-grid plan's current coefficients are used."""
    import torch
    y0, y1 = ex.partition.y_ranges[rank]
    kp = ((y1 - y0) + 1) & ~1
    zplan = get_plan(grid.n_x, grid.n_y, grid.n_z, recv.device)
    with zplan.lock:
        if scheme is not None:
            device_coefficients(zplan, scheme, profile, grid)
        nck = (grid.n_z + 7) // 8
        cp = torch.empty(nck * grid.n_x * kp, dtype=torch.float64, device=recv.device)
        check(zplan.lib.hfb_solve_modes(zplan.handle, ptr(recv), kp, y1 - y0, y0, ptr(cp),
                                        zplan.stream()), "solve_modes")
    return zplan


def blocks_to_solution(back, modes, grid, ex, rank, out=None):
    """Stage 3 (per rank): unpack the returned blocks into the mode rows and run
    the inverse 2D DST into the natural-layout solution slab."""
    import torch
    z0, z1 = ex.partition.z_ranges[rank]
    kpz = z1 - z0
    tplan = get_plan(grid.n_x, grid.n_y, kpz, back.device)
    if out is None:
        out = torch.empty((kpz, grid.n_y, grid.n_x), dtype=torch.float64, device=back.device)
    with tplan.lock:
        st = tplan.stream()
        ys = y_starts(ex)
        ysp = ys.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
        if fused_blocks(ex):
            check(tplan.lib.hfb_inverse_blocks(tplan.handle, ptr(back), ptr(modes), ptr(out), ysp,
                                               ex.n_parts, st), "inverse_blocks")
        else:
            check(tplan.lib.hfb_unpack_modes(tplan.handle, ptr(back), ptr(modes), ysp,
                                             ex.n_parts, st), "unpack_modes")
            check(tplan.lib.hfb_inverse_modes(tplan.handle, ptr(modes), ptr(out), st),
                  "inverse_modes")
    return out


def check_status(grid, group=None, device=None):
    """Agree across ranks on a latched vanishing pivot (synchronises); raises
    SingularSystemError on every rank if any rank hit one."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    zplan = get_plan(grid.n_x, grid.n_y, grid.n_z, dev)
    flag = torch.zeros(1, dtype=torch.int64, device=dev)
    try:
        zplan.fetch_status()
    except Exception:
        flag.fill_(1)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if int(flag.item()):
        from .errors import SingularSystemError
        raise SingularSystemError("vanishing pivot on at least one rank")


def chunk_layout(ex, chunks):
    """Chunked exchange geometry. Every rank's z-range is cut into `chunks` plane
    ranges (some may be empty); chunk c of all ranks travels in one all-to-all,
    so the receiver's y-slab holds chunk 0 of every sender, then chunk 1, ...
    Returns (ranges, level_plane): ranges[r][c] = (c0, c1) local plane range of
    rank r's chunk c, level_plane[l] = plane of global level l in the y-slab."""
    zr = ex.partition.z_ranges
    ranges = []
    for z0, z1 in zr:
        n = z1 - z0
        cuts = [round(c * n / chunks) for c in range(chunks + 1)]
        ranges.append([(cuts[c], cuts[c + 1]) for c in range(chunks)])
    level_plane = np.empty(ex.n_z, dtype=np.int32)
    plane = 0
    for c in range(chunks):
        for r, (z0, _) in enumerate(zr):
            c0, c1 = ranges[r][c]
            level_plane[z0 + c0:z0 + c1] = np.arange(plane, plane + c1 - c0)
            plane += c1 - c0
    return ranges, level_plane


def chunk_split_sizes(ex, ranges, rank, c):
    """(send, recv) element counts of chunk c's all-to-all for `rank`."""
    yr = ex.partition.y_ranges
    kp = [((y1 - y0) + 1) & ~1 for y0, y1 in yr]
    c0, c1 = ranges[rank][c]
    send = [(c1 - c0) * ex.n_x * k for k in kp]
    recv = [(ranges[p][c][1] - ranges[p][c][0]) * ex.n_x * kp[rank] for p in range(ex.n_parts)]
    return send, recv


def forward_chunk(z_slab, modes, grid, ex, rank, c0, c1):
    """Forward 2D DST of local planes [c0, c1) into their mode rows (a slice of
    `modes`) and pack their exchange blocks; returns the send buffer."""
    import torch
    dev = z_slab.device
    tplan = get_plan(grid.n_x, grid.n_y, c1 - c0, dev)
    ldm = int(tplan.lib.hfb_modes_ld(tplan.handle))
    m = modes[c0 * grid.n_x * ldm:c1 * grid.n_x * ldm]
    with tplan.lock:
        st = tplan.stream()
        work = tplan.workspace(5)
        kp = [((y1 - y0) + 1) & ~1 for y0, y1 in ex.partition.y_ranges]
        send = torch.empty((c1 - c0) * grid.n_x * sum(kp), dtype=torch.float64, device=dev)
        ys = y_starts(ex)
        ysp = ys.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
        if fused_blocks(ex):
            check(tplan.lib.hfb_forward_blocks(tplan.handle, ptr(z_slab[c0:c1]), ptr(send),
                                               ptr(work), ysp, ex.n_parts, st), "forward_blocks")
        else:
            check(tplan.lib.hfb_forward_modes(tplan.handle, ptr(z_slab[c0:c1]), ptr(m), ptr(work),
                                              st), "forward_modes")
            check(tplan.lib.hfb_pack_modes(tplan.handle, ptr(m), ptr(send), ysp, ex.n_parts, st),
                  "pack_modes")
    return send


def inverse_chunk(back, modes, out, grid, ex, c0, c1):
    """Unpack chunk blocks into the mode rows of local planes [c0, c1) and run
    their inverse 2D DST into out[c0:c1]."""
    tplan = get_plan(grid.n_x, grid.n_y, c1 - c0, back.device)
    ldm = int(tplan.lib.hfb_modes_ld(tplan.handle))
    m = modes[c0 * grid.n_x * ldm:c1 * grid.n_x * ldm]
    with tplan.lock:
        st = tplan.stream()
        ys = y_starts(ex)
        ysp = ys.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
        if fused_blocks(ex):
            check(tplan.lib.hfb_inverse_blocks(tplan.handle, ptr(back), ptr(m), ptr(out[c0:c1]),
                                               ysp, ex.n_parts, st), "inverse_blocks")
        else:
            check(tplan.lib.hfb_unpack_modes(tplan.handle, ptr(back), ptr(m), ysp, ex.n_parts, st),
                  "unpack_modes")
            check(tplan.lib.hfb_inverse_modes(tplan.handle, ptr(m), ptr(out[c0:c1]), st),
                  "inverse_modes")


def solve_received_chunked(recv, level_plane, scheme, profile, grid, ex, rank):
    """solve_received for a y-slab assembled chunk by chunk (levels permuted)."""
    import torch
    y0, y1 = ex.partition.y_ranges[rank]
    kp = ((y1 - y0) + 1) & ~1
    zplan = get_plan(grid.n_x, grid.n_y, grid.n_z, recv.device)
    with zplan.lock:
        if scheme is not None:
            device_coefficients(zplan, scheme, profile, grid)
        nck = (grid.n_z + 7) // 8
        cp = torch.empty(nck * grid.n_x * kp, dtype=torch.float64, device=recv.device)
        lp = np.ascontiguousarray(level_plane, dtype=np.int32)
        check(zplan.lib.hfb_solve_modes_perm(zplan.handle, ptr(recv), kp, y1 - y0, y0,
                                             lp.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                             ptr(cp), zplan.stream()), "solve_modes_perm")
    return zplan


def require_mode_space(grid):
    """The multi-GPU paths run the mode-row transforms (hfb_forward_modes), which
    need n_x + 1 and n_y + 1 powers of two in [16, 4096] (the FFT engine). Any
    other extent raises here, clearly, instead of deep inside the library; the
    one-device Partitioned mode and the one-call solve take every size."""
    ok = lambda n: 16 <= n + 1 <= 4096 and (n + 1) & n == 0
    if not (ok(grid.n_x) and ok(grid.n_y)):
        raise ValueError(
            f"multi-GPU solve needs n_x + 1 and n_y + 1 powers of two in [16, 4096], got "
            f"n_x = {grid.n_x}, n_y = {grid.n_y} (use the one-device solve for this grid)")


def solve_partitioned(z_slab, scheme, profile, grid, group=None, timings=None, chunks=4,
                      check=True):
    """Solve with the grid split over the ranks of `group`; z_slab is this rank's
    (kpz, n_y, n_x) CUDA float64 part of the folded RHS. Returns the solution slab
    (a new tensor). Raises SingularSystemError on every rank if any rank hit a
    vanishing pivot.

    Mode-space exchange: the forward 2D DST leaves padded mode rows (l, n, m);
    the block for rank q is (kpz, n_x, kp(q)); the receive buffer is directly
    the y-slab of mode rows the TMA z-solve streams (no unpack on the way in).
    With chunks > 1 the z-slab goes in `chunks` plane ranges: the all-to-all of
    chunk c runs (NCCL stream) while chunk c + 1 is transformed, and on the way
    back chunk c is unpacked and inverse-transformed while chunk c + 1 is in
    flight; the z-solve reads the chunk-ordered y-slab through a level table.

    check=False skips the per-call pivot agreement (a host synchronisation);
    call check_status(grid, group) after a batch of solves instead."""
    import torch
    import torch.distributed as dist
    require_mode_space(grid)
    rank, parts = dist.get_rank(group), dist.get_world_size(group)
    ex = make_exchange_plan(grid, parts)
    z0, z1 = ex.partition.z_ranges[rank]
    kpz = z1 - z0
    if tuple(z_slab.shape) != (kpz, grid.n_y, grid.n_x):
        raise ValueError(f"z-slab shape {tuple(z_slab.shape)} != {(kpz, grid.n_y, grid.n_x)}")
    dev = z_slab.device
    chunks = max(1, min(chunks, min(z1 - z0 for z0, z1 in ex.partition.z_ranges)))
    ranges, level_plane = chunk_layout(ex, chunks)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timings is not None else None

    def mark(i):
        if ev is not None:
            ev[i].record()

    local = z_slab.contiguous()
    ldm = int(get_plan(grid.n_x, grid.n_y, kpz, dev).lib.hfb_modes_ld(
        get_plan(grid.n_x, grid.n_y, kpz, dev).handle))
    modes = torch.empty(kpz * grid.n_x * ldm, dtype=torch.float64, device=dev)
    y0, y1 = ex.partition.y_ranges[rank]
    kp_me = ((y1 - y0) + 1) & ~1
    recv = torch.empty(grid.n_z * grid.n_x * kp_me, dtype=torch.float64, device=dev)
    offs, off = [], 0
    for c in range(chunks):
        offs.append(off)
        off += sum(chunk_split_sizes(ex, ranges, rank, c)[1])
    mark(0)
    works, keep = [], []
    for c in range(chunks):
        c0, c1 = ranges[rank][c]
        send = forward_chunk(local, modes, grid, ex, rank, c0, c1)
        s, r = chunk_split_sizes(ex, ranges, rank, c)
        keep.append(send)
        works.append(dist.all_to_all_single(recv[offs[c]:offs[c] + sum(r)], send,
                                            output_split_sizes=r, input_split_sizes=s,
                                            group=group, async_op=True))
    for w in works:
        w.wait()
    mark(1)
    solve_received_chunked(recv, level_plane, scheme, profile, grid, ex, rank)
    mark(2)
    out = torch.empty((kpz, grid.n_y, grid.n_x), dtype=torch.float64, device=dev)
    backs, works = [], []
    for c in range(chunks):
        s, r = chunk_split_sizes(ex, ranges, rank, c)
        back = torch.empty(sum(s), dtype=torch.float64, device=dev)
        backs.append(back)
        works.append(dist.all_to_all_single(back, recv[offs[c]:offs[c] + sum(r)],
                                            output_split_sizes=s, input_split_sizes=r,
                                            group=group, async_op=True))
    for c in range(chunks):
        works[c].wait()
        c0, c1 = ranges[rank][c]
        inverse_chunk(backs[c], modes, out, grid, ex, c0, c1)
    mark(3)
    if check:
        check_status(grid, group, dev)
    if timings is not None:
        torch.cuda.synchronize(dev)
        timings.update(forward_exchange_s=ev[0].elapsed_time(ev[1]) / 1e3,
                       tridiag_s=ev[1].elapsed_time(ev[2]) / 1e3,
                       exchange_inverse_s=ev[2].elapsed_time(ev[3]) / 1e3)
    return out


def solve_partitioned_local(values, scheme, profile, grid, parts, clock=None):
    """The Partitioned mode on ONE device: every part runs the per-rank stages of
    solve_partitioned (mode-row blocks, TMA z-solve on its y-slab) and the
    all-to-alls are device copies between the parts' buffers. Bit-identical to
    the one-call solve. Returns (solution, (transform_s, exchange_s, tridiag_s))
    or None when the mode-space stages do not apply (non power-of-two lines)."""
    import torch
    ex = make_exchange_plan(grid, parts)
    dev = values.device
    for z0, z1 in ex.partition.z_ranges:
        tp = get_plan(grid.n_x, grid.n_y, z1 - z0, dev)
        if not int(tp.lib.hfb_workspace_bytes(tp.handle, 5)):
            return None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record()
    sends, modes = [], []
    for r, (z0, z1) in enumerate(ex.partition.z_ranges):
        s, m = forward_to_blocks(values[z0:z1].contiguous(), grid, ex, r)
        sends.append(s)
        modes.append(m)
    ev[1].record()
    ssz = [mode_split_sizes(ex, r)[0] for r in range(parts)]
    rsz = [mode_split_sizes(ex, r)[1] for r in range(parts)]

    def chunk(buf, sizes, q):
        off = sum(sizes[:q])
        return buf[off:off + sizes[q]]

    recvs = [torch.cat([chunk(sends[p], ssz[p], q) for p in range(parts)])
             for q in range(parts)]
    ev[2].record()
    zplan = None
    for r in range(parts):
        zplan = solve_received(recvs[r], scheme, profile, grid, ex, r)
    ev[3].record()
    backs = [torch.cat([chunk(recvs[q], rsz[q], p) for q in range(parts)])
             for p in range(parts)]
    ev[4].record()
    out = torch.empty_like(values)
    for r, (z0, z1) in enumerate(ex.partition.z_ranges):
        blocks_to_solution(backs[r], modes[r], grid, ex, r, out=out[z0:z1])
    ev[5].record()
    zplan.fetch_status()
    ev[5].synchronize()
    sec = lambda a, b: ev[a].elapsed_time(ev[b]) / 1e3
    return out, (sec(0, 1) + sec(4, 5), sec(1, 2) + sec(3, 4), sec(2, 3))


# ---------------------------------------------------------------------------
# Transpose-free distributed z-solve (carries through peer memory)

def carry_neighbours(rank, parts):
    """(previous, next) rank of `rank` in the z-order of the slabs, None at the ends:
    the forward carry goes rank -> next, the backward carry rank -> previous."""
    return (rank - 1 if rank > 0 else None, rank + 1 if rank + 1 < parts else None)


def carry_layout(plan, ld):
    """(doubles of one rank's carry region, flag blocks) for the full-grid plan."""
    size, nb = ctypes.c_longlong(0), ctypes.c_int(0)
    check(plan.lib.hfb_carry_layout(plan.handle, ld, ctypes.byref(size), ctypes.byref(nb)),
          "carry_layout")
    return size.value, nb.value


def carry_layout_z(plan, ld):
    """carry_layout for a complex table (complex carries)."""
    size, nb = ctypes.c_longlong(0), ctypes.c_int(0)
    check(plan.lib.hfb_carry_layout_z(plan.handle, ld, ctypes.byref(size), ctypes.byref(nb)),
          "carry_layout_z")
    return size.value, nb.value


def carry_status_code(plan):
    """0, or the latched missing-carry direction (1 forward, 2 backward); synchronises."""
    code = ctypes.c_int(0)
    rc = plan.lib.hfb_carry_check(plan.handle, plan.stream(), ctypes.byref(code))
    if rc != HFB_ERR_EXCHANGE:
        check(rc, "carry_check")
    return code.value


def exchange_error_for(code, rank):
    """ExchangeError(sender, receiver) of a latched missing carry on `rank`."""
    sender = rank - 1 if code == 1 else rank + 1
    return ExchangeError(f"the z-solve carry from rank {sender} to rank {rank} never arrived",
                         sender=sender, receiver=rank)


class CarryLinks:
    """One rank's carry region (zeroed device memory) and its neighbours'
    regions mapped by CUDA IPC; the handles travel by all_gather_object on
    `group` (any backend). `epoch` counts this rank's solves; every rank of the
    group runs the same solves, so the epochs agree."""

    def __init__(self, grid, group, device):
        import torch
        import torch.distributed as dist
        self.rank, self.parts = dist.get_rank(group), dist.get_world_size(group)
        self.plan = get_plan(grid.n_x, grid.n_y, grid.n_z, device)
        lib = self.plan.lib
        self.ld = int(lib.hfb_modes_ld(self.plan.handle))
        # one region per carry layout (real and complex tables): their flags sit at
        # different offsets, so a rank that alternates the two never reads one
        # layout's carries as the other's flags. Both live in ONE allocation
        # (one IPC handle to open per neighbour): real at 0, complex at `zoff`.
        size, self.blocks = carry_layout(self.plan, self.ld)
        size_z, _ = carry_layout_z(self.plan, self.ld)
        zoff = (size + 63) // 64 * 64
        self._buf = torch.zeros(zoff + size_z, dtype=torch.float64, device=device)
        self.region, self.region_z = self._buf[:size], self._buf[zoff:zoff + size_z]
        torch.cuda.synchronize(device)
        handle, off = (ctypes.c_char * 64)(), ctypes.c_longlong(0)
        check(lib.hfb_ipc_handle(ptr(self._buf), handle, ctypes.byref(off)), "ipc_handle")
        infos = [None] * self.parts
        dist.all_gather_object(infos, (bytes(handle), off.value), group=group)
        self._opened = []
        prev, nxt = carry_neighbours(self.rank, self.parts)
        zb = 8 * zoff
        if prev is not None:
            base = self._open(infos[prev])
            self.prev, self.prev_z = base, base + zb
        else:
            self.prev = self.prev_z = None
        if nxt is not None:
            base = self._open(infos[nxt])
            self.next, self.next_z = base, base + zb
        else:
            self.next = self.next_z = None
        self.epoch = 0

    def _open(self, info):
        import torch
        h, off = info
        buf = (ctypes.c_char * 64).from_buffer_copy(h)
        p = ctypes.c_void_p()
        # the mapping is made on the current device: the slab's, not the caller's
        with torch.cuda.device(self.plan.device):
            check(self.plan.lib.hfb_ipc_open(buf, off, ctypes.byref(p)), "ipc_open")
        self._opened.append((p.value, off))
        return p.value

    def next_epoch(self):
        self.epoch = self.epoch % 0xFFFFFFFF + 1  # never 0: the flags start at 0
        return self.epoch

    def close(self):
        for p, off in self._opened:
            self.plan.lib.hfb_ipc_close(p, off)
        self._opened = []


_links = {}


def _links_key(grid, group, device):
    """Cache key of a group's carry links: the group's member ranks (stable,
    unlike id(group), which a recreated group can reuse)."""
    import torch.distributed as dist
    try:
        members = tuple(dist.get_process_group_ranks(group)) if group is not None \
            else ("world", dist.get_world_size())
    except Exception:
        members = (id(group),)
    return (grid.n_x, grid.n_y, grid.n_z, members, str(device))


def carry_links(grid, group, device):
    key = _links_key(grid, group, device)
    links = _links.get(key)
    if links is not None and links.parts != _group_size(group):
        links.close()
        links = None
    if links is None:
        links = _links[key] = CarryLinks(grid, group, device)
    return links


def _group_size(group):
    import torch.distributed as dist
    return dist.get_world_size(group)


def close_carry_links():
    """Unmap every neighbour's carry region (call before destroying the groups)."""
    for links in _links.values():
        links.close()
    _links.clear()


def carry_zsolve(plan, modes, ld, z0, kpz, cp, mine, peer_next, peer_prev, epoch):
    """Forward then backward sweep of one rank's slab of mode rows (both
    launches on the current stream; the kernels wait for the neighbours)."""
    st = plan.stream()
    check(plan.lib.hfb_zsolve_carry(plan.handle, 0, ptr(modes), ld, z0, kpz, ptr(cp), ptr(mine),
                                    peer_next, epoch, st), "zsolve_carry forward")
    check(plan.lib.hfb_zsolve_carry(plan.handle, 1, ptr(modes), ld, z0, kpz, ptr(cp), ptr(mine),
                                    peer_prev, epoch, st), "zsolve_carry backward")


def carry_zsolve_z(plan, modes_re, modes_im, ld, z0, kpz, cp, mine, peer_next, peer_prev,
                   epoch):
    """carry_zsolve for a complex table: (re, im) mode-row volumes, cp with two
    planes per checkpoint."""
    st = plan.stream()
    for d, peer in ((0, peer_next), (1, peer_prev)):
        check(plan.lib.hfb_zsolve_carry_z(plan.handle, d, ptr(modes_re), ptr(modes_im), ld, z0,
                                          kpz, ptr(cp), ptr(mine), peer, epoch, st),
              f"zsolve_carry_z dir {d}")


def check_status_carry(grid, group=None, device=None):
    """Agree across ranks on a latched vanishing pivot or a missing carry
    (synchronises); raises SingularSystemError / ExchangeError on every rank."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    rank = dist.get_rank(group)
    zplan = get_plan(grid.n_x, grid.n_y, grid.n_z, dev)
    links = _links.get(_links_key(grid, group, dev))
    # singular, exchange, rank*4+code of it, solve epoch
    flags = torch.zeros(4, dtype=torch.int64, device=dev)
    code = carry_status_code(zplan)
    if code:
        flags[1] = 1
        flags[2] = rank * 4 + code
    try:
        zplan.fetch_status()
    except Exception:
        flags[0] = 1
    if links is not None:
        flags[3] = links.epoch
    dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
    if links is not None:
        # a rank that skipped a solve (an error before its launches) rejoins the
        # others' epoch, so the next solve's flags agree again
        links.epoch = int(flags[3].item())
    if int(flags[1].item()):
        r, c = divmod(int(flags[2].item()), 4)
        raise exchange_error_for(c, r)
    if int(flags[0].item()):
        from .errors import SingularSystemError
        raise SingularSystemError("vanishing pivot on at least one rank")


def solve_partitioned_carry(z_slab, scheme, profile, grid, group=None, timings=None,
                            check=True):
    """solve_partitioned without the all-to-alls: the 2D DSTs run on the local
    z-slab (mode rows, as in solve_partitioned) and the z-solve is swept across
    the ranks with carries through peer memory. Same arguments and result.
    A complex table (complex k(z)) takes a complex128 (or real) slab and returns
    a complex128 slab; its real and imaginary parts are transformed separately.

    check=False skips the per-call agreement on pivots and carries (a host
    synchronisation); call check_status_carry(grid, group) after a batch."""
    import torch
    import torch.distributed as dist
    require_mode_space(grid)
    rank, parts = dist.get_rank(group), dist.get_world_size(group)
    ex = make_exchange_plan(grid, parts)
    z0, z1 = ex.partition.z_ranges[rank]
    kpz = z1 - z0
    if tuple(z_slab.shape) != (kpz, grid.n_y, grid.n_x):
        raise ValueError(f"z-slab shape {tuple(z_slab.shape)} != {(kpz, grid.n_y, grid.n_x)}")
    dev = z_slab.device
    links = carry_links(grid, group, dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timings is not None else None

    def mark(i):
        if ev is not None:
            ev[i].record()

    tplan = get_plan(grid.n_x, grid.n_y, kpz, dev)
    ld = links.ld
    zplan = links.plan
    with zplan.lock:
        if scheme is not None:
            device_coefficients(zplan, scheme, profile, grid)
        cplx = zplan.complex_coef
    if torch.is_complex(z_slab) and not cplx:
        raise ValueError("complex right-hand side with a real table: solve re and im separately")
    parts_in = ((z_slab.real.contiguous(), z_slab.imag.contiguous()) if torch.is_complex(z_slab)
                else (z_slab.contiguous(), torch.zeros_like(z_slab)) if cplx
                else (z_slab.contiguous(),))
    modes = [torch.empty(kpz * grid.n_x * ld, dtype=torch.float64, device=dev) for _ in parts_in]
    mark(0)
    with tplan.lock:
        work = tplan.workspace(5)
        for src, m in zip(parts_in, modes):
            _check(tplan.lib.hfb_forward_modes(tplan.handle, ptr(src), ptr(m), ptr(work),
                                               tplan.stream()), "forward_modes")
    mark(1)
    with zplan.lock:
        nck = (kpz + 7) // 8
        if cplx:
            cp = torch.empty(2 * nck * grid.n_x * ld, dtype=torch.float64, device=dev)
            carry_zsolve_z(zplan, modes[0], modes[1], ld, z0, kpz, cp, links.region_z,
                           links.next_z, links.prev_z, links.next_epoch())
        else:
            cp = torch.empty(nck * grid.n_x * ld, dtype=torch.float64, device=dev)
            carry_zsolve(zplan, modes[0], ld, z0, kpz, cp, links.region, links.next,
                         links.prev, links.next_epoch())
    mark(2)
    outs = [torch.empty((kpz, grid.n_y, grid.n_x), dtype=torch.float64, device=dev)
            for _ in modes]
    with tplan.lock:
        for m, o in zip(modes, outs):
            _check(tplan.lib.hfb_inverse_modes(tplan.handle, ptr(m), ptr(o), tplan.stream()),
                   "inverse_modes")
    out = torch.complex(outs[0], outs[1]) if cplx else outs[0]
    mark(3)
    if check:
        check_status_carry(grid, group, dev)
    if timings is not None:
        torch.cuda.synchronize(dev)
        timings.update(transform_s=(ev[0].elapsed_time(ev[1]) + ev[2].elapsed_time(ev[3])) / 1e3,
                       exchange_s=0.0, tridiag_s=ev[1].elapsed_time(ev[2]) / 1e3)
    return out


def solve_partitioned_carry_coop(values, scheme, profile, grid, parts):
    """The carry path with `parts` virtual ranks on ONE device, each direction's
    sweeps of ALL ranks in one cooperative launch (hfb_zsolve_carry_vranks):
    rank r's CTAs spin on flags rank r -/+ 1's CTAs publish while both run —
    the live cross-rank protocol, not a sequenced emulation. The transforms are
    the per-rank stages of solve_partitioned_carry. Real tables. Returns the
    solution volume (bit-identical to the one-call solve)."""
    import ctypes
    import torch
    ex = make_exchange_plan(grid, parts)
    dev = values.device
    zplan = get_plan(grid.n_x, grid.n_y, grid.n_z, dev)
    ld = int(zplan.lib.hfb_modes_ld(zplan.handle))
    with zplan.lock:
        if scheme is not None:
            device_coefficients(zplan, scheme, profile, grid)
        if zplan.complex_coef:
            raise ValueError("solve_partitioned_carry_coop takes a real table")
    size, _ = carry_layout(zplan, ld)
    zr = ex.partition.z_ranges
    regions = [torch.zeros(size, dtype=torch.float64, device=dev) for _ in range(parts)]
    modes, cps = [], []
    for z0, z1 in zr:
        kpz = z1 - z0
        tplan = get_plan(grid.n_x, grid.n_y, kpz, dev)
        m = torch.empty(kpz * grid.n_x * ld, dtype=torch.float64, device=dev)
        with tplan.lock:
            work = tplan.workspace(5)
            _check(tplan.lib.hfb_forward_modes(tplan.handle, ptr(values[z0:z1].contiguous()),
                                               ptr(m), ptr(work), tplan.stream()),
                   "forward_modes")
        modes.append(m)
        cps.append(torch.empty(((kpz + 7) // 8) * grid.n_x * ld, dtype=torch.float64,
                               device=dev))
    P = ctypes.c_void_p * parts
    I = ctypes.c_int * parts
    mp = P(*[t.data_ptr() for t in modes])
    cpp = P(*[t.data_ptr() for t in cps])
    rp = P(*[t.data_ptr() for t in regions])
    z0s = I(*[a for a, _ in zr])
    nzs = I(*[b - a for a, b in zr])
    with zplan.lock:
        for d in (0, 1):
            _check(zplan.lib.hfb_zsolve_carry_vranks(zplan.handle, d, parts, mp, ld, z0s, nzs,
                                                     cpp, rp, 1, zplan.stream()),
                   "zsolve_carry_vranks")
    out = torch.empty(values.shape, dtype=torch.float64, device=dev)
    for r, (z0, z1) in enumerate(zr):
        tplan = get_plan(grid.n_x, grid.n_y, z1 - z0, dev)
        with tplan.lock:
            _check(tplan.lib.hfb_inverse_modes(tplan.handle, ptr(modes[r]), ptr(out[z0:z1]),
                                               tplan.stream()), "inverse_modes")
    code = carry_status_code(zplan)
    if code:
        raise exchange_error_for(code, 0)
    zplan.fetch_status()
    return out


def solve_partitioned_carry_local(values, scheme, profile, grid, parts):
    """The carry path's per-rank stages for `parts` virtual ranks on ONE device,
    run rank after rank: forward sweeps in rank order, backward sweeps in
    reverse order, so every carry a launch waits for was published by an
    earlier launch on the same stream (nothing waits on a concurrent kernel).
    The peer regions are the other virtual ranks' device buffers. Bit-identical
    to the one-call solve. Returns the solution volume."""
    import torch
    ex = make_exchange_plan(grid, parts)
    dev = values.device
    zplan = get_plan(grid.n_x, grid.n_y, grid.n_z, dev)
    ld = int(zplan.lib.hfb_modes_ld(zplan.handle))
    with zplan.lock:
        if scheme is not None:
            device_coefficients(zplan, scheme, profile, grid)
        cplx = zplan.complex_coef
    if torch.is_complex(values) and not cplx:
        raise ValueError("complex right-hand side with a real table: solve re and im separately")
    vols = ((values.real.contiguous(), values.imag.contiguous()) if torch.is_complex(values)
            else (values.contiguous(), torch.zeros_like(values)) if cplx else (values,))
    size, _ = (carry_layout_z if cplx else carry_layout)(zplan, ld)
    regions = [torch.zeros(size, dtype=torch.float64, device=dev) for _ in range(parts)]
    zr = ex.partition.z_ranges
    modes, cps = [], []
    for r, (z0, z1) in enumerate(zr):
        kpz = z1 - z0
        tplan = get_plan(grid.n_x, grid.n_y, kpz, dev)
        ms = []
        with tplan.lock:
            work = tplan.workspace(5)
            for v in vols:
                m = torch.empty(kpz * grid.n_x * ld, dtype=torch.float64, device=dev)
                _check(tplan.lib.hfb_forward_modes(tplan.handle, ptr(v[z0:z1].contiguous()),
                                                   ptr(m), ptr(work), tplan.stream()),
                       "forward_modes")
                ms.append(m)
        modes.append(ms)
        cps.append(torch.empty(len(vols) * ((kpz + 7) // 8) * grid.n_x * ld,
                               dtype=torch.float64, device=dev))

    def sweep(r, d, peer):
        if cplx:
            return zplan.lib.hfb_zsolve_carry_z(zplan.handle, d, ptr(modes[r][0]), ptr(modes[r][1]),
                                                ld, zr[r][0], zr[r][1] - zr[r][0], ptr(cps[r]),
                                                ptr(regions[r]), peer, 1, zplan.stream())
        return zplan.lib.hfb_zsolve_carry(zplan.handle, d, ptr(modes[r][0]), ld, zr[r][0],
                                          zr[r][1] - zr[r][0], ptr(cps[r]), ptr(regions[r]), peer,
                                          1, zplan.stream())

    with zplan.lock:
        for r in range(parts):
            _check(sweep(r, 0, ptr(regions[r + 1]) if r + 1 < parts else None),
                   "zsolve_carry forward")
        for r in reversed(range(parts)):
            _check(sweep(r, 1, ptr(regions[r - 1]) if r > 0 else None), "zsolve_carry backward")
    outs = [torch.empty(values.shape, dtype=torch.float64, device=dev) for _ in vols]
    for r, (z0, z1) in enumerate(zr):
        tplan = get_plan(grid.n_x, grid.n_y, z1 - z0, dev)
        with tplan.lock:
            for m, o in zip(modes[r], outs):
                _check(tplan.lib.hfb_inverse_modes(tplan.handle, ptr(m), ptr(o[z0:z1]),
                                                   tplan.stream()), "inverse_modes")
    out = torch.complex(outs[0], outs[1]) if cplx else outs[0]
    code = carry_status_code(zplan)
    if code:
        raise exchange_error_for(code, 0)
    zplan.fetch_status()
    return out
