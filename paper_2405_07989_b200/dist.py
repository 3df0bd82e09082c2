"""Multi-GPU: one process per GPU (torchrun), each rank enumerates its contiguous,
equal-weight block of the canonical lex order (PAPER.md:196-200 bounds; P:230-231
"distributed nodes") and the partial results are combined with ONE collective on the
compute stream (NCCL over NVLink/NVSwitch; gloo in CPU tests):

  count / length histogram : all_reduce(SUM) of [count] or hist[0..L]    (8 B .. 160 KB)
  any-predicate            : all_reduce(MAX) of the found flag
  rows                     : all_gather of the per-rank row counts -> exclusive scan =
                             global offsets, checked against the DP offsets known a priori;
                             rows stay sharded (each rank's block is already canonical).

The data path has no other exchange: ranks never talk while enumerating.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

from . import _lib as L
from .api import Plan, hist_len


def _dist():
    import torch.distributed as dist

    return dist


def _world():
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def _host_staged() -> bool:
    """gloo (CPU tests, or several ranks sharing one GPU) reduces host tensors: device
    partials are staged through the host; NCCL reduces them in place on the stream."""
    dist = _dist()
    return dist.get_backend() == "gloo"


def _all_reduce(t, op):
    dist = _dist()
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return t
    if t.is_cuda and _host_staged():
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op)
    return t


def combine_sum(t):
    """In-place all_reduce(SUM) of a partial count/histogram tensor (int64)."""
    return _all_reduce(t, _dist().ReduceOp.SUM)


def combine_max(t):
    return _all_reduce(t, _dist().ReduceOp.MAX)


def exclusive_offsets(counts: Sequence[int]) -> List[int]:
    out, s = [], 0
    for c in counts:
        out.append(s)
        s += int(c)
    return out


def gather_counts(local: int, device) -> List[int]:
    import torch

    dist = _dist()
    t = torch.tensor([int(local)], dtype=torch.int64, device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [int(local)]
    if t.is_cuda and _host_staged():
        t = t.cpu()
    outs = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(outs, t)
    return [int(x.item()) for x in outs]


def count(n: int, gens: Sequence[int], *, slice_units: int = 0) -> int:
    """|Z| over all ranks of the default process group (every rank gets the total)."""
    import torch

    rank, world = _world()
    p = Plan(n, gens, L.FS_CONSUMER_COUNT, device=torch.cuda.current_device(),
             stream=torch.cuda.current_stream().cuda_stream, rank=rank, world=world, slice_units=slice_units,
             gen_order=L.FS_GENORDER_AUTO, tail=L.FS_TAIL_CLOSED)  # same configuration as fs_count
    t = torch.zeros(1, dtype=torch.int64, device="cuda")
    p.count_async(t)
    combine_sum(t)
    return int(t.item())


def length_set(n: int, gens: Sequence[int], *, slice_units: int = 0):
    import torch

    rank, world = _world()
    p = Plan(n, gens, L.FS_CONSUMER_HIST, device=torch.cuda.current_device(),
             stream=torch.cuda.current_stream().cuda_stream, rank=rank, world=world, slice_units=slice_units,
             gen_order=L.FS_GENORDER_AUTO, tail=L.FS_TAIL_CLOSED)  # same configuration as fs_length_set
    h = torch.zeros(hist_len(n, gens), dtype=torch.int64, device="cuda")
    p.hist_async(h)
    return combine_sum(h)


def any_pred(n: int, gens: Sequence[int], pred: int, arg: int, *, slice_units: int = 0) -> bool:
    import torch

    rank, world = _world()
    p = Plan(n, gens, L.FS_CONSUMER_ANY, device=torch.cuda.current_device(),
             stream=torch.cuda.current_stream().cuda_stream, rank=rank, world=world, slice_units=slice_units,
             gen_order=L.FS_GENORDER_AUTO, tail=L.FS_TAIL_CLOSED)  # same configuration as fs_any
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    p.any_async(pred, arg, f)
    return bool(combine_max(f).item())


def enumerate_rows(n: int, gens: Sequence[int], B: int = 16, out=None, *, slice_units: int = 0,
                   order: int = L.FS_ORDER_CANONICAL) -> Tuple[int, int, "object"]:
    """This rank's block of canonical rows.  Returns (global_offset, rows, tensor); the
    offsets are exchanged with one all_gather and checked against the DP partition."""
    import torch

    rank, world = _world()
    p = Plan(n, gens, L.FS_CONSUMER_ROWS, device=torch.cuda.current_device(),
             stream=torch.cuda.current_stream().cuda_stream, rank=rank, world=world, slice_units=slice_units,
             order=order)
    info = p.info
    rows = info["row_end"] - info["row_begin"]
    if out is None:
        out = torch.empty((rows, len(gens)), dtype=torch.uint16 if B == 16 else torch.int32, device="cuda")
    p.enumerate_async(B, out, rows)
    if order == L.FS_ORDER_ANY:
        p.rows_check()  # the M2 cursors met exactly: every row of the block written once
    counts = gather_counts(rows, out.device)
    offs = exclusive_offsets(counts)
    if offs[rank] != info["row_begin"]:
        raise RuntimeError("row offsets disagree with the DP partition")
    return info["row_begin"], rows, out[:rows]
