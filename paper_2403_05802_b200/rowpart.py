"""Row-partitioned multi-GPU plumbing.

Rows are independent for the row-local formats (CSR/DCSR/ELL/COO/hybrid),
so the path shards by contiguous row blocks with nnz-balanced boundaries;
the only exchange is the reassembly of the output vector/matrix, an NCCL
all-gather of equal padded chunks (torch.distributed is the plumbing).

`row_bounds` restates the boundary rule of `sfg_row_partition` (the device
version reads the same quantile entries), so the rule can be tested on CPU.
"""
from __future__ import annotations

import numpy as np


def row_bounds(rows: np.ndarray, m: int, parts: int) -> list[int]:
    """Partition p starts at the row holding entry floor(p * nnz / P) of the
    row-sorted COO: nnz balanced to within one row; monotone; [0, m]."""
    nnz = len(rows)
    b = [0] * (parts + 1)
    b[parts] = m
    for p in range(1, parts):
        if nnz == 0:
            b[p] = m * p // parts
            continue
        e = nnz * p // parts
        b[p] = max(int(rows[e]) if e < nnz else m, b[p - 1])
    return b


def padded_chunk(local_rows: int, group=None) -> int:
    """Largest row block over the group: the all-gather chunk size."""
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([local_rows], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


def gather_rows(y_local, chunk: int, group=None):
    """All-gather equal chunks: rank r's rows land at [r*chunk, r*chunk+m_r).
    y_local must already be padded to `chunk` rows (any trailing shape)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    assert y_local.shape[0] == chunk
    out = torch.empty((world * chunk,) + tuple(y_local.shape[1:]), dtype=y_local.dtype,
                      device=y_local.device)
    dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
    return out


def unpad(y_gathered, bounds: list[int], chunk: int):
    """Global y (rows in order) from the padded all-gather result."""
    import torch

    parts = [y_gathered[r * chunk: r * chunk + (bounds[r + 1] - bounds[r])]
             for r in range(len(bounds) - 1)]
    return torch.cat(parts, dim=0)
