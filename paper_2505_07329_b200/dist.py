"""Multi-GPU partitioning of W.[x]_HE.

Every output LWE ciphertext (tau, j) is independent, so the work shards with no
collective on the data path:
  * token sharding ("S identical HE servers"): rank r owns tokens shard_range(T, W, r)
    and every weight; weak scaling when each rank brings its own batch.
  * row sharding (north_star): rank r owns rows shard_range(R, W, r) of each linear for all
    tokens; the input ciphertexts (seeds + bodies, ~1.1 MB/token) are replicated.
The only collective is the optional gather of output ciphertexts to one rank (NCCL over
NVLink on the GPU box; gloo in the CPU tests).  This module is device-agnostic plumbing: the
compute is the caller's (libphe on GPU).
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of [0, n): the first n % world ranks get one extra item."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def row_sharded(compute: Callable[[int, int], Sequence[torch.Tensor]], R: int, world: int,
                rank: int) -> tuple[tuple[int, int], Sequence[torch.Tensor]]:
    """Run `compute(row_begin, row_end)` on this rank's rows (mask [T][r][N], body [T][r])."""
    r0, r1 = shard_range(R, world, rank)
    return (r0, r1), compute(r0, r1)


def gather_rows(mask: torch.Tensor, body: torch.Tensor, R: int, world: int, rank: int, dst: int = 0,
                group=None):
    """Gather row shards [T][r_k][N] / [T][r_k] of every rank into [T][R][N] / [T][R] on `dst`.
    Point-to-point (send/recv to dst): each rank's shard crosses the link once.  Returns the
    full tensors on dst, None elsewhere."""
    T = mask.shape[0]
    if rank != dst:
        dist.send(mask.contiguous(), dst, group=group)
        dist.send(body.contiguous(), dst, group=group)
        return None, None
    full_m = torch.empty((T, R) + tuple(mask.shape[2:]), dtype=mask.dtype, device=mask.device)
    full_b = torch.empty((T, R), dtype=body.dtype, device=body.device)
    for k in range(world):
        r0, r1 = shard_range(R, world, k)
        if k == dst:
            full_m[:, r0:r1] = mask
            full_b[:, r0:r1] = body
            continue
        bm = torch.empty((T, r1 - r0) + tuple(mask.shape[2:]), dtype=mask.dtype, device=mask.device)
        bb = torch.empty((T, r1 - r0), dtype=body.dtype, device=body.device)
        dist.recv(bm, k, group=group)
        dist.recv(bb, k, group=group)
        full_m[:, r0:r1] = bm
        full_b[:, r0:r1] = bb
    return full_m, full_b


def gather_tokens(mask: torch.Tensor, body: torch.Tensor, T: int, world: int, rank: int, dst: int = 0,
                  group=None):
    """Gather token shards [t_k][R][N] / [t_k][R] into [T][R][N] / [T][R] on `dst`."""
    if rank != dst:
        dist.send(mask.contiguous(), dst, group=group)
        dist.send(body.contiguous(), dst, group=group)
        return None, None
    R = body.shape[1]
    full_m = torch.empty((T,) + tuple(mask.shape[1:]), dtype=mask.dtype, device=mask.device)
    full_b = torch.empty((T, R), dtype=body.dtype, device=body.device)
    for k in range(world):
        t0, t1 = shard_range(T, world, k)
        if k == dst:
            full_m[t0:t1] = mask
            full_b[t0:t1] = body
        else:
            dist.recv(full_m[t0:t1], k, group=group)  # token slices are contiguous
            dist.recv(full_b[t0:t1], k, group=group)
    return full_m, full_b
