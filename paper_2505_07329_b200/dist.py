"""Multi-GPU partitioning of W.[x]_HE.

Every output LWE ciphertext (tau, j) is independent, so the work shards with no
collective on the data path:
  * token sharding ("S identical HE servers"): rank r owns tokens shard_range(T, W, r)
    and every weight; weak scaling when each rank brings its own batch.
  * row sharding (north_star): rank r owns rows shard_range(R, W, r) of each linear for all
    tokens; the input ciphertexts (seeds + bodies, ~1.1 MB/token) are replicated.
The only collective is the optional gather of output ciphertexts to one rank: NCCL P2P of the
26-bit wire form of each row shard, chunk by chunk on a side stream so it overlaps the next
chunk's GEMMs (`gather_wire_shards`, driven by bench.py), send/recv of the uint32 form after the
GEMM (`gather_rows`), or fused into the GEMM itself (`PeerGather`): rank 0's
gather buffer is mapped into every rank through CUDA IPC and each rank's mask kernel TMA-stores
its row block straight into it (NVLink peer writes, overlapped with the contraction tile by
tile; `phe_matmul_clear_into`).  This module is plumbing: the compute is libphe's.
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


def gather_wire_shards(shard: torch.Tensor | None, recv: Sequence[torch.Tensor | None] | None, world: int,
                       rank: int, dst: int = 0, group=None, staged: bool = False):
    """One gather step of serialized row shards (phe_wire_serialize_lwe bytes, 26-bit LWE at
    Table 1) to `dst`: rank k != dst sends its shard [n][bytes_k]; dst receives rank k's shard
    straight into its destination recv[k] (no temporaries).  All point-to-point ops of the step
    are issued as one batch (NCCL group: every peer's transfer is in flight at once, so dst's
    NVLink ingress is the only limit).  Returns the works; the caller waits on them on the stream
    that must observe completion.  `staged`: bounce device tensors through host memory (gloo
    plumbing of the shared-GPU test hook only; gloo moves CPU tensors) -- completes before return."""
    if staged:
        if rank != dst:
            dist.send(shard.cpu(), dst, group=group)
        else:
            for k in range(world):
                if k != dst:
                    h = torch.empty(recv[k].shape, dtype=recv[k].dtype)
                    dist.recv(h, k, group=group)
                    recv[k].copy_(h)
        return []
    ops = []
    if rank != dst:
        ops.append(dist.P2POp(dist.isend, shard, dst, group))
    else:
        ops += [dist.P2POp(dist.irecv, recv[k], k, group) for k in range(world) if k != dst]
    return dist.batch_isend_irecv(ops) if ops else []


class PeerGather:
    """Fused gather for row sharding: rank `root` allocates the [T][R][N] mask and [T][R] body
    buffers and shares them through CUDA IPC (torch's reduce_tensor handles, broadcast over the
    process group); every other rank rebuilds tensors aliasing root's memory (peer-mapped: its
    kernels' stores go over NVLink).  `block(r0, r1)` is a rank's row block, a strided view that
    `paper_2505_07329_b200.matmul_clear_into` writes directly.  After the kernels: synchronize,
    then barrier -- root may read once every rank has passed it."""

    def __init__(self, T: int, R: int, N: int, dtype=torch.int32, root: int = 0, group=None, device=None):
        from torch.multiprocessing.reductions import reduce_tensor
        self.root = root
        self.group = group
        rank = dist.get_rank(group)
        if rank == root:
            dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
            self.mask = torch.empty((T, R, N), dtype=dtype, device=dev)
            self.body = torch.empty((T, R), dtype=dtype, device=dev)
            obj = [(reduce_tensor(self.mask), reduce_tensor(self.body))]
        else:
            obj = [None]
        dist.broadcast_object_list(obj, src=root, group=group)
        if rank != root:
            (fm, am), (fb, ab) = obj[0]
            self.mask = fm(*am)
            self.body = fb(*ab)

    def block(self, r0: int, r1: int):
        return self.mask[:, r0:r1], self.body[:, r0:r1]

    def complete(self):
        """Make every rank's stores visible to root (call on all ranks after the kernels)."""
        torch.cuda.synchronize()
        dist.barrier(group=self.group)

