"""World-size-2 gloo tests (CPU) of the multi-GPU path: row and token sharding with the
ciphertext gather reproduce the unsharded result bit-exactly.  The per-rank compute is the
CPU oracle here (on the GPU box it is libphe); the sharding/gather logic under test is
paper_2505_07329_b200/dist.py, the same code bench.py runs under torchrun."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_07329_b200.dist import gather_rows, gather_tokens, shard_range


def test_shard_range_partitions():
    for n in [0, 1, 7, 2048, 3072, 16384]:
        for w in [1, 2, 3, 4, 8]:
            parts = [shard_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(5, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import phe_oracle as O
        P = O.Params(N=16, q_in=39, q_out=26, beta=27, gamma=12)
        R, d_in, T = 7, 40, 5
        W = synth.uniform_int8((R, d_in), 3)
        x = synth.uniform_int8((T, d_in), 4)
        S = O.keygen(9, P.N)
        seeds = O.block_seeds(11, T, P.L(d_in))
        bodies = np.stack([O.encrypt(P, S, x[t], seeds[t])[1] for t in range(T)])
        if mode == "rows":
            r0, r1 = shard_range(R, world, rank)
            m, b = O.server_matmul(P, W[r0:r1], seeds, bodies, out_bits=26)
            fm, fb = gather_rows(torch.from_numpy(m.astype(np.int64)), torch.from_numpy(b.astype(np.int64)),
                                 R, world, rank)
        else:
            t0, t1 = shard_range(T, world, rank)
            m, b = O.server_matmul(P, W, seeds[t0:t1], bodies[t0:t1], out_bits=26)
            fm, fb = gather_tokens(torch.from_numpy(m.astype(np.int64)), torch.from_numpy(b.astype(np.int64)),
                                   T, world, rank)
        if rank == 0:
            ref_m, ref_b = O.server_matmul(P, W, seeds, bodies, out_bits=26)
            q.put(bool(np.array_equal(fm.numpy().astype(np.uint64), ref_m)
                       and np.array_equal(fb.numpy().astype(np.uint64), ref_b)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["rows", "tokens"])
def test_sharded_equals_unsharded_world2(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def _wire_worker(rank, world, port, staged, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_07329_b200.dist import gather_wire_shards
        R, n = 23, 3
        # each rank's "wire shard": n tokens x bytes of its rows (here 7 bytes per row)
        sizes = [(b - a) * 7 for a, b in (shard_range(R, world, k) for k in range(world))]
        shard = torch.full((n, sizes[rank]), rank + 1, dtype=torch.uint8)
        shard[:, 0] = torch.arange(n, dtype=torch.uint8)
        recv = [torch.zeros((n, s_), dtype=torch.uint8) for s_ in sizes] if rank == 0 else None
        if rank == 0:
            recv[0].copy_(shard)
        for wk in gather_wire_shards(shard, recv, world, rank, 0, staged=staged):
            wk.wait()
        if rank == 0:
            ok = all(bool((r[:, 1:] == k + 1).all()) and r[:, 0].tolist() == list(range(n))
                     for k, r in enumerate(recv))
            q.put(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("staged", [False, True])
def test_gather_wire_shards_world3(staged):
    """dist.gather_wire_shards (bench.py's NCCL gather, here over gloo on CPU tensors): rank 0 ends
    with every rank's shard in its own destination block, batched P2P or staged send/recv."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_wire_worker, args=(r, 3, port, staged, q)) for r in range(3)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(timeout=180)
    assert all(p_.exitcode == 0 for p_ in procs)
    assert q.get(timeout=5) is True
