"""The row-sharded gather of output ciphertexts ("S identical HE servers",
P:249 outputs "returned" to the client) through the path bench.py runs: every rank computes its
row shard of W.[x] with the fused 39 -> 26 switch (phe_matmul_clear, row_begin/row_end), packs it
to the 26-bit wire form (phe_wire_serialize_lwe) and dist.gather_wire_shards moves it to rank 0
(NCCL batch_isend_irecv when two GPUs are visible; on a one-GPU box two ranks share cuda:0 with
gloo plumbing staged through host memory).  Rank 0 unpacks every shard and checks sampled mask
words and every body against the oracle's closed forms (Eq. 6 with SampleExtract at N-1,
P:176-182, masks re-expanded by the oracle's own ChaCha20) and the oracle's modswitch --
not against the CUDA path's own unsharded output."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

D_OUT, D_IN, T = 600, 2048, 5


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, backend, q, fused=False):
    import torch.distributed as dist

    import paper_2505_07329_b200 as phe
    import synth
    from paper_2505_07329_b200.dist import gather_wire_shards, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev_i = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev_i)
    dev = f"cuda:{dev_i}"
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = phe.params(phe.PRESET_PAPER)
        W = synth.weights_int8(D_OUT, D_IN, seed=synth.MASTER_SEED + 77)
        x = synth.activations_int8(T, D_IN, seed=synth.MASTER_SEED + 78)
        S = phe.keygen(p, 5)
        seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(dev), synth.seed_base(3))
        w = phe.Weights(p, torch.from_numpy(W).to(dev))
        opnd = phe.ct_prepare(p, seeds, body)
        r0, r1 = shard_range(D_OUT, world, rank)
        if fused:
            # bench.py's fused gather: every rank's GEMMs store their row block straight into
            # rank 0's IPC-mapped slot (NVLink peer stores), a 4-byte all-reduce is the fence
            from paper_2505_07329_b200.dist import PeerGather
            pg = PeerGather(T, D_OUT, p.N, dtype=torch.int32, root=0)
            phe.matmul_clear_into(p, w, opnd, T, pg.mask[:, r0:r1], pg.body[:, r0:r1], r0, r1)
            fence = torch.zeros(1, dtype=torch.int32, device=dev)
            dist.all_reduce(fence)
            pg.complete()
            if rank == 0:
                q.put((pg.mask.cpu().numpy().astype(np.uint32).astype(np.uint64),
                       pg.body.cpu().numpy().astype(np.uint32).astype(np.uint64),
                       seeds.cpu().numpy().view(np.uint64), body.cpu().numpy().view(np.uint64)))
            dist.barrier()
            return
        m, b = phe.matmul_clear(p, w, opnd, T, row_begin=r0, row_end=r1)
        shard = phe.wire_serialize_lwe(p, m, b)
        blocks = None
        if rank == 0:
            blocks = [torch.empty((T, phe.wire_lwe_bytes(p, e - s)), dtype=torch.uint8, device=dev)
                      for s, e in (shard_range(D_OUT, world, k) for k in range(world))]
            blocks[0].copy_(shard)
        for wk in gather_wire_shards(shard, blocks, world, rank, 0, staged=(backend == "gloo")):
            wk.wait()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            parts = [phe.wire_deserialize_lwe(p, blk, e - s)
                     for blk, (s, e) in zip(blocks, (shard_range(D_OUT, world, k) for k in range(world)))]
            mask = torch.cat([a for a, _ in parts], dim=1).cpu().numpy().astype(np.uint32).astype(np.uint64)
            bod = torch.cat([c for _, c in parts], dim=1).cpu().numpy().astype(np.uint32).astype(np.uint64)
            q.put((mask, bod, seeds.cpu().numpy().view(np.uint64), body.cpu().numpy().view(np.uint64)))
    finally:
        dist.destroy_process_group()


def _run(backend, world=2, fused=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, q, fused)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    return out


def _check_against_oracle(coracle, mask, bod, seeds, body):
    import synth
    from oracle import phe_oracle as O
    op = O.PAPER
    W = synth.weights_int8(D_OUT, D_IN, seed=synth.MASTER_SEED + 77)
    assert mask.shape == (T, D_OUT, op.N) and bod.shape == (T, D_OUT)
    rng = np.random.default_rng(12)
    for tau in range(T):
        A = np.stack([coracle.expand_mask(int(s), op.N, op.q_in) for s in seeds[tau]])
        js, ts = rng.integers(0, D_OUT, 400), rng.integers(0, op.N, 400)
        js[:2] = [0, D_OUT - 1]  # both shard edges' outermost rows
        ref = O.modswitch(coracle.mask_entries(op, W, A, js, ts), op.q_in, op.q_out)
        assert np.array_equal(mask[tau, js, ts], ref), tau
        refb = O.modswitch(O.body_closed_form(op, W, body[tau]), op.q_in, op.q_out)
        assert np.array_equal(bod[tau], refb), tau


def test_gather_two_ranks_one_gpu_gloo(phe, coracle):
    """Two ranks on the box's GPU (gloo, staged): the gather's host logic + wire round trip."""
    _check_against_oracle(coracle, *_run("gloo"))


def test_gather_nccl_two_gpus(phe, coracle):
    """NCCL over NVLink: rank 0 receives rank 1's shard straight into its destination block."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL P2P); the one-GPU variant above runs the same logic over gloo")
    _check_against_oracle(coracle, *_run("nccl"))


def test_fused_gather_two_ranks_one_gpu(phe, coracle):
    """The fused form (bench.py --gather fused): rank 1's GEMM epilogue writes its rows into rank 0's
    IPC-mapped buffer; rank 0's buffer then holds every row, checked against the oracle."""
    _check_against_oracle(coracle, *_run("gloo", fused=True))


def test_fused_gather_nccl_two_gpus(phe, coracle):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (peer stores over NVLink); the one-GPU variant above runs the same code")
    _check_against_oracle(coracle, *_run("nccl", fused=True))
