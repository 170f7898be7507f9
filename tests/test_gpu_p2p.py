"""GPU tests (-m gpu) of the fused gather for row sharding (phe_matmul_clear_into + dist.PeerGather).

(i) Row blocks written with a row stride into one [T][R][N] buffer equal the unsharded result,
for the tcgen05 and NTT contractions, forward and W^T.  (ii) Two processes on one GPU (gloo for
the control plane, CUDA IPC for the data): rank 1's kernels write its row block straight into
rank 0's buffer through the IPC mapping -- the mechanism the multi-GPU run uses over NVLink
(peer-mapped memory); only NVLink itself is not exercised here.
"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _problem(phe, ntt, transpose=False, d_out=300, d_in=2100, T=7):
    p = phe.params(phe.PRESET_PAPER)
    W = torch.from_numpy(synth.weights_int8(d_out, d_in, seed=5)).to(DEV)
    x = synth.activations_int8(T, d_out if transpose else d_in, seed=6)
    S = phe.keygen(p, 1)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 77)
    if ntt:
        tabs = phe.NttTables(p)
        w = phe.NttWeights(p, tabs, W, transpose=transpose)
        op = phe.ntt_ct_prepare(p, tabs, seeds, body)
        full = phe.matmul_clear_ntt(p, w, op, T)
    else:
        w = phe.Weights(p, W, transpose=transpose)
        op = phe.ct_prepare(p, seeds, body)
        full = (phe.matmul_clear_T if transpose else phe.matmul_clear)(p, w, op, T)
    return p, w, op, T, full


@pytest.mark.parametrize("ntt,transpose", [(False, False), (True, False), (False, True)])
def test_row_blocks_into_one_buffer(phe, ntt, transpose):
    from paper_2505_07329_b200.dist import shard_range
    p, w, op, T, (fm, fb) = _problem(phe, ntt, transpose)
    R = w.rows
    gm = torch.full((T, R, p.N), -1, dtype=torch.int32, device=DEV)
    gb = torch.full((T, R), -1, dtype=torch.int32, device=DEV)
    for k in range(3):
        r0, r1 = shard_range(R, 3, k)
        phe.matmul_clear_into(p, w, op, T, gm[:, r0:r1], gb[:, r0:r1], r0, r1)
    torch.cuda.synchronize()
    assert torch.equal(gm, fm) and torch.equal(gb, fb)


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        import paper_2505_07329_b200 as phe
        from paper_2505_07329_b200.dist import PeerGather, shard_range
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        phe.load()
        p, w, op, T, (fm, fb) = _problem(phe, ntt=False)
        g = PeerGather(T, w.rows, p.N, root=0)
        r0, r1 = shard_range(w.rows, world, rank)
        bm, bb = g.block(r0, r1)
        phe.matmul_clear_into(p, w, op, T, bm, bb, r0, r1)
        g.complete()
        ok = None
        if rank == 0:
            ok = bool(torch.equal(g.mask, fm) and torch.equal(g.body, fb))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception as e:  # report, do not hang the parent
        q.put((rank, None, repr(e)))


def test_peer_gather_two_processes_one_gpu(phe):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
    errs = [r for r in res if r[2]]
    assert not errs, errs
    assert any(r[0] == 0 and r[1] is True for r in res)
