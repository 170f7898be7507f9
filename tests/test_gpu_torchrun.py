"""bench.py's N > 1 path under torchrun on a 1-GPU box: two ranks share cuda:0
(PHE_BENCH_SHARED_GPU=1 -> gloo plumbing instead of NCCL, which refuses two ranks on one device).
Exercises what the driver's scaling run executes at N = 2..8: token and row sharding, the barrier
+ max-over-ranks timing, the fused P2P gather, e2e under torchrun, and the rank-0 JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _torchrun(extra, timeout=900):
    env = dict(os.environ, PHE_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline"] + extra
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("extra,tokens_total", [
    (["--workload", "q_proj", "--tokens", "256", "--shard", "tokens"], 512),          # weak: tokens per rank
    (["--workload", "q_proj", "--tokens", "256", "--shard", "tokens", "--contraction", "ntt", "--no-e2e"], 512),
    (["--workload", "q_proj", "--tokens", "256", "--gather", "p2p", "--no-e2e"], 256),  # rows + fused gather
    (["--workload", "q_proj_packed", "--tokens", "64"], 128),           # KeySwitch packing, wire e2e
    (["--layers", "1", "--tokens", "8"], 8),                             # the default: rows-sharded stack
])
def test_bench_two_ranks_one_gpu(extra, tokens_total):
    d = _torchrun(extra)
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0
    # value = all tokens processed / max-over-ranks step time
    assert d["value"] == pytest.approx(tokens_total / (d["ms_per_step"] / 1e3), rel=1e-3)
    assert d["gpu_launches"] > 0
    if "--no-e2e" not in extra:
        assert d["e2e"]["value"] > 0
    if "--layers" in extra:
        # default N > 1 stack line: row-sharded (strong) with the separately timed gather pass
        assert d["scaling"] == "strong" and d["config"]["parallelism"] == "row-sharded x2"
        # the fused pass (GEMM epilogue stores into rank 0's IPC-mapped slots) and the NCCL pass
        g, gn = d["gather"], d["gather_nccl"]
        assert g["mode"].startswith("fused") and gn["mode"].startswith("nccl")
        assert g["ms_step_with_gather"] > 0 and gn["ms_step_with_gather"] > 0 and gn["chunk_tokens"] >= 1
        # rank 1's bytes of every call: its half of each linear's rows, uint32 words (fused) and
        # 26-bit wire words (nccl)
        import paper_2505_07329_b200 as phe
        import bench
        from paper_2505_07329_b200.dist import shard_range
        p = phe.params(phe.PRESET_PAPER)
        exp_wire = exp_u32 = 0
        for _, d_out, d_in, tr, _ in bench.linears("stack", 1):
            rows = d_in if tr else d_out
            a, b = shard_range(rows, 2, 1)
            exp_wire += 8 * phe.wire_lwe_bytes(p, b - a)
            exp_u32 += 8 * (b - a) * (p.N + 1) * 4
        assert gn["bytes_to_rank0"] == exp_wire and g["bytes_to_rank0"] == exp_u32
