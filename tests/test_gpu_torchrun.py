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
    (["--tokens", "256"], 512),                                           # weak: tokens per rank
    (["--tokens", "256", "--contraction", "ntt", "--no-e2e"], 512),
    (["--tokens", "256", "--shard", "rows", "--gather", "p2p", "--no-e2e"], 256),  # strong + fused gather
    (["--workload", "q_proj_packed", "--tokens", "64"], 128),           # KeySwitch packing, wire e2e
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
