#!/usr/bin/env python
"""bench.py — encrypted tokens/s through all Llama-3.2-1B linears on B200 (BASELINE.json metric).

Default workload = BASELINE configs[3]: the full 16-layer Llama-3.2-1B linear stack, forward
(qkv fused 3072x2048, o 2048x2048, gate_up fused 16384x2048, down 2048x8192) plus backward W^T
(q/k/v/o, gate/up/down transposes, GQA k/v 512x2048), B=8 x C=256 = 2048 tokens, Table 1
parameters (N=2048, q 2^39 -> 2^26).  This is the per-token HE work of the paper's training step
("invokes the W.[x]_HE primitive for the various weight matrices in each transformer
layer ... forward and backward").  One step = one pass of the whole server hot path over the
batch, for every linear call of the stack:
    ct_prepare   seed expansion (ChaCha20) + limb split of masks and bodies      (a3, a4)
    body GEMM    b = W . B  (tcgen05 limb GEMM, plain operand)                    (a6-a8)
    mask GEMM    a = Hankel(W) . A-limbs (tcgen05 limb GEMM) + recombine + switch (a5, a7, a8)
Inputs are resident in HBM when the timed region starts (client-side keygen/encrypt_pack run
untimed); L2 is flushed (256 MiB write) between timed steps, outside the per-step events.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                  [--workload stack|q_proj|ffn|q_proj_packed|stack_packed]
Multi-GPU (torchrun, one rank per GPU): LWE workloads are row-sharded by default (north_star:
rank r owns rows shard_range(R, N, r) of every linear for the same tokens, "scaling": "strong";
no collective on the data path), and the gather of the output ciphertexts to rank 0 (26-bit wire
form, NCCL P2P on a side stream, overlapped with the next chunk's GEMMs) is timed in a separate
pass and reported under "gather".  --shard tokens gives the paper's "S identical HE servers"
(weak scaling).  --impl reference times the CPU oracle (oracle/) on host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted tokens/sec through all Llama-3.2-1B linears; % int8 TC peak"
NOMINAL_INT8_TOPS = 4500.0
LWE_WORKLOADS = ("stack", "q_proj", "ffn")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["stack", "q_proj", "ffn", "q_proj_packed", "stack_packed"],
                    default="stack")
    ap.add_argument("--bwd", choices=["per-matrix", "fused"], default="per-matrix",
                    help="stack backward: per-matrix = one W^T call per weight matrix on its own gradient "
                         "(q, k, v, o, gate, up, down; R26, the default); fused = dx of the fused projections, "
                         "W_qkv^T [g_q; g_k; g_v] and W_gate_up^T [g_gate; g_up] (the input gradient a training "
                         "step needs: one output per input coordinate instead of one per matrix)")
    ap.add_argument("--layers", type=int, default=16,
                    help="stack workloads: transformer layers (Llama-3.2-1B has 16; fewer only for tests)")
    ap.add_argument("--pack", choices=["tc", "ntt"], default="ntt",
                    help="packed workloads, stage 2 (KeySwitch Eq. 8 + rotate-sum Eq. 7): tc = int8 packing GEMM "
                         "on tcgen05, ntt = sum_{l,i} D_{l,i} * KSK_{l,i} in the NTT domain (ntt_keyswitch.cu)")
    ap.add_argument("--contraction", choices=["tc", "ntt", "hybrid"], default=None,
                    help="mask contraction a5: tc = int8 limb GEMM on tcgen05 (north_star; the default), ntt = NTT "
                         "domain (NEXT #4, CUDA cores), hybrid = ntt for multi-block (L >= 2) linears, tc otherwise; "
                         "packed workloads default to ntt for stage 1 (T = 16: a 16-token batch fills a third of a "
                         "51-token tensor-core tile)")
    ap.add_argument("--tokens", type=int, default=None,
                    help="tokens per step (default B*C = 8*256 = 2048; stack_packed: the paper's training "
                         "step, B*C = 1*16)")
    ap.add_argument("--e2e-tokens", type=int, default=None,
                    help="tokens of the e2e pass (host buffers, PCIe-bound); default 102 for the stack, T otherwise")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (no e2e/cpu/clocks/gather)")
    ap.add_argument("--shard", choices=["tokens", "rows"], default=None,
                    help="N>1: rows = W rows split, same tokens (strong; default for LWE workloads); "
                         "tokens = each rank its own batch (weak; default for packed workloads)")
    ap.add_argument("--gather", choices=["none", "both", "fused", "nccl", "p2p"], default=None,
                    help="rows mode, gather of the output ciphertexts to rank 0, in separately timed passes: "
                         "fused = every rank's GEMM epilogue TMA-stores its row block straight into one of two "
                         "IPC-mapped slots on rank 0 (NVLink peer stores, tile by tile), a 4-byte all-reduce per "
                         "call orders the slot reuse; nccl = row shards serialized to the 26-bit wire form and sent "
                         "with NCCL P2P on a side stream, overlapped with the next call's GEMMs; both (default); "
                         "p2p (q_proj) = the fused form over the whole [T][R][N] output inside the timed step; none")
    args = ap.parse_args()
    if args.tokens is None:  # B*C = 8*256; the paper's training step is B = 1, C = 16
        args.tokens = 16 if args.workload == "stack_packed" else 2048
    if args.contraction is None:
        args.contraction = "ntt" if args.workload.endswith("_packed") else "tc"
    return args


# ----------------------------------------------------------------------------- environment
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return mp, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(gpu_index)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.count(",") >= 8]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- workloads
def linears(workload: str, layers: int = 16, bwd: str = "per-matrix"):
    """Calls one step makes: (name, d_out, d_in, transpose, input_key).  Llama-3.2-1B:
    d = 2048, m = 8192, GQA k/v 512x2048, 16 layers.  Linears that share an input ciphertext
    are registered fused (qkv 3072x2048, gate_up 16384x2048), so the input is expanded once and
    read by one GEMM.  Backward W^T takes each output's own gradient."""
    if workload in ("q_proj", "q_proj_packed"):  # configs[1] (LWE outputs / + Eq. 7 packing)
        return [("q_proj", 2048, 2048, False, "x")]
    if workload == "ffn":     # configs[2]: gate/up 8192x2048, down 2048x8192, fwd + W^T bwd
        return [("gate", 8192, 2048, False, "h"), ("up", 8192, 2048, False, "h"),
                ("down", 2048, 8192, False, "m"),
                ("gate_T", 8192, 2048, True, "g_gate"), ("up_T", 8192, 2048, True, "g_up"),
                ("down_T", 2048, 8192, True, "g_down")]
    calls = []                # configs[3]: the full 16-layer stack, forward + backward
    if bwd == "fused":        # dx = W_qkv^T [g_q; g_k; g_v], W_gate_up^T [g_gate; g_up] (same MACs)
        for l in range(layers):
            calls += [(f"L{l}.qkv", 3072, 2048, False, f"L{l}.x"), (f"L{l}.o", 2048, 2048, False, f"L{l}.a"),
                      (f"L{l}.gate_up", 16384, 2048, False, f"L{l}.h"),
                      (f"L{l}.down", 2048, 8192, False, f"L{l}.m"),
                      (f"L{l}.qkv_T", 3072, 2048, True, f"L{l}.gqkv"), (f"L{l}.o_T", 2048, 2048, True, f"L{l}.go"),
                      (f"L{l}.gate_up_T", 16384, 2048, True, f"L{l}.ggu"),
                      (f"L{l}.down_T", 2048, 8192, True, f"L{l}.gd")]
        return calls
    for l in range(layers):
        calls += [(f"L{l}.qkv", 3072, 2048, False, f"L{l}.x"), (f"L{l}.o", 2048, 2048, False, f"L{l}.a"),
                  (f"L{l}.gate_up", 16384, 2048, False, f"L{l}.h"), (f"L{l}.down", 2048, 8192, False, f"L{l}.m"),
                  (f"L{l}.q_T", 2048, 2048, True, f"L{l}.gq"), (f"L{l}.k_T", 512, 2048, True, f"L{l}.gk"),
                  (f"L{l}.v_T", 512, 2048, True, f"L{l}.gv"), (f"L{l}.o_T", 2048, 2048, True, f"L{l}.go"),
                  (f"L{l}.gate_T", 8192, 2048, True, f"L{l}.gg"), (f"L{l}.up_T", 8192, 2048, True, f"L{l}.gu"),
                  (f"L{l}.down_T", 2048, 8192, True, f"L{l}.gd")]
    return calls


def rows_cols(d_out, d_in, tr):
    """Output rows and contracted width of one call (W^T for the backward calls)."""
    return (d_in, d_out) if tr else (d_out, d_in)


def alg_imad_ops(p, rows, cols, T):
    """NTT path (NEXT #4): algorithmic 32-bit integer multiplies per output coefficient =
    2 primes x (3 per Shoup twiddle product x log2(N)/2 butterflies + 3 per Montgomery product
    x L blocks) + 4 for the CRT (Shoup + one wide multiply)."""
    L = (cols + p.N - 1) // p.N
    per_coef = 2 * (3 * (p.N.bit_length() - 1) / 2 + 3 * L) + 4
    return per_coef * rows * p.N * T


def alg_int8_ops(p, rows, cols, T, part):
    """per token per linear d_out*d_in*(N+1) Z_Q-MACs = N mask + 1 body; each costs
    ell int8 MACs; 2 ops per MAC.  K is the unpadded d_in."""
    macs = rows * cols * (p.N if part == "mask" else 1)
    return 2.0 * p.ell * macs * T


def tile_round(n, tpt):
    """Largest multiple of the 51-token tensor-core tile <= n (at least one tile)."""
    return max(tpt, n // tpt * tpt)


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2505_07329_b200 as phe
    import synth

    rank, world, local = dist_env()
    # PHE_BENCH_SHARED_GPU=1 (test hook, tests/test_gpu_torchrun.py): every rank on the box's one
    # GPU with gloo plumbing, so the N > 1 path (sharding, max-over-ranks, gathers) runs under
    # torchrun on a 1-GPU box.  The driver's runs leave it unset: one GPU per rank, NCCL.
    shared = os.environ.get("PHE_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(dev))
    phe.load()
    p = phe.params(phe.PRESET_PAPER)
    T = args.tokens
    packed = args.workload.endswith("_packed")
    if args.shard is None:
        args.shard = "tokens" if packed else "rows"
    rows_mode = args.shard == "rows" and world > 1
    if args.gather is None:
        args.gather = "both" if rows_mode and not packed else "none"
    lins = linears(args.workload, args.layers, args.bwd)
    # ---------------- untimed setup: weights (server registration) and client encryption
    from paper_2505_07329_b200.dist import PeerGather, gather_wire_shards, shard_range
    regs = []   # (name, Weights | NttWeights, input_key)
    tabs = phe.NttTables(p, device=dev) if args.contraction != "tc" else None

    def use_ntt(d_out, d_in, tr):
        L = p.L(d_out if tr else d_in)
        return args.contraction == "ntt" or (args.contraction == "hybrid" and L >= 2)
    for name, d_out, d_in, tr, ikey in lins:
        W = synth.weights_int8_torch(d_out, d_in, seed=synth.MASTER_SEED + len(regs), device=dev)
        if use_ntt(d_out, d_in, tr):
            regs.append((name, phe.NttWeights(p, tabs, W, transpose=tr), ikey))
        else:
            regs.append((name, phe.Weights(p, W, transpose=tr), ikey))
        del W
    is_ntt = {name: isinstance(w, phe.NttWeights) for name, w, _ in regs}
    # this rank's output rows of each linear (all rows unless row-sharded)
    rr = {name: (shard_range(w.rows, world, rank) if rows_mode else (0, w.rows)) for name, w, _ in regs}
    S = phe.keygen(p, synth.MASTER_SEED + 17)
    if packed:  # NEXT #1: KeySwitch key (client keygen, server registration), untimed setup
        ksk = phe.ksk_gen(p, S, synth.MASTER_SEED + 23)
        K = phe.KeySwitchKey(p, ksk) if args.pack == "tc" else phe.NttKeySwitchKey(p, ksk)
        del ksk
    # input ciphertexts: one per distinct (shape, role) -- layers reuse the resident synthetic
    # ciphertexts of the same shape, but every call still expands (ct_prepare) and contracts its own
    inputs = {}
    for name, w, ikey in regs:
        base = (w.cols, w.transpose)
        if base not in inputs:
            gen = synth.activations_int8 if not w.transpose else synth.gradients_int8
            xr = 0 if rows_mode else rank  # row sharding: every rank sees the same tokens
            x = torch.from_numpy(gen(T, w.cols, seed=synth.MASTER_SEED + 1000 * xr + w.cols + 7 * w.transpose)).to(dev)
            seeds, body = phe.encrypt_pack(p, S, x, synth.seed_base(xr * 131 + w.cols + 7 * w.transpose))
            inputs[base] = (seeds, body)
    max_rows = max(rr[name][1] - rr[name][0] for name, _, _ in regs)
    # token chunks: outputs (LWE form: 4 B per coefficient; packed path: the Decomp digits,
    # 4 levels x 1 B) stay <= ~34 GB (gate_up: 275 GB at T=2048) and a chunk is a whole number
    # of 51-token tiles (no extra tile-padding waste)
    tpt = 256 // p.ell
    per_row = (phe.KS_LEVELS if packed else 4) * p.N
    rows_for_chunk = (max_rows + 255) // 256 * 256 if packed else max_rows
    cap = 34_400_000_000 // (rows_for_chunk * per_row)
    chunk = T if T <= cap else tile_round(cap, tpt)  # chunk only when the output does not fit
    if not packed:
        out_mask = torch.empty((chunk, max_rows, p.N), dtype=torch.int32, device=dev)
        out_body = torch.empty((chunk, max_rows), dtype=torch.int32, device=dev)
    if packed:  # flat buffers sized for the largest linear, viewed per linear
        r256m = (max_rows + 255) // 256 * 256
        Gm = (max_rows + p.N - 1) // p.N
        dig_flat = torch.empty(chunk * r256m * phe.KS_LEVELS * p.N, dtype=torch.int8, device=dev)
        bod_flat = torch.empty(chunk * max_rows, dtype=torch.int64, device=dev)
        acc_fn = phe.load().phe_pack_acc_bytes if args.pack == "tc" else phe.load().phe_pack_ntt_ws_bytes
        # the workspace need is not monotone in T (the K-split follows wave fill): size it for
        # the full chunk and for the ragged last chunk
        tail = T % chunk
        acc_buf = torch.empty(max(acc_fn(__import__("ctypes").byref(p), w.rows, n_)
                                  for _, w, _ in regs for n_ in {chunk, tail} if n_ > 0),
                              dtype=torch.uint8, device=dev)
        pk_flat = torch.empty(chunk * Gm * 2 * p.N, dtype=torch.int32, device=dev)
        out_mask = torch.empty(1, dtype=torch.int32, device=dev)  # unused: no LWE-form outputs
    max_L = max(p.L(w.cols) for _, w, _ in regs)
    operand = torch.empty(phe.load().phe_ct_operand_bytes(__import__("ctypes").byref(p), chunk, max_L),
                          dtype=torch.uint8, device=dev)
    ntt_L = max([p.L(w.cols) for n_, w, _ in regs if is_ntt[n_]] or [0])
    ntt_operand = (torch.empty(phe.load().phe_ntt_operand_bytes(__import__("ctypes").byref(p), chunk, ntt_L),
                               dtype=torch.uint8, device=dev) if ntt_L else None)
    peer = None
    if rows_mode and args.gather == "p2p":
        if args.workload != "q_proj":
            raise SystemExit("--gather p2p needs the whole [T][R][N] output resident on rank 0: q_proj only")
        peer = PeerGather(T, regs[0][1].rows, p.N, dtype=torch.int32, root=0)  # 34 GB on rank 0
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    parts_ms = {"ct_prepare": [], "body_gemm": [], "mask_gemm": []}
    launches = [0]

    def step(chunk_=chunk, after=None, into=None):
        """One pass over all calls.  `after(name, w, t0, n, mask_view, body_view)` runs after each
        (chunk, linear)'s GEMMs on the compute stream; `into(name, w, t0, n, r0, r1)` may return
        (mask_block, body_block) row-block views the GEMMs write instead (the gather passes)."""
        evs = []
        for t0 in range(0, T, chunk_):
            n = min(chunk_, T - t0)
            for name, w, ikey in regs:
                seeds, body = inputs[(w.cols, w.transpose)]
                e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                e[0].record(stream)
                if is_ntt[name]:  # NEXT #4: masks expanded straight into the NTT domain
                    phe.ntt_ct_prepare(p, tabs, seeds[t0:t0 + n], body[t0:t0 + n], out=ntt_operand)
                    launches[0] += 2
                else:
                    phe.ct_prepare(p, seeds[t0:t0 + n], body[t0:t0 + n], out=operand)  # a3, a4
                    launches[0] += 1
                e[1].record(stream)
                if packed:  # Eq. 6 -> digits + bodies, then Eq. 8 + Eq. 7 + switch
                    r256, G = (w.rows + 255) // 256 * 256, (w.rows + p.N - 1) // p.N
                    dig = dig_flat[: n * r256 * phe.KS_LEVELS * p.N].view(n, r256, phe.KS_LEVELS, p.N)
                    bod = bod_flat[: n * w.rows].view(n, w.rows)
                    if is_ntt[name]:  # NEXT #4 for stage 1 (Eq. 6 -> digits)
                        phe.matmul_clear_digits_ntt(p, w, ntt_operand, n, digits=dig, body=bod)
                    else:
                        phe.matmul_clear_digits(p, w, operand, n, digits=dig, body=bod)
                    launches[0] += phe.last_launch_count()
                    e[2].record(stream)
                    pko = pk_flat[: n * G * 2 * p.N].view(n, G, 2, p.N)
                    if args.pack == "tc":
                        phe.pack(p, dig, bod, K, out=pko, acc=acc_buf)
                    else:
                        phe.pack_ntt(p, dig, bod, K, out=pko, ws=acc_buf)
                    launches[0] += phe.last_launch_count()
                    e[3].record(stream)
                    evs.append((name, e))
                    continue
                if is_ntt[name]:
                    f, opnd = phe.matmul_clear_ntt, ntt_operand
                else:
                    f, opnd = (phe.matmul_clear_T if w.transpose else phe.matmul_clear), operand
                r0, r1 = rr[name]
                nr = r1 - r0
                blocks = ((peer.mask[t0:t0 + n, r0:r1], peer.body[t0:t0 + n, r0:r1]) if peer is not None
                          else into(name, w, t0, n, r0, r1) if into is not None else None)
                if blocks is not None:  # fused gather: a5 + a6 stores land in rank 0's buffer
                    e[2].record(stream)
                    phe.matmul_clear_into(p, w, opnd, n, blocks[0], blocks[1], r0, r1)
                    launches[0] += phe.last_launch_count()
                    e[3].record(stream)
                    evs.append((name, e))
                    if after is not None:
                        after(name, w, t0, n, None, None)
                    continue
                mview = out_mask.view(-1)[: n * nr * p.N].view(n, nr, p.N)
                bview = out_body.view(-1)[: n * nr].view(n, nr)
                f(p, w, opnd, n, out_mask=phe.SKIP, out_body=bview, row_begin=r0, row_end=r1)  # a6
                launches[0] += phe.last_launch_count()
                e[2].record(stream)
                f(p, w, opnd, n, out_mask=mview, out_body=phe.SKIP, row_begin=r0, row_end=r1)  # a5
                launches[0] += phe.last_launch_count()
                e[3].record(stream)
                evs.append((name, e))
                if after is not None:
                    after(name, w, t0, n, mview, bview)
        return evs

    # ---------------- warmup
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # ---------------- timed region (re-measured once if the clock record shows a thermal /
    # HW slowdown or SM clocks stuck well below max with no reason: the run would be rejected)
    BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    for attempt in range(2):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk = None if args.profile else ClockSampler(local)
        step_ms = []
        per_kind = {}
        mask_by_path = {}
        for k in parts_ms:
            parts_ms[k] = []
        launches[0] = 0
        for _ in range(args.steps):
            evs = step()
            torch.cuda.synchronize()
            step_ms.append(sum(e[0].elapsed_time(e[3]) for _, e in evs))
            parts_ms["ct_prepare"].append(sum(e[0].elapsed_time(e[1]) for _, e in evs))
            parts_ms["body_gemm"].append(sum(e[1].elapsed_time(e[2]) for _, e in evs))
            parts_ms["mask_gemm"].append(sum(e[2].elapsed_time(e[3]) for _, e in evs))
            for name, e in evs:
                kind = name.split(".")[-1]
                per_kind.setdefault(kind, []).append(e[0].elapsed_time(e[3]))
                key = "mask_ntt" if is_ntt[name] else "mask_tc"
                mask_by_path.setdefault(key, []).append(e[2].elapsed_time(e[3]))
            flush.zero_()  # L2 flush between timed steps (outside the events)
        torch.cuda.synchronize()
        clocks = clk.stop() if clk else None
        if world > 1:
            dist.barrier()
        bad = 0.0
        if clocks and clocks.get("sm_mhz") and clocks.get("sm_max_mhz"):
            stuck = clocks["sm_mhz"] < 0.5 * clocks["sm_max_mhz"] and not clocks["reasons"]
            bad = 1.0 if (BAD & set(clocks["reasons"])) or stuck else 0.0
        tb = torch.tensor([bad], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        if tb.item() == 0.0 or attempt == 1:
            if clocks is not None:
                clocks["remeasured"] = attempt == 1
            break
    launches_total = launches[0]
    ms = statistics.mean(step_ms)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = (T if rows_mode else world * T) / (ms_max / 1e3)

    # ---------------- gather of the output ciphertexts to rank 0 (rows mode)
    gather = None
    if peer is not None:
        peer.complete()
        gather = {"mode": "p2p: fused into the kernels' stores (dist.PeerGather, phe_matmul_clear_into); "
                          "included in ms_per_step",
                  "bytes": int(T * regs[0][1].rows * (p.N + 1) * 4)}
    gather_nccl = None
    # NCCL pass first (library transport), then the fused pass (our kernels' stores into peer
    # memory); a Python-level failure of either is recorded in its record instead of losing the line
    if rows_mode and args.gather in ("both", "nccl") and not args.profile:
        try:
            gather_nccl = gather_pass(args, p, phe, regs, rr, world, rank, T, tpt, step, stream, dev, shared,
                                      gather_wire_shards, shard_range, ms_max)
        except Exception as ex:  # noqa: BLE001
            gather_nccl = {"mode": "nccl", "error": repr(ex)[:300]}
    if rows_mode and args.gather in ("both", "fused") and not args.profile:
        try:
            gather = gather_pass_fused(p, phe, regs, rr, world, rank, T, tpt, step, stream, dev, ms_max)
        except Exception as ex:  # noqa: BLE001
            gather = {"mode": "fused", "error": repr(ex)[:300]}
    if gather is None and gather_nccl is not None:
        gather, gather_nccl = gather_nccl, None

    # ---------------- roofline of the dominant kernel (mask limb GEMM, or the NTT kernel if the
    # NTT-domain contraction takes more of the step)
    mp, src = measured_peaks()
    peak = 2.0 * float(mp["bf16_tflops"])  # int8 dense = 2x bf16 (guide's nominal ratio)
    mask_ops = sum(alg_int8_ops(p, rr[n_][1] - rr[n_][0], w.cols, T, "mask") for n_, w, _ in regs
                   if not is_ntt[n_])
    mask_ms = sum(mask_by_path.get("mask_tc", [0.0])) / args.steps
    # packed workloads: events [2]..[3] time the pack GEMM (the dominant kernel), not the NTT
    ntt_ms = 0.0 if packed else sum(mask_by_path.get("mask_ntt", [0.0])) / args.steps
    pack_ops = 0.0
    if packed:  # Eq. 8: 2 parts x Decomp(A_LWE) [rows x 4N] x KSK [4N x N], ell int8 MACs each
        pack_ops = sum(2.0 * 2 * p.ell * phe.KS_LEVELS * p.N * p.N * w.rows * T for _, w, _ in regs)
        mask_ops, mask_ms = pack_ops, statistics.mean(parts_ms["mask_gemm"])
    achieved = mask_ops / (mask_ms / 1e3) / 1e12 if mask_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.workload)
        except Exception:
            traffic = None
    total_ops = sum(alg_int8_ops(p, rr[n_][1] - rr[n_][0], w.cols, T, "mask") +
                    alg_int8_ops(p, rr[n_][1] - rr[n_][0], w.cols, T, "body") for n_, w, _ in regs) + pack_ops
    smax = (clocks or {}).get("sm_max_mhz") or 1965.0
    peak_imad = 148 * 4 * 16 * smax * 1e6 / 1e12  # T IMAD/s: 148 SMs x 4 SMSPs x 16 lanes/clk
    imad_src = ("IMAD issue rate from B300_MICROARCH.md (fma pipe, rt_SMSP = 2 -> 16 lanes/clk/SMSP) x 148 SMs "
                "x sm_max clock (DESIGN.md §6)")
    if packed and args.pack == "ntt":  # stage 2 in the NTT domain dominates: integer-multiply roofline
        lg = p.N.bit_length() - 1
        per_col = 1.5 * p.N * lg + 12 * p.N  # forward NTT (3 per Shoup product) + 4 Montgomery products
        imad = sum(T * ((w.rows + p.N - 1) // p.N) * 2 * phe.KS_LEVELS * p.N * per_col for _, w, _ in regs)
        ach = imad / (mask_ms / 1e3) / 1e12
        roofline = {"bound": "alu", "achieved": round(ach, 3), "peak": round(peak_imad, 3), "unit": "T IMAD/s",
                    "frac": round(ach / peak_imad, 4),
                    "traffic": traffic if args.workload == "q_proj_packed" and T == 2048 else None,
                    "kernel": "ks_ntt_kernel<11> + ks_finalize_kernel + pack_finalize_kernel (NTT-domain "
                              "KeySwitch packing, Eq. 7/8)",
                    "ops": "algorithmic 32-bit multiplies: per (l, i) row, prime and packed ciphertext "
                           "1.5 N log2 N (forward NTT) + 12 N (4 Montgomery products); 4N rows x 2 primes",
                    "peak_source": imad_src}
    elif ntt_ms > mask_ms:  # NTT kernel dominates: ALU (integer-multiply pipe) roofline
        imad = sum(alg_imad_ops(p, rr[n_][1] - rr[n_][0], w.cols, T) for n_, w, _ in regs if is_ntt[n_])
        ach = imad / (ntt_ms / 1e3) / 1e12
        roofline = {"bound": "alu", "achieved": round(ach, 3), "peak": round(peak_imad, 3), "unit": "T IMAD/s",
                    "frac": round(ach / peak_imad, 4), "traffic": None,
                    "kernel": "ntt_mask_kernel<11,SW,1,1> (NTT-domain mask contraction, NEXT #4)",
                    "ops": "algorithmic 32-bit multiplies: (2*(3*log2(N)/2 + 3L) + 4) per output coefficient",
                    "peak_source": imad_src}
    else:
        roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": round(peak, 1), "unit": "TFLOP/s",
                    "frac": round(achieved / peak, 4), "traffic": None if packed else traffic,
                    "kernel": ("pack_gemm_2sm_kernel<5> (KeySwitch GEMM Eq. 8 + rotate-sum Eq. 7)" if packed else
                               "limb_gemm_2sm_kernel<5,SW,13> (mask contraction, tcgen05 cta_group::2)"),
                    "ops": ("int8 tensor ops (2 per MAC), algorithmic: 2*ell*d_out*d_in*N per token per call, "
                            "summed over every call of the step; achieved = that / the summed mask-GEMM time"),
                    "peak_source": f"{src}: 2 x bf16_tflops (burst) of MEASURED_PEAKS.json",
                    "frac_of_nominal_4500": round(achieved / NOMINAL_INT8_TOPS, 4),
                    "step_frac": round(total_ops / (ms_max / 1e3) / 1e12 / peak, 4)}
        if traffic is not None and not packed:
            roofline["traffic_note"] = ("dram bytes of one mask-GEMM launch from ncu --set full "
                                        "(profiles/ncu_traffic.json); per launch, see _source there")

    # ---------------- e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e and not args.profile and args.workload == "q_proj_packed" and not rows_mode:
        e2e = e2e_packed(args, p, phe, synth, regs, inputs, K, pk_flat, chunk, T, world, dev)
    elif (not args.no_e2e and not args.profile and args.workload in LWE_WORKLOADS
          and all(not is_ntt[n_] for n_, _, _ in regs)):
        e2e = e2e_lwe(args, p, phe, regs, rr, inputs, T, world, dev)

    # ---------------- CPU baseline: the oracle on host cores, bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile and not packed:
        cpu = oracle_sample(lins, budget_s=15.0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 3),
            "higher_is_better": True, "scaling": "strong" if rows_mode else "weak", "vs_baseline": None,
            "dtype": "int8",
            "data": "synthetic (seeded int8 Llama-like W, DTok int8 activations, ChaCha20 masks)",
            "config": config_dict(args, world, T, rows_mode),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_total,
            "clocks": clocks,
            "breakdown_ms": ({"ct_prepare": round(statistics.mean(parts_ms["ct_prepare"]), 3),
                              "lwe_digits_gemms": round(statistics.mean(parts_ms["body_gemm"]), 3),
                              ("pack_gemm_finalize" if args.pack == "tc" else "pack_ntt_finalize"):
                                  round(statistics.mean(parts_ms["mask_gemm"]), 3)} if packed else
                             {k: round(statistics.mean(v), 3) for k, v in parts_ms.items()}),
        }
        if len(regs) > 1:
            line["per_linear_ms"] = {k: round(sum(v) / args.steps, 3) for k, v in per_kind.items()}
        if args.workload == "stack" and "o" in per_kind and not rows_mode:
            # configs[1]'s shape inside the stack: o is 2048x2048 forward, exactly q_proj's GEMM
            o_ms = sum(per_kind["o"]) / args.steps / args.layers
            o_ops = alg_int8_ops(p, 2048, 2048, T, "mask") + alg_int8_ops(p, 2048, 2048, T, "body")
            line["sub"] = {"q_proj_shape": {
                "what": "the 2048x2048 forward calls of the stack (o_proj; q_proj's shape, BASELINE configs[1])",
                "tokens_per_s": round(T / (o_ms / 1e3), 1), "ms_per_call": round(o_ms, 3),
                "frac_of_peak": round(o_ops / (o_ms / 1e3) / 1e12 / peak, 4)}}
        if gather is not None:
            line["gather"] = gather
        if gather_nccl is not None:
            line["gather_nccl"] = gather_nccl
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def gather_pass_fused(p, phe, regs, rr, world, rank, T, tpt, step, stream, dev, ms_compute):
    """The gather fused into the contraction (one kernel does the GEMM and the
    transfer): rank 0 allocates two output slots sized for the widest linear and maps them into
    every rank (CUDA IPC, dist.PeerGather); for call k every rank's GEMMs (phe_matmul_clear_into)
    write their row block of slot k % 2 directly -- the mask epilogue's TMA stores and the body
    GEMM's stores go over NVLink into rank 0's HBM tile by tile as the tiles finish.  A 4-byte
    all-reduce on the compute stream after each call is the ordering fence: call k+1 (which
    reuses the slot of k-1) starts on any rank only after every rank finished call k, so slot
    (k-1) % 2 holds call k-1's complete outputs while call k runs (rank 0 may consume it then)."""
    import torch
    import torch.distributed as dist

    from paper_2505_07329_b200.dist import PeerGather
    R_max = max(w.rows for _, w, _ in regs)
    gchunk = min(T, tile_round(14_000_000_000 // (R_max * (p.N + 1) * 4), tpt))
    ok = torch.ones(1, dtype=torch.int32, device=dev)
    err = None
    try:  # every rank maps rank 0's slots (CUDA IPC); agree on success before any fence runs
        pg = PeerGather(2 * gchunk, R_max, p.N, dtype=torch.int32, root=0)
    except Exception as ex:  # noqa: BLE001
        pg, err = None, ex
        ok.zero_()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok.item()) == 0:
        raise RuntimeError(f"fused gather unavailable: {err!r}" if err else "fused gather unavailable on a peer rank")
    mslots, bslots = pg.mask.view(2, -1), pg.body.view(2, -1)
    fence = torch.zeros(1, dtype=torch.int32, device=dev)
    count = [0]
    sent = [0]

    def into(name, w, t0, n, r0, r1):
        s = count[0] % 2
        count[0] += 1
        R = w.rows
        for k in range(1, world):  # bytes other ranks store into rank 0's slot
            a, b = rr_of(w.rows, k)
            sent[0] += n * (b - a) * (p.N + 1) * 4
        return (mslots[s][: n * R * p.N].view(n, R, p.N)[:, r0:r1], bslots[s][: n * R].view(n, R)[:, r0:r1])

    def after(*_):
        dist.all_reduce(fence)  # stream-ordered fence: every rank finished this call

    from paper_2505_07329_b200.dist import shard_range

    def rr_of(R, k):
        return shard_range(R, world, k)
    dist.all_reduce(fence)
    torch.cuda.synchronize()
    dist.barrier()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    step(gchunk, after, into)
    g1.record(stream)
    torch.cuda.synchronize()
    pg.complete()
    tg = torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64, device=dev)
    dist.all_reduce(tg, op=dist.ReduceOp.MAX)
    ms_g = float(tg.item())
    del pg
    return {"mode": "fused: GEMM epilogue stores into 2 IPC-mapped slots on rank 0 (NVLink peer stores, "
                    "phe_matmul_clear_into + dist.PeerGather), 4-byte all-reduce per call as the slot-reuse "
                    "fence; uint32 words; separate pass, not in ms_per_step",
            "ms_step_with_gather": round(ms_g, 2), "ms_step_compute_only": round(ms_compute, 2),
            "exposed_ms": round(ms_g - ms_compute, 2), "bytes_to_rank0": int(sent[0]),
            "rank0_ingress_GBps": round(sent[0] / (ms_g / 1e3) / 1e9, 1), "chunk_tokens": gchunk}


def gather_pass(args, p, phe, regs, rr, world, rank, T, tpt, step, stream, dev, shared, gather_wire_shards,
                shard_range, ms_compute):
    """One extra step with the gather to rank 0: after each (chunk, linear)'s
    GEMMs every rank serializes its row shard to the 26-bit wire form (phe_wire_serialize_lwe,
    0.8125 of the uint32 bytes) into one of two slots, and a side stream sends it to rank 0 with
    NCCL P2P (rank 0 receives each peer's shard straight into its destination block), so the
    transfer of call c overlaps the GEMMs of call c+1.  Rank 0 double-buffers its receive blocks.
    Chunks are smaller than in the compute-only step so that two receive slots of the widest
    linear (gate_up, 16384 rows) stay <= 2 x 16 GB on rank 0."""
    import torch
    import torch.distributed as dist

    def shard_bytes(w, k):
        a, b = shard_range(w.rows, world, k)
        return phe.wire_lwe_bytes(p, b - a)
    per_tok_full = max(sum(shard_bytes(w, k) for k in range(world)) for _, w, _ in regs)
    gchunk = min(T, tile_round(16_000_000_000 // per_tok_full, tpt))
    send_max = gchunk * max(shard_bytes(w, rank) for _, w, _ in regs)
    recv_max = gchunk * per_tok_full if rank == 0 else 0
    slots = [torch.empty(send_max, dtype=torch.uint8, device=dev) for _ in range(2)]
    recv = [torch.empty(recv_max, dtype=torch.uint8, device=dev) for _ in range(2)] if rank == 0 else None
    comm = torch.cuda.Stream(device=dev)
    ev_ready = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]
    count = [0]
    sent = [0]

    def after(name, w, t0, n, mview, bview):
        s = count[0] % 2
        count[0] += 1
        if used[s]:
            stream.wait_event(ev_free[s])  # the transfer that last used slot s has completed
        used[s] = True
        nb = [shard_bytes(w, k) for k in range(world)]
        shard = slots[s][: n * nb[rank]].view(n, nb[rank])
        phe.wire_serialize_lwe(p, mview, bview, out=shard)
        ev_ready[s].record(stream)
        blocks = None
        if rank == 0:
            blocks, off = [], 0
            for k in range(world):
                blocks.append(recv[s][off: off + n * nb[k]].view(n, nb[k]))
                off += n * nb[k]
        sent[0] += sum(n * nb[k] for k in range(world) if k != 0)
        with torch.cuda.stream(comm):
            comm.wait_event(ev_ready[s])
            if rank == 0:  # rank 0's own shard joins the gathered set with a local D2D copy
                blocks[0].copy_(shard)
            works = gather_wire_shards(shard, blocks, world, rank, 0, staged=shared)
            for wk in works:
                wk.wait()  # the comm stream waits for the NCCL transfer
            ev_free[s].record(comm)

    # untimed: one small exchange per peer pair first (NCCL builds its P2P connections lazily)
    warm = torch.zeros((1, 8), dtype=torch.uint8, device=dev)
    wblocks = [torch.empty((1, 8), dtype=torch.uint8, device=dev) for _ in range(world)] if rank == 0 else None
    for wk in gather_wire_shards(warm, wblocks, world, rank, 0, staged=shared):
        wk.wait()
    dist.barrier()
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    step(gchunk, after)
    stream.wait_stream(comm)
    g1.record(stream)
    torch.cuda.synchronize()
    tg = torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64, device=dev)
    dist.all_reduce(tg, op=dist.ReduceOp.MAX)
    ms_g = float(tg.item())
    return {"mode": "nccl: 26-bit wire shards (phe_wire_serialize_lwe), P2P to rank 0 on a side stream, "
                    "overlapped with the next call's GEMMs; separate pass, not in ms_per_step",
            "ms_step_with_gather": round(ms_g, 2), "ms_step_compute_only": round(ms_compute, 2),
            "exposed_ms": round(ms_g - ms_compute, 2), "bytes_to_rank0": int(sent[0]),
            "rank0_ingress_GBps": round(sent[0] / (ms_g / 1e3) / 1e9, 1), "chunk_tokens": gchunk,
            "transport": "gloo via host (shared-GPU test hook)" if shared else "NCCL batch_isend_irecv"}


def e2e_lwe(args, p, phe, regs, rr, inputs, T, world, dev):
    """The step as a client sees it, through the C ABI with HOST buffers: for every call of the
    workload, phe_server_matvec_wire_host takes the wire-format input blocks (9992 B) from
    pinned host memory and returns the switched LWE outputs at 26 bits into pinned host memory
    (chunked H2D / GEMM / D2H on two streams).  PCIe-bound: the stack returns 4.69 GB of
    ciphertext per token, so the pass runs over a stated token subset."""
    import torch
    import torch.distributed as dist
    Te = args.e2e_tokens or (102 if args.workload == "stack" else T)
    Te = min(Te, T)
    max_out = max(phe.wire_lwe_bytes(p, rr[n_][1] - rr[n_][0]) for n_, _, _ in regs)
    try:
        import psutil
        avail = psutil.virtual_memory().available
        while Te > 51 and world * Te * max_out > 0.4 * avail:
            Te //= 2
    except Exception:
        pass
    wire_in = {}
    for name, w, _ in regs:
        key = (w.cols, w.transpose)
        if key not in wire_in:
            seeds, body = inputs[key]
            wire_in[key] = phe.wire_serialize_inputs(p, seeds[:Te], body[:Te]).cpu().pin_memory()
    ho = torch.empty(Te * max_out, dtype=torch.uint8, pin_memory=True)
    h2d = sum(wire_in[(w.cols, w.transpose)].numel() for _, w, _ in regs)
    d2h = sum(Te * phe.wire_lwe_bytes(p, rr[n_][1] - rr[n_][0]) for n_, _, _ in regs)
    chunk_e = 51 if Te >= 102 else Te

    def run():
        for name, w, _ in regs:
            r0, r1 = rr[name]
            out = ho[: Te * phe.wire_lwe_bytes(p, r1 - r0)].view(Te, -1)
            phe.server_matvec_wire_host(p, w, wire_in[(w.cols, w.transpose)], out, chunk_tokens=chunk_e,
                                        row_begin=r0, row_end=r1)
    run()  # warm
    if world > 1:
        dist.barrier()
    wall = []
    for _ in range(2):
        t0 = time.perf_counter()
        run()
        wall.append(time.perf_counter() - t0)
    te = torch.tensor([statistics.mean(wall)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    s = float(te.item())
    return {"value": round(Te / s, 3), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(s * 1e3, 1), "tokens_per_step": Te,
            "api": "phe_server_matvec_wire_host per call (wire bytes in/out: 9992 B input blocks, LWE outputs at "
                   f"26 bits; pinned host buffers, {chunk_e}-token chunks, 2 streams)",
            "note": f"a {Te}-token subset of the step's batch (D2H-bound: the outputs cross PCIe)"}


def e2e_packed(args, p, phe, synth, regs, inputs, K, pk_flat, chunk, T, world, dev):
    """q_proj_packed: wire-format input blocks (9992 B) in, wire-format packed RLWE
    ciphertexts (13312 B) out, through host buffers; checked equal to the device step."""
    import torch
    import torch.distributed as dist
    name, w, _ = regs[0]
    seeds, body = inputs[(w.cols, w.transpose)]
    hi = phe.wire_serialize_inputs(p, seeds, body).cpu().pin_memory()
    G0 = (w.rows + p.N - 1) // p.N
    ho = torch.empty((T, G0, phe.wire_output_bytes(p)), dtype=torch.uint8, pin_memory=True)
    if isinstance(w, phe.NttWeights) and args.pack == "ntt":   # both stages in the NTT domain
        swh, api = phe.server_wire_host_nttw, "phe_server_wire_host_nttw"
    else:  # tensor-core stage 1: the registration the host pipeline takes
        if isinstance(w, phe.NttWeights):
            W0 = synth.weights_int8_torch(w.d_out, w.d_in, seed=synth.MASTER_SEED, device=dev)
            w = phe.Weights(p, W0, transpose=w.transpose)
            del W0
        swh, api = ((phe.server_wire_host, "phe_server_wire_host") if args.pack == "tc" else
                    (phe.server_wire_host_ntt, "phe_server_wire_host_ntt"))
    swh(p, w, K, hi, ho, chunk_tokens=255)
    verified = None
    if chunk >= T:  # the device step's packed outputs for the same inputs are still in pk_flat
        dev_wire = phe.wire_serialize_packed(p, pk_flat[: T * G0 * 2 * p.N].view(T, G0, 2, p.N)).cpu()
        verified = bool(torch.equal(dev_wire.view(-1), ho.view(-1)))
        if not verified:
            raise RuntimeError(f"e2e: {api} output differs from the device step's packed ciphertexts")
    wall = []
    for _ in range(max(2, min(args.steps, 3))):
        t0 = time.perf_counter()
        swh(p, w, K, hi, ho, chunk_tokens=255)
        wall.append(time.perf_counter() - t0)
    te = torch.tensor([statistics.mean(wall)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    return {"value": round(world * T / float(te.item()), 2), "unit": "tokens/s",
            "h2d_bytes_per_step": int(hi.numel()), "d2h_bytes_per_step": int(ho.numel()),
            "ms_per_step": round(float(te.item()) * 1e3, 2),
            "api": api + " (wire-format bytes in/out, pinned host buffers, 255-token chunks)",
            "output_equals_device_step": verified}


def config_dict(args, world, T, rows_mode=False):
    wl = {"q_proj": "Llama-3.2-1B q_proj 2048x2048 forward W.[x]_HE (BASELINE configs[1])",
          "ffn": "Llama-3.2-1B FFN gate/up 8192x2048 + down 2048x8192, fwd + W^T bwd (configs[2])",
          "q_proj_packed": "Llama-3.2-1B q_proj 2048x2048 forward, full primitive: Eq. 6 + KeySwitch packing "
                           "Eq. 7/8 -> RLWE(Wx), 39->26 switch (configs[1] + SURVEY NEXT #1)",
          "stack": f"Llama-3.2-1B all linears x {args.layers} layers (qkv fused 3072x2048, o 2048x2048, gate_up "
                   "fused 16384x2048, down 2048x8192; bwd W^T of q/k/v/o/gate/up/down incl. GQA k/v 512x2048), "
                   "fwd + bwd (BASELINE configs[3])",
          "stack_packed": f"Llama-3.2-1B all linears x {args.layers} layers fwd + bwd, full primitive (Eq. 6 + "
                          "KeySwitch packing Eq. 7/8 + switch): the HE server work of the paper's training step "
                          "(P:432-435, B=1, C=16 by default)"}[args.workload]
    if args.contraction != "tc":
        wl += {"ntt": "; mask contraction in the NTT domain (NEXT #4, CUDA cores)",
               "hybrid": "; NTT-domain mask contraction for L >= 2 linears (NEXT #4), tcgen05 otherwise"}[args.contraction]
    if args.workload.endswith("_packed"):
        wl += {"tc": "; packing stage (Eq. 8 MatMul + rotate-sum) on tcgen05",
               "ntt": "; packing stage as sum_{l,i} D_{l,i} * KSK_{l,i} in the NTT domain"}[args.pack]
    B, C = (1, T) if args.workload == "stack_packed" else (8, T // 8)
    cfg = {"workload": wl, "contraction": args.contraction,
           **({"pack": args.pack} if args.workload.endswith("_packed") else {}),
           "tokens_per_gpu": T if not rows_mode else None, "tokens": T, "B": B, "C": C,
           "N": 2048, "q_in": 39, "q_out": 26, "beta": 27,
           "parallelism": (f"row-sharded x{world}" if rows_mode else f"token-sharded x{world}") if world > 1
           else "single GPU",
           "l2": ("flushed between steps (256 MiB write)" if args.workload.endswith("_packed") else
                  "flushed between steps (256 MiB write); outputs >= 8.6 GB per call >> L2"),
           "output": ("packed RLWE ciphertexts (Eq. 7), uint32 A', B' after the 39->26 switch"
                      if args.workload.endswith("_packed") else
                      "LWE ciphertexts, uint32 per coefficient after 39->26 modulus switch")}
    if args.workload.startswith("stack"):
        cfg["layers"] = args.layers
        cfg["calls_per_step"] = (11 if args.bwd == "per-matrix" else 8) * args.layers
        if args.bwd == "fused":
            cfg["workload"] += ("; backward as dx of the fused projections (W_qkv^T [g_q; g_k; g_v], "
                                "W_gate_up^T [g_gate; g_up]), same MACs")
    return cfg


def oracle_sample(lins, budget_s=15.0, nthreads=None):
    """Times the oracle as it stands (oracle/phe_oracle.py: ChaCha20 expansion + the C literal
    Eq. 6 path with OpenMP over output rows + modswitch) on the host's cores, on a bounded sample
    of the workload: for each distinct contracted width (2048, 8192 and the 512-wide k/v
    transposes) token(s) through row subsets of that width's first matrix.  The oracle's cost per
    call is a + b * rows (a: expanding the token's masks; b: L schoolbook N x N negacyclic
    products per row + the switch), linear in tokens and identical across layers, so tokens/s of
    the whole workload is 1 / sum_calls (a + b rows_call)  (SURVEY §8(d) "Oracle timing")."""
    import numpy as np

    import synth
    from oracle import c_oracle
    from oracle import phe_oracle as O

    lib = c_oracle.load()
    op = O.PAPER
    cores = nthreads or os.cpu_count() or 1
    S = O.keygen(synth.MASTER_SEED + 17, op.N)
    first = {}
    for idx, (name, d_out, d_in, tr, _) in enumerate(lins):
        rows, cols = rows_cols(d_out, d_in, tr)
        first.setdefault(cols, (idx, name, d_out, d_in, tr))
    fit, desc = {}, []
    share = budget_s / len(first)
    for cols, (idx, name, d_out, d_in, tr) in sorted(first.items()):
        W = synth.weights_int8(d_out, d_in, seed=synth.MASTER_SEED + idx)
        M = np.ascontiguousarray(W.T) if tr else W

        def run(r, n):
            xs = (synth.gradients_int8 if tr else synth.activations_int8)(n, cols, seed=synth.MASTER_SEED + 5)
            sd = O.block_seeds(synth.seed_base(99), n, op.L(cols))
            bd = np.stack([O.encrypt(op, S, xs[i], sd[i])[1] for i in range(n)])
            t0 = time.perf_counter()
            O.server_matmul(op, M[:r], sd, bd, out_bits=op.q_out, lib=lib, nthreads=cores)
            return time.perf_counter() - t0
        # grow the row count until the sample fills its share of the budget (or the matrix),
        # then fit t(r) = a + b r over the last two sizes: a = the per-call work (mask expansion
        # of the token's blocks), b = the per-row work (L schoolbook products + switch)
        r, n = min(M.shape[0], cores), 1
        pts = [(r, run(r, n))]
        while pts[-1][1] < 0.5 * share and r < M.shape[0]:
            r = int(min(M.shape[0], max(2 * r, r * 0.6 * share / max(pts[-1][1], 1e-4))))
            pts.append((r, run(r, n)))
        (r1, t1), (r2, t2) = (pts[-2], pts[-1]) if len(pts) > 1 else ((0, 0.0), pts[-1])
        b = (t2 - t1) / (r2 - r1)
        a = max(0.0, t2 - b * r2)
        if r == M.shape[0] and t2 < 0.5 * share:  # whole matrix in well under the share: more tokens
            n = int(min(64, share / max(t2, 1e-4)))
            if n > 1:
                tn = run(r, n)
                a, b = a * tn / (n * t2), b * tn / (n * t2)
        fit[cols] = (a, b)
        desc.append(f"{n} token(s) x {r} rows of {name.split('.')[-1]} (width {cols}) in {pts[-1][1]:.2f} s "
                    f"(per call {a * 1e3:.1f} ms + per row {b * 1e3:.3f} ms)")
    per_token = 0.0
    for _, d_out, d_in, tr, _ in lins:
        rows, cols = rows_cols(d_out, d_in, tr)
        per_token += fit[cols][0] + fit[cols][1] * rows
    return {"value": round(1.0 / per_token, 6), "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": ("; ".join(desc) + f" (seed expansion + literal Eq. 6 in C/OpenMP "
                       f"+ modswitch, {cores} threads); extrapolated over all {len(lins)} calls of the step "
                       "as sum_calls (a + b rows) per width (the oracle's cost is linear in rows and "
                       "identical across layers)"),
            "s_per_token": round(per_token, 3)}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The base contract's reference arm for this tier: the CPU oracle as it stands, on this
    arm's config and metric.  Each step times oracle_sample (a bounded sample: token(s) through a
    row subset of each distinct width) and converts it to tokens/s of the whole workload;
    ms_per_step is the wall time of one such sample, value the mean extrapolated tokens/s."""
    rank, world, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle; other ranks exit 0 without work
    lins = linears(args.workload, args.layers, args.bwd)
    cores = os.cpu_count() or 1
    budget = 2.0 if len({rows_cols(d, e, t)[1] for _, d, e, t, _ in lins}) > 1 else 1.0
    for _ in range(args.warmup):
        oracle_sample(lins, budget_s=budget)
    vals, walls, last = [], [], None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        last = oracle_sample(lins, budget_s=budget)
        walls.append(time.perf_counter() - t0)
        vals.append(last["value"])
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(statistics.mean(walls) * 1e3, 1), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "uint64", "data": "synthetic",
            "config": config_dict(args, world, args.tokens),
            "cpu_baseline": {"value": round(value, 6), "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": last["sample"], "wall_s_per_sample": round(statistics.mean(walls), 2)},
            "e2e": {"value": round(value, 6), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
