#!/usr/bin/env python
"""bench.py — encrypted tokens/s through the W.[x]_HE hot path on B200 (BASELINE.json metric).

Default workload = BASELINE configs[1]: Llama-3.2-1B q_proj 2048x2048 forward, B=8 x C=256 =
2048 tokens per GPU, Table 1 parameters (N=2048, q 2^39 -> 2^26).  One step = one pass of the
whole server hot path over one batch:
    ct_prepare   seed expansion (ChaCha20) + limb split of masks and bodies      (a3, a4)
    body GEMM    b = W . B  (tcgen05 limb GEMM, plain operand)                    (a6-a8)
    mask GEMM    a = Hankel(W) . A-limbs (tcgen05 limb GEMM) + recombine + switch (a5, a7, a8)
Inputs are resident in HBM when the timed region starts (client-side keygen/encrypt_pack run
untimed); L2 is flushed (256 MiB write) between timed steps, outside the per-step events.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload q_proj|ffn]
Multi-GPU (torchrun, one rank per GPU): tokens are sharded (each rank its own 2048-token
batch, "scaling": "weak"); no collective on the data path; the NCCL all-reduce only takes
the max step time over ranks.  --impl reference times the CPU oracle (oracle/) on host cores.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["q_proj", "ffn", "stack", "q_proj_packed", "stack_packed"],
                    default="q_proj")
    ap.add_argument("--pack", choices=["tc", "ntt"], default="ntt",
                    help="packed workloads, stage 2 (KeySwitch Eq. 8 + rotate-sum Eq. 7): tc = int8 packing GEMM "
                         "on tcgen05, ntt = sum_{l,i} D_{l,i} * KSK_{l,i} in the NTT domain (ntt_keyswitch.cu)")
    ap.add_argument("--contraction", choices=["tc", "ntt", "hybrid"], default=None,
                    help="mask contraction a5: tc = int8 limb GEMM on tcgen05 (north_star; the default), ntt = NTT "
                         "domain (NEXT #4, CUDA cores), hybrid = ntt for multi-block (L >= 2) linears, tc otherwise; "
                         "packed workloads default to ntt for stage 1 (T = 16: a 16-token batch fills a third of a "
                         "51-token tensor-core tile; T = 2048: 45 vs 50 ms, and the step then stays at the "
                         "uncapped clock for the NTT KeySwitch: 6.85k vs 6.40k tok/s)")
    ap.add_argument("--tokens", type=int, default=None,
                    help="tokens per rank (default B*C = 8*256 = 2048; stack_packed: the paper's training "
                         "step, B*C = 1*16)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (no e2e/cpu/clocks)")
    ap.add_argument("--shard", choices=["tokens", "rows"], default="tokens",
                    help="N>1: tokens = each rank its own batch (weak); rows = W rows split (strong)")
    ap.add_argument("--gather", nargs="?", const="nccl", default="none", choices=["none", "nccl", "p2p"],
                    help="rows mode (q_proj): nccl = time an NCCL send/recv gather to rank 0 after the step; "
                         "p2p = fused gather: every rank's kernels write their row block straight into rank "
                         "0's buffer (CUDA IPC / NVLink peer stores) inside the timed step")
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
def linears(workload: str):
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
    for l in range(16):
        calls += [(f"L{l}.qkv", 3072, 2048, False, f"L{l}.x"), (f"L{l}.o", 2048, 2048, False, f"L{l}.a"),
                  (f"L{l}.gate_up", 16384, 2048, False, f"L{l}.h"), (f"L{l}.down", 2048, 8192, False, f"L{l}.m"),
                  (f"L{l}.q_T", 2048, 2048, True, f"L{l}.gq"), (f"L{l}.k_T", 512, 2048, True, f"L{l}.gk"),
                  (f"L{l}.v_T", 512, 2048, True, f"L{l}.gv"), (f"L{l}.o_T", 2048, 2048, True, f"L{l}.go"),
                  (f"L{l}.gate_T", 8192, 2048, True, f"L{l}.gg"), (f"L{l}.up_T", 8192, 2048, True, f"L{l}.gu"),
                  (f"L{l}.down_T", 2048, 8192, True, f"L{l}.gd")]
    return calls


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


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
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
    lins = linears(args.workload)
    # ---------------- untimed setup: weights (server registration) and client encryption
    from paper_2505_07329_b200.dist import PeerGather, gather_rows, shard_range
    rows_mode = args.shard == "rows" and world > 1
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
    packed = args.workload.endswith("_packed")
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
    per_row = (phe.KS_LEVELS if args.workload.endswith("_packed") else 4) * p.N
    rows_for_chunk = (max_rows + 255) // 256 * 256 if args.workload.endswith("_packed") else max_rows
    cap = 34_400_000_000 // (rows_for_chunk * per_row)
    chunk = T if T <= cap else max(tpt, cap // tpt * tpt)  # chunk only when the output does not fit
    if not args.workload.endswith("_packed"):
        out_mask = torch.empty((chunk, max_rows, p.N), dtype=torch.int32, device=dev)
        out_body = torch.empty((chunk, max_rows), dtype=torch.int32, device=dev)
    if packed:  # flat buffers sized for the largest linear, viewed per linear
        r256m = (max_rows + 255) // 256 * 256
        Gm = (max_rows + p.N - 1) // p.N
        dig_flat = torch.empty(chunk * r256m * phe.KS_LEVELS * p.N, dtype=torch.int8, device=dev)
        bod_flat = torch.empty(chunk * max_rows, dtype=torch.int64, device=dev)
        acc_fn = phe.load().phe_pack_acc_bytes if args.pack == "tc" else phe.load().phe_pack_ntt_ws_bytes
        acc_buf = torch.empty(max(acc_fn(__import__("ctypes").byref(p), w.rows, chunk)
                                  for _, w, _ in regs), dtype=torch.uint8, device=dev)
        pk_flat = torch.empty(chunk * Gm * 2 * p.N, dtype=torch.int32, device=dev)
        out_mask = torch.empty(1, dtype=torch.int32, device=dev)  # unused: no LWE-form outputs
    max_L = max(p.L(w.cols) for _, w, _ in regs)
    operand = torch.empty(phe.load().phe_ct_operand_bytes(__import__("ctypes").byref(p), chunk, max_L),
                          dtype=torch.uint8, device=dev)
    ntt_L = max([p.L(w.cols) for n_, w, _ in regs if is_ntt[n_]] or [0])
    ntt_operand = (torch.empty(phe.load().phe_ntt_operand_bytes(__import__("ctypes").byref(p), chunk, ntt_L),
                               dtype=torch.uint8, device=dev) if ntt_L else None)
    peer = None
    if rows_mode and args.gather == "p2p" and args.workload == "q_proj" and not packed:
        peer = PeerGather(T, regs[0][1].rows, p.N, dtype=torch.int32, root=0)  # 34 GB on rank 0
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    parts_ms = {"ct_prepare": [], "body_gemm": [], "mask_gemm": []}
    launches = [0]

    def step(record):
        evs = []
        for t0 in range(0, T, chunk):
            n = min(chunk, T - t0)
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
                if peer is not None:  # fused gather: a5 + a6 stores land in rank 0's buffer
                    e[2].record(stream)
                    phe.matmul_clear_into(p, w, opnd, n, peer.mask[t0:t0 + n, r0:r1], peer.body[t0:t0 + n, r0:r1],
                                          r0, r1)
                    launches[0] += phe.last_launch_count()
                    e[3].record(stream)
                    evs.append((name, e))
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
        return evs

    # ---------------- warmup
    for _ in range(args.warmup):
        step(False)
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
            evs = step(True)
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
    ms = statistics.mean(step_ms)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = (T if rows_mode else world * T) / (ms_max / 1e3)

    # ---------------- optional: NCCL gather of the row-sharded output ciphertexts to rank 0
    gather = None
    if peer is not None:
        peer.complete()
        gather = {"mode": "p2p: fused into the kernels' stores (dist.PeerGather, phe_matmul_clear_into); "
                          "included in ms_per_step",
                  "bytes": int(T * regs[0][1].rows * (p.N + 1) * 4)}
    if rows_mode and args.gather == "nccl" and args.workload == "q_proj":
        name, w, _ = regs[0]
        r0, r1 = rr[name]
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        nr = r1 - r0
        gather_rows(out_mask.view(-1)[: T * nr * p.N].view(T, nr, p.N), out_body.view(-1)[: T * nr].view(T, nr),
                    w.rows, world, rank)
        g1.record(stream)
        torch.cuda.synchronize()
        tg = torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64, device=dev)
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        gather = {"ms": round(float(tg.item()), 2), "bytes": int(T * w.rows * (p.N + 1) * 4),
                  "api": "paper_2505_07329_b200.dist.gather_rows (NCCL send/recv to rank 0)"}

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
                    "ops": "int8 tensor ops (2 per MAC), algorithmic: 2*ell*d_out*d_in*N per token",
                    "peak_source": f"{src}: 2 x bf16_tflops (burst) of MEASURED_PEAKS.json",
                    "frac_of_nominal_4500": round(achieved / NOMINAL_INT8_TOPS, 4),
                    "step_frac": round(total_ops / (ms_max / 1e3) / 1e12 / peak, 4)}

    # ---------------- e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e and not args.profile and args.workload == "q_proj_packed" and not rows_mode:
        # the server step as the network sees it: wire-format input blocks (9992 B) in,
        # wire-format packed RLWE ciphertexts (13312 B) out, through host buffers
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
        e2e_s = statistics.mean(wall)
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * T / float(te.item()), 2), "unit": "tokens/s",
               "h2d_bytes_per_step": int(hi.numel()), "d2h_bytes_per_step": int(ho.numel()),
               "ms_per_step": round(float(te.item()) * 1e3, 2),
               "api": api + " (wire-format bytes in/out, pinned host buffers, 255-token chunks)",
               "output_equals_device_step": verified}
    if (not args.no_e2e and not args.profile and args.workload == "q_proj" and not rows_mode
            and args.contraction == "tc"):
        name, w, _ = regs[0]
        seeds, body = inputs[(w.cols, w.transpose)]
        # pinned host memory: 28 GB (wire) [+ 34 GB uint32 variant] per rank; with several ranks on
        # one host measure the wire form only, and over fewer tokens if host RAM is short
        # (tokens/s is per-chunk throughput: 256-token chunks either way)
        lwe_b = phe.wire_lwe_bytes(p, w.rows)
        Te = T
        try:
            import psutil
            avail = psutil.virtual_memory().available
            while Te > 256 and world * Te * (lwe_b + (0 if world > 1 else w.rows * p.N * 4)) > 0.5 * avail:
                Te //= 2
        except Exception:
            pass
        e2e_u32 = None
        if world == 1:
            hs = seeds[:Te].cpu().pin_memory()
            hb = body[:Te].cpu().pin_memory()
            hm = torch.empty((Te, w.rows, p.N), dtype=torch.int32, pin_memory=True)
            hbo = torch.empty((Te, w.rows), dtype=torch.int32, pin_memory=True)
            phe.server_matvec_host(p, w, hs, hb, hm, hbo, chunk_tokens=256)  # warm
            wall = []
            for _ in range(max(2, min(args.steps, 3))):
                t0 = time.perf_counter()
                phe.server_matvec_host(p, w, hs, hb, hm, hbo, chunk_tokens=256)
                wall.append(time.perf_counter() - t0)
            e2e_u32 = {"value": round(Te / statistics.mean(wall), 2), "unit": "tokens/s",
                       "h2d_bytes_per_step": int(hs.numel() * 8 + hb.numel() * 8),
                       "d2h_bytes_per_step": int(hm.numel() * 4 + hbo.numel() * 4),
                       "ms_per_step": round(statistics.mean(wall) * 1e3, 2),
                       "api": "phe_server_matvec_host (uint64 inputs / uint32 outputs, pinned, 256-token chunks)"}
            del hm, hbo, hs, hb
        # the same step on wire bytes: 39-bit input blocks (9992 B) in, LWE outputs at
        # q_out = 26 bits out (0.8125 of the uint32 bytes) -- the D2H-bound headline
        hi = phe.wire_serialize_inputs(p, seeds[:Te], body[:Te]).cpu().pin_memory()
        ho = torch.empty((Te, lwe_b), dtype=torch.uint8, pin_memory=True)
        phe.server_matvec_wire_host(p, w, hi, ho, chunk_tokens=256)  # warm
        if world > 1:
            dist.barrier()
        wall = []
        for _ in range(max(2, min(args.steps, 3))):
            t0 = time.perf_counter()
            phe.server_matvec_wire_host(p, w, hi, ho, chunk_tokens=256)
            wall.append(time.perf_counter() - t0)
        te = torch.tensor([statistics.mean(wall)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * Te / float(te.item()), 2), "unit": "tokens/s",
               "h2d_bytes_per_step": int(hi.numel()), "d2h_bytes_per_step": int(ho.numel()),
               "ms_per_step": round(float(te.item()) * 1e3, 2), "tokens_per_rank": Te,
               "api": "phe_server_matvec_wire_host (wire bytes in/out: 9992 B input blocks, LWE outputs at "
                      "26 bits; pinned host buffers, 256-token chunks, 2 streams)",
               "uint32_outputs": e2e_u32}
        del ho

    # ---------------- CPU baseline: the oracle on host cores, bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        cpu = cpu_baseline(args, lins[0], budget_s=12.0)

    launches_total = launches[0]
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
        if gather is not None:
            line["gather"] = gather
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def config_dict(args, world, T, rows_mode=False):
    wl = {"q_proj": "Llama-3.2-1B q_proj 2048x2048 forward W.[x]_HE (BASELINE configs[1])",
          "ffn": "Llama-3.2-1B FFN gate/up 8192x2048 + down 2048x8192, fwd + W^T bwd (configs[2])",
          "q_proj_packed": "Llama-3.2-1B q_proj 2048x2048 forward, full primitive: Eq. 6 + KeySwitch packing "
                           "Eq. 7/8 -> RLWE(Wx), 39->26 switch (configs[1] + SURVEY NEXT #1)",
          "stack": "Llama-3.2-1B all linears x 16 layers (qkv fused 3072x2048, o, gate_up fused 16384x2048, "
                   "down; bwd W^T incl. GQA k/v 512x2048), fwd + bwd (configs[3])",
          "stack_packed": "Llama-3.2-1B all linears x 16 layers fwd + bwd, full primitive (Eq. 6 + KeySwitch "
                          "packing Eq. 7/8 + switch): the HE server work of the paper's training step "
                          "(P:432-435, B=1, C=16 by default)"}[args.workload]
    if args.contraction != "tc":
        wl += {"ntt": "; mask contraction in the NTT domain (NEXT #4, CUDA cores)",
               "hybrid": "; NTT-domain mask contraction for L >= 2 linears (NEXT #4), tcgen05 otherwise"}[args.contraction]
    if args.workload.endswith("_packed"):
        wl += {"tc": "; packing stage (Eq. 8 MatMul + rotate-sum) on tcgen05",
               "ntt": "; packing stage as sum_{l,i} D_{l,i} * KSK_{l,i} in the NTT domain"}[args.pack]
    B, C = (1, T) if args.workload == "stack_packed" else (8, T // 8)
    return {"workload": wl, "contraction": args.contraction,
            **({"pack": args.pack} if args.workload.endswith("_packed") else {}), "tokens_per_gpu": T if not rows_mode else None, "tokens": T, "B": B, "C": C, "N": 2048, "q_in": 39, "q_out": 26,
            "beta": 27,
            "parallelism": (f"row-sharded x{world}" if rows_mode else f"token-sharded x{world}") if world > 1
            else "single GPU",
            "l2": ("flushed between steps (256 MiB write)" if args.workload.endswith("_packed") else
                   "flushed between steps (256 MiB write), outputs 34 GB/step >> L2"),
            "output": ("packed RLWE ciphertexts (Eq. 7), uint32 A', B' after the 39->26 switch"
                       if args.workload.endswith("_packed") else
                       "LWE ciphertexts, uint32 per coefficient after 39->26 modulus switch")}


def cpu_baseline(args, lin, budget_s=12.0):
    """Times the oracle (oracle/phe_oracle.py + the C literal path) as it stands on the host's
    cores: server-side expansion + literal Eq. 6 + modswitch, on a bounded token sample."""
    import numpy as np

    import synth
    from oracle import c_oracle
    from oracle import phe_oracle as O

    name, d_out, d_in, tr, _ = lin
    lib = c_oracle.load()
    op = O.PAPER
    W = synth.weights_int8(d_out, d_in, seed=synth.MASTER_SEED)
    M = np.ascontiguousarray(W.T) if tr else W
    cols = M.shape[1]
    S = O.keygen(synth.MASTER_SEED + 17, op.N)
    cores = os.cpu_count() or 1

    def sample(n):
        x = synth.activations_int8(n, cols, seed=synth.MASTER_SEED + 5)
        seeds = O.block_seeds(synth.seed_base(99), n, op.L(cols))
        bodies = np.stack([O.encrypt(op, S, x[t], seeds[t])[1] for t in range(n)])
        t0 = time.perf_counter()
        O.server_matmul(op, M, seeds, bodies, out_bits=op.q_out, lib=lib, nthreads=cores)
        return time.perf_counter() - t0

    t1 = sample(1)
    n = int(max(1, min(64, budget_s // max(t1, 1e-3))))
    tn = sample(n) if n > 1 else t1
    return {"value": round(n / tn, 4), "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} tokens of {name} {d_out}x{d_in} (seed expansion + literal Eq.6 in C/OpenMP + "
                      f"modswitch), {tn:.1f} s wall"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle; other ranks exit 0 without work
    import numpy as np

    import synth
    from oracle import c_oracle
    from oracle import phe_oracle as O

    lib = c_oracle.load()
    op = O.PAPER
    cores = os.cpu_count() or 1
    lin = linears(args.workload)[0]
    name, d_out, d_in, tr, _ = lin
    W = synth.weights_int8(d_out, d_in, seed=synth.MASTER_SEED)
    M = np.ascontiguousarray(W.T) if tr else W
    cols = M.shape[1]
    S = O.keygen(synth.MASTER_SEED + 17, op.N)
    per_step = 2  # tokens per step: a bounded sample of the workload
    x = synth.activations_int8(per_step, cols, seed=synth.MASTER_SEED + 5)
    seeds = O.block_seeds(synth.seed_base(7), per_step, op.L(cols))
    bodies = np.stack([O.encrypt(op, S, x[t], seeds[t])[1] for t in range(per_step)])

    def step():
        O.server_matmul(op, M, seeds, bodies, out_bits=op.q_out, lib=lib, nthreads=cores)

    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    ms = statistics.mean(ts) * 1e3
    value = per_step / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "uint64",
            "data": "synthetic", "config": config_dict(args, world, args.tokens),
            "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} tokens of {name} {d_out}x{d_in} per step (literal Eq. 6, "
                                       f"C/OpenMP, {cores} threads)"},
            "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0,
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
