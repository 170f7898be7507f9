"""BASELINE configs[4] measured per GPU: one Llama-3.2-1B layer forward (qkv
3072x2048, o 2048x2048, gate_up 16384x2048, down 2048x8192) swept over T = B*C in {256 ... 16384}
tokens x the parameter sets P0 (Table 1), P1, P2, P3, toy-A, through both mask contractions
(tcgen05 limb GEMM, NTT domain).  The 16 layers are identical, so forward-stack tokens/s =
layer tokens/s / 16 (exact).  Each step = ct_prepare + body GEMM + mask contraction of every
linear over token chunks (outputs <= 34 GB, reused buffer), CUDA events, inputs resident.
Writes gpurun_out/r1_sweep_c5.json.  Not the bench contract (fewer steps at large T)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_07329_b200 as phe  # noqa: E402
import synth  # noqa: E402

SETS = {  # SURVEY §8(d) "C5 parameter sets"
    "P0": dict(),
    "P1": dict(N=1024),
    "P2": dict(q_in=32, q_out=24),
    "P3": dict(N=4096),
    "toyA": "TOY",
}
LAYER = [("qkv", 3072, 2048), ("o", 2048, 2048), ("gate_up", 16384, 2048), ("down", 2048, 8192)]


def params(name):
    v = SETS[name]
    return phe.params(phe.PRESET_TOY) if v == "TOY" else phe.params(phe.PRESET_PAPER, **v)


def run(p, T, contraction, steps, warmup):
    dev = "cuda"
    tabs = phe.NttTables(p) if contraction == "ntt" else None
    regs = []
    for k, (name, d_out, d_in) in enumerate(LAYER):
        W = synth.weights_int8_torch(d_out, d_in, seed=synth.MASTER_SEED + k, device=dev)
        regs.append((name, phe.NttWeights(p, tabs, W) if tabs else phe.Weights(p, W), d_in))
        del W
    S = phe.keygen(p, 3)
    inputs = {}
    for d_in in {2048, 8192}:
        x = torch.from_numpy(synth.activations_int8(T, d_in, seed=d_in)).to(dev)
        inputs[d_in] = phe.encrypt_pack(p, S, x, synth.seed_base(d_in))
    tpt = 256 // p.ell
    max_rows = max(d for _, d, _ in LAYER)
    cap = 34_400_000_000 // (max_rows * p.N * 4)
    chunk = T if T <= cap else max(tpt, cap // tpt * tpt)
    out_mask = torch.empty((chunk, max_rows, p.N), dtype=torch.int32, device=dev)
    out_body = torch.empty((chunk, max_rows), dtype=torch.int32, device=dev)
    max_L = max(p.L(d) for _, _, d in LAYER)
    import ctypes
    nb = (phe.load().phe_ntt_operand_bytes(ctypes.byref(p), chunk, max_L) if tabs else
          phe.load().phe_ct_operand_bytes(ctypes.byref(p), chunk, max_L))
    operand = torch.empty(nb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        for t0 in range(0, T, chunk):
            n = min(chunk, T - t0)
            for name, w, d_in in regs:
                seeds, body = inputs[d_in]
                mv = out_mask.view(-1)[: n * w.rows * p.N].view(n, w.rows, p.N)
                bv = out_body.view(-1)[: n * w.rows].view(n, w.rows)
                if tabs:
                    phe.ntt_ct_prepare(p, tabs, seeds[t0:t0 + n], body[t0:t0 + n], out=operand)
                    phe.matmul_clear_ntt(p, w, operand, n, out_mask=mv, out_body=bv)
                else:
                    phe.ct_prepare(p, seeds[t0:t0 + n], body[t0:t0 + n], out=operand)
                    phe.matmul_clear(p, w, operand, n, out_mask=mv, out_body=bv)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); step(); b.record(stream); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.mean(ts)
    ops = sum(2.0 * p.ell * d_out * d_in * (p.N + 1) for _, d_out, d_in in LAYER) * T
    return {"ms_per_layer": round(ms, 2), "layer_tok_s": round(T / (ms / 1e3), 1),
            "fwd_stack_tok_s": round(T / (ms / 1e3) / 16, 2),
            "int8_TOPS_equiv": round(ops / (ms / 1e3) / 1e12, 1),
            "ms_std": round(statistics.pstdev(ts), 2) if len(ts) > 1 else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", default="P0,P1,P2,P3,toyA")
    ap.add_argument("--tokens", default="256,512,1024,2048,4096,8192,16384")
    ap.add_argument("--contractions", default="tc,ntt")
    a = ap.parse_args()
    res = []
    for sname in a.sets.split(","):
        p = params(sname)
        for c in a.contractions.split(","):
            for T in map(int, a.tokens.split(",")):
                steps, warm = (3, 2) if T <= 2048 else (2, 1)
                r = run(p, T, c, steps, warm)
                r.update({"set": sname, "N": p.N, "q_in": p.q_in, "q_out": p.q_out, "T": T, "contraction": c,
                          "steps": steps, "warmup": warm})
                print(json.dumps(r), flush=True)
                res.append(r)
                torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump({"what": __doc__.split("\n")[0], "results": res},
              open(os.path.join(ROOT, "gpurun_out", "r1_sweep_c5.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
