"""SURVEY §8(d) "extra": the paper's Table 3 shape set at T = 1 (latency) and
T = 2048 (throughput).  Table 3 times the paper's whole primitive (Eq. 6 + KeySwitch packing
Eq. 7/8 + switch) for one token on an RTX 4060 Laptop; the like-for-like computation here is
matmul_clear_packed (NEXT #1).  The LWE hot path (north_star) is timed through both
contractions too.  Context only (different GPU).  Writes gpurun_out/r2_table3.json."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_07329_b200 as phe  # noqa: E402
import synth  # noqa: E402

SHAPES = [(768, 768, 0.0809), (3072, 768, 0.1528), (2048, 2048, 0.2402), (768, 3072, 0.3389),
          (8192, 2048, 0.6368), (2048, 8192, 1.0539)]  # (d_in, d_out, paper latency s)


def timeit(fn, reps):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), (statistics.pstdev(ts) if len(ts) > 1 else 0.0)


def main():
    p = phe.params(phe.PRESET_PAPER)
    S = phe.keygen(p, 1)
    K = phe.KeySwitchKey(p, phe.ksk_gen(p, S, 2))
    tabs = phe.NttTables(p)
    out = []
    for d_in, d_out, paper_s in SHAPES:
        W = synth.weights_int8_torch(d_out, d_in, device="cuda")
        w = phe.Weights(p, W)
        wn = phe.NttWeights(p, tabs, W)
        for T in (1, 2048):
            x = torch.from_numpy(synth.activations_int8(T, d_in, seed=T + d_in)).cuda()
            seeds, body = phe.encrypt_pack(p, S, x, 9)
            reps = 20 if T == 1 else 3
            C = min(T, 255)  # token chunks (5 x 51-token tiles): bounded outputs / workspace
            op = torch.empty(phe.load().phe_ct_operand_bytes(__import__("ctypes").byref(p), C, p.L(d_in)),
                             dtype=torch.uint8, device="cuda")
            opn = torch.empty(phe.load().phe_ntt_operand_bytes(__import__("ctypes").byref(p), C, p.L(d_in)),
                              dtype=torch.uint8, device="cuda")
            m = torch.empty((C, d_out, p.N), dtype=torch.int32, device="cuda")
            bo = torch.empty((C, d_out), dtype=torch.int32, device="cuda")

            def chunks(f):
                for t0 in range(0, T, C):
                    n = min(C, T - t0)
                    f(t0, n)

            # full primitive: prepare + Eq. 6 + Eq. 7/8 + switch (packed RLWE outputs)
            pk = lambda: chunks(lambda t0, n: (phe.ct_prepare(p, seeds[t0:t0 + n], body[t0:t0 + n], out=op),
                                               phe.matmul_clear_packed(p, w, op, n, K)))
            t_pk, s_pk = timeit(pk, reps)
            # LWE hot path (north_star), both contractions
            tc = lambda: chunks(lambda t0, n: (phe.ct_prepare(p, seeds[t0:t0 + n], body[t0:t0 + n], out=op),
                                               phe.matmul_clear(p, w, op, n, out_mask=m[:n], out_body=bo[:n])))
            t_tc, _ = timeit(tc, reps)
            nt = lambda: chunks(lambda t0, n: (phe.ntt_ct_prepare(p, tabs, seeds[t0:t0 + n], body[t0:t0 + n], out=opn),
                                               phe.matmul_clear_ntt(p, wn, opn, n, out_mask=m[:n], out_body=bo[:n])))
            t_nt, _ = timeit(nt, reps)
            r = {"d_in": d_in, "d_out": d_out, "T": T, "paper_latency_s_T1_rtx4060": paper_s,
                 "packed_ms": round(t_pk, 3), "packed_ms_std": round(s_pk, 3),
                 "lwe_tc_ms": round(t_tc, 3), "lwe_ntt_ms": round(t_nt, 3),
                 "packed_tok_s": round(T / (t_pk / 1e3), 1)}
            if T == 1:
                r["speedup_vs_paper_packed"] = round(paper_s / (t_pk / 1e3), 1)
            print(json.dumps(r), flush=True)
            out.append(r)
            del m, bo, op, opn
            phe._ws_cache.clear() if hasattr(phe, "_ws_cache") else None
            torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump({"what": __doc__.split("\n")[0], "results": out},
              open(os.path.join(ROOT, "gpurun_out", "r2_table3.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
