"""Ad-hoc probe (not product, not the bench contract): times the mask contraction of one linear
through the NTT path (phe_matmul_clear_ntt) and the tensor-core path (phe_matmul_clear), same
inputs, and reports ms, output coefficients/s and the SM clock.  PHE_NTT_TOK varies tokens/CTA
(experiment builds only: -DPHE_KERNEL_EXPERIMENTS=1)."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_07329_b200 as phe  # noqa: E402
import synth  # noqa: E402
from bench import ClockSampler  # noqa: E402


def timeit(fn, reps):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="2048x2048x2048,2048x8192x512,8192x2048x512")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dense", type=int, default=1)
    a = ap.parse_args()
    p = phe.params(phe.PRESET_PAPER)
    tabs = phe.NttTables(p)
    S = phe.keygen(p, 1)
    for shp in a.shapes.split(","):
        d_out, d_in, T = map(int, shp.split("x"))
        W = torch.from_numpy(synth.weights_int8(d_out, d_in)).cuda()
        x = torch.from_numpy(synth.activations_int8(T, d_in)).cuda()
        seeds, body = phe.encrypt_pack(p, S, x, 5)
        wn = phe.NttWeights(p, tabs, W)
        opn = phe.ntt_ct_prepare(p, tabs, seeds, body)
        out = torch.empty((T, d_out, p.N), dtype=torch.int32, device="cuda")
        f_ntt = lambda: phe.matmul_clear_ntt(p, wn, opn, T, out_mask=out, out_body=phe.SKIP)
        f_ntt(); torch.cuda.synchronize()
        clk = ClockSampler(0)
        t_ntt = timeit(f_ntt, a.reps)
        c = clk.stop()
        t_prep = timeit(lambda: phe.ntt_ct_prepare(p, tabs, seeds, body, out=opn), a.reps)
        coef = T * d_out * p.N
        msg = (f"{d_out}x{d_in} T={T}: ntt {t_ntt:.2f} ms ({coef / t_ntt / 1e9:.2f} Gcoef/s, "
               f"clk {c.get('sm_mhz')} MHz) ntt_prep {t_prep:.3f} ms")
        if a.dense:
            del opn, wn
            wd = phe.Weights(p, W)
            opd = phe.ct_prepare(p, seeds, body)
            f_d = lambda: phe.matmul_clear(p, wd, opd, T, out_mask=out, out_body=phe.SKIP)
            f_d(); torch.cuda.synchronize()
            clk = ClockSampler(0)
            t_d = timeit(f_d, a.reps)
            c2 = clk.stop()
            msg += f" | dense {t_d:.2f} ms (clk {c2.get('sm_mhz')} MHz) ratio dense/ntt {t_d / t_ntt:.2f}"
            del wd, opd
        print(msg, flush=True)
        del out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
