"""Ad-hoc kernel probe (not part of the product or the bench contract): times matmul_clear
(mask GEMM only) for a given linear shape and reports int8 TOP/s and the SM clock."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2505_07329_b200 as phe  # noqa: E402
import synth  # noqa: E402

if os.environ.get("PHE_LIB"):  # experiment builds (tools/build_variant.sh)
    phe.load(os.environ["PHE_LIB"])
from bench import ClockSampler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d_out", type=int, default=2048)
    ap.add_argument("--d_in", type=int, default=2048)
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--transpose", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--wire", action="store_true", help="phe_matmul_clear_wire (bit-packed outputs)")
    a = ap.parse_args()
    p = phe.params(phe.PRESET_PAPER)
    W = torch.from_numpy(synth.weights_int8(a.d_out, a.d_in)).cuda()
    w = phe.Weights(p, W, transpose=a.transpose)
    S = phe.keygen(p, 1)
    x = torch.from_numpy(synth.activations_int8(a.T, w.cols)).cuda()
    seeds, body = phe.encrypt_pack(p, S, x, 5)
    op = phe.ct_prepare(p, seeds, body)
    out = torch.empty((a.T, w.rows, p.N), dtype=torch.int32, device="cuda")
    f = phe.matmul_clear_T if a.transpose else phe.matmul_clear
    if a.wire:
        del out
        wout = torch.empty((a.T, phe.wire_lwe_bytes(p, w.rows)), dtype=torch.uint8, device="cuda")
        wws = torch.empty(phe.load().phe_matmul_clear_wire_ws_bytes(__import__("ctypes").byref(p), a.T, w.rows),
                          dtype=torch.uint8, device="cuda")
        f = lambda p_, w_, op_, T_, out_mask=None, out_body=None: phe.matmul_clear_wire(p_, w_, op_, T_, out=wout, ws=wws)  # noqa: E731
        out = None
    for _ in range(2):
        f(p, w, op, a.T, out_mask=out, out_body=phe.SKIP)
    torch.cuda.synchronize()
    clk = ClockSampler(0)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f(p, w, op, a.T, out_mask=out, out_body=phe.SKIP)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    c = clk.stop()
    ms = statistics.median(ts)
    ops = 2.0 * p.ell * w.rows * w.cols * p.N * a.T
    mhz = c["sm_mhz"] or 0
    cyc = ms * 1e-3 * mhz * 1e6
    ideal = ops / 2 / (8192 * 148)
    print(f"{w.rows}x{w.cols} T={a.T} {'T' if a.transpose else ''}: {ms:.3f} ms, {ops / ms / 1e9:.1f} TOP/s, "
          f"sm {mhz} MHz, cycles {cyc / 1e6:.1f}M vs ideal {ideal / 1e6:.1f}M -> {ideal / max(cyc, 1):.3f} {c['reasons']}")


if __name__ == "__main__":
    main()
