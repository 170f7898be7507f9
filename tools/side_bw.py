"""Side-kernel bandwidth report (north_star: "achieved HBM GB/s for the pack and modswitch
kernels").  Times each non-GEMM kernel of the path with CUDA events at bench-scale sizes
(q_proj, T = 2048, Table 1 parameters) and reports ALGORITHMIC bytes / time against the measured
HBM peak (MEASURED_PEAKS.json).  ALU-bound kernels (ChaCha20 expansion, binary-key products,
NTTs) are reported with their bytes too, marked bound "alu".  Run under ncu with --reps 1 for
the DRAM-bytes cross-check.  Not part of the product or the bench contract."""
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


def timeit(fn, reps):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--T", type=int, default=2048)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 7700.0
    p = phe.params(phe.PRESET_PAPER)
    N, T, d = p.N, a.T, 2048
    ell = p.ell
    out = []

    def rep(name, ms, rd, wr, bound="hbm", note=""):
        gbs = (rd + wr) / (ms / 1e3) / 1e9
        out.append({"kernel": name, "ms": round(ms, 4), "bytes_read": int(rd), "bytes_written": int(wr),
                    "achieved_GBps": round(gbs, 1), "bound": bound,
                    "frac_of_hbm_peak": round(gbs / peak, 3) if bound == "hbm" else None, "note": note})

    S = phe.keygen(p, 1)
    x = torch.from_numpy(synth.activations_int8(T, d)).cuda()
    f = lambda: phe.encrypt_pack(p, S, x, 5)
    f(); ms = timeit(f, a.reps)
    rep("encrypt_kernel (encrypt_pack, client)", ms, T * d + N, T * 8 + T * N * 8, "alu",
        "B = A*S + E + Delta*x: N^2/2 adds per block (binary S), ChaCha20 expansion of A")
    tabs = phe.NttTables(p)
    f = lambda: phe.encrypt_pack_ntt(p, tabs, S, x, 5)
    f(); ms = timeit(f, a.reps)
    rep("ntt_encrypt_kernel (encrypt_pack_ntt, client)", ms, T * d + N, T * 8 + T * N * 8, "alu",
        "A*S through NTT(A) o NTT(S) mod 2 primes + CRT: O(N log N) per block; bit-identical to encrypt_kernel")
    seeds, body = phe.encrypt_pack(p, S, x, 5)
    op = phe.ct_prepare(p, seeds, body)
    f = lambda: phe.ct_prepare(p, seeds, body, out=op)
    f(); ms = timeit(f, a.reps)
    rep("ct_prepare_kernel (a3+a4)", ms, T * 8 + T * N * 8, 2 * T * ell * N, "alu",
        "ChaCha20 mask expansion (N/8 blocks per input block) + limb planes of masks and bodies")
    opn = phe.ntt_ct_prepare(p, tabs, seeds, body)
    f = lambda: phe.ntt_ct_prepare(p, tabs, seeds, body, out=opn)
    f(); ms = timeit(f, a.reps)
    rep("ntt_masks_kernel + body planes (phe_ntt_ct_prepare)", ms, T * 8 + T * N * 8, T * 2 * N * 4 + T * ell * N,
        "alu", "ChaCha20 + forward NTT mod 2 primes per input block")
    # modswitch: 2^29 words (4 GiB in, 2 GiB out)
    n = 1 << 29
    v = torch.randint(0, 2 ** 39, (n,), dtype=torch.int64, device="cuda")
    o32 = torch.empty(n, dtype=torch.int32, device="cuda")
    f = lambda: phe.modswitch(v, 39, 26, out=o32)
    f(); ms = timeit(f, a.reps)
    rep("modswitch_kernel (a8 standalone, 2^29 words)", ms, 8 * n, 4 * n)
    del v, o32
    # decrypt of the q_proj outputs (T x 2048 LWE ciphertexts, u32 words): 34 GB read
    w = phe.Weights(p, torch.from_numpy(synth.weights_int8(d, d)).cuda())
    m26, b26 = phe.matmul_clear(p, w, op, T)
    f = lambda: phe.decrypt_unpack(p, S, m26, b26, p.q_out)
    f(); ms = timeit(f, a.reps)
    rep("decrypt_kernel (decrypt_unpack of q_proj outputs, client)", ms, T * d * (N + 1) * 4 + N, T * d * 4)
    del m26, b26, w, op, opn
    torch.cuda.empty_cache()
    # wire format (NEXT #2) at 8x the tokens (0.4 GB per direction: bandwidth, not launch, bound)
    Tw = 8 * T
    sw_ = seeds.repeat(8, 1).contiguous()
    bw_ = body.repeat(8, 1, 1).contiguous()
    wi = phe.wire_serialize_inputs(p, sw_, bw_)
    f = lambda: phe.wire_serialize_inputs(p, sw_, bw_)
    ms = timeit(f, a.reps)
    rep(f"wire serialize input blocks ({Tw} blocks, NEXT #2)", ms, Tw * 8 + Tw * N * 8, wi.numel())
    f = lambda: phe.wire_deserialize_inputs(p, wi)
    f(); ms = timeit(f, a.reps)
    rep(f"wire deserialize input blocks ({Tw} blocks, NEXT #2)", ms, wi.numel(), Tw * 8 + Tw * N * 8)
    del sw_, bw_, wi
    pk = torch.randint(0, 2 ** p.q_out, (Tw, 1, 2, N), dtype=torch.int32, device="cuda")
    wo = phe.wire_serialize_packed(p, pk)
    f = lambda: phe.wire_serialize_packed(p, pk)
    ms = timeit(f, a.reps)
    rep(f"wire serialize packed RLWE outputs ({Tw} ciphertexts, NEXT #2)", ms, pk.numel() * 4, wo.numel())
    f = lambda: phe.wire_deserialize_packed(p, wo)
    f(); ms = timeit(f, a.reps)
    rep(f"wire deserialize packed RLWE outputs ({Tw} ciphertexts, NEXT #2)", ms, wo.numel(), pk.numel() * 4)
    for r in out:
        print(json.dumps(r))
    json.dump({"hbm_peak_GBps": peak, "T": T, "kernels": out},
              open(os.path.join(ROOT, "gpurun_out", "r1_side_kernels.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
