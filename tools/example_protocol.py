"""End-to-end use of the public API for one private-inference linear, as the protocol runs it
(P:174-191): the client encrypts int8 activations and ships wire-format input blocks (9992 B
each at Table 1); the server, holding the public int8 weights, returns either LWE
ciphertexts at q_out bits (the hot path, Eq. 6 + the 39 -> 26 switch) or packed RLWE ciphertexts
(13312 B each; Eq. 7/8); the client decrypts and recovers W.x up to the gamma-MSB contract
(P:198).  Host buffers on both sides of the "network", so this is exactly what a deployment calls.

  python tools/example_protocol.py [--d_out 2048 --d_in 2048 --tokens 16] [--packed]

Not part of the bench contract; tests/test_gpu_example.py runs it small."""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(d_out=2048, d_in=2048, tokens=16, packed=False, noise_eta=21, seed=7):
    import numpy as np
    import torch

    import paper_2505_07329_b200 as phe
    import synth

    # ---- client: parameters (Table 1 with CBD(21) encryption noise: the presets' E = 0 is for
    # parity runs only), secret key, quantized activations, encryption, wire serialization
    p = phe.params(phe.PRESET_PAPER, noise_eta=noise_eta)
    S = phe.keygen(p, seed)
    x = synth.activations_int8(tokens, d_in, seed=seed + 1)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).cuda(), synth.seed_base(seed), noise_seed=seed + 2)
    wire_in = phe.wire_serialize_inputs(p, seeds, body).cpu().pin_memory()      # -> network

    # ---- server: public weights registered once; one call per request on host buffers
    W = synth.weights_int8(d_out, d_in, seed=seed + 3)
    w = phe.Weights(p, torch.from_numpy(W).cuda())
    if packed:
        # client-made KeySwitch key (sigma_ksk rounds to 0 at q = 2^39, R19), server-registered
        p_ksk = phe.params(phe.PRESET_PAPER, noise_eta=0)
        K = phe.NttKeySwitchKey(p, phe.ksk_gen(p_ksk, S, seed + 4))
        G = (d_out + p.N - 1) // p.N
        wire_out = torch.empty((tokens, G, phe.wire_output_bytes(p)), dtype=torch.uint8, pin_memory=True)
        phe.server_wire_host_ntt(p, w, K, wire_in, wire_out)                     # -> network
    else:
        wire_out = torch.empty((tokens, phe.wire_lwe_bytes(p, d_out)), dtype=torch.uint8, pin_memory=True)
        phe.server_matvec_wire_host(p, w, wire_in, wire_out)                      # -> network

    # ---- client: deserialize, decrypt, compare with the plaintext product
    if packed:
        ct = phe.wire_deserialize_packed(p, wire_out.cuda())                   # [T][G][2][N]
        y = phe.decrypt_packed(p, S, ct, d_out).cpu().numpy().astype(np.int64)
    else:
        m, b = phe.wire_deserialize_lwe(p, wire_out.cuda(), d_out)
        y = phe.decrypt_unpack(p, S, m, b, p.q_out).cpu().numpy().astype(np.int64)
    wx = x.astype(np.int64) @ W.astype(np.int64).T
    t = 1 << p.beta
    err = (y - wx + t // 2) % t - t // 2            # centred difference mod t
    return {"tokens": tokens, "d_out": d_out, "d_in": d_in, "packed": packed,
            "bytes_up": int(wire_in.numel()), "bytes_down": int(wire_out.numel()),
            "max_abs_error": int(np.abs(err).max()),
            "msb_bound": 1 << (p.beta - p.gamma),   # the gamma = 12 MSBs of beta = 27 bits
            "ok": bool(np.abs(err).max() < (1 << (p.beta - p.gamma)))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d_out", type=int, default=2048)
    ap.add_argument("--d_in", type=int, default=2048)
    ap.add_argument("--tokens", type=int, default=16)
    ap.add_argument("--packed", action="store_true")
    a = ap.parse_args()
    print(run(a.d_out, a.d_in, a.tokens, a.packed))


if __name__ == "__main__":
    main()
