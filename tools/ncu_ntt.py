"""One NTT-path mask launch for ncu (tools/gpu_*.sh): q_proj 2048x2048 (or --shape), T tokens."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2505_07329_b200 as phe  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="2048x2048x512")
ap.add_argument("--launches", type=int, default=2)
a = ap.parse_args()
d_out, d_in, T = map(int, a.shape.split("x"))
p = phe.params(phe.PRESET_PAPER)
tabs = phe.NttTables(p)
S = phe.keygen(p, 1)
W = torch.from_numpy(synth.weights_int8(d_out, d_in)).cuda()
x = torch.from_numpy(synth.activations_int8(T, d_in)).cuda()
seeds, body = phe.encrypt_pack(p, S, x, 5)
wn = phe.NttWeights(p, tabs, W)
op = phe.ntt_ct_prepare(p, tabs, seeds, body)
out = torch.empty((T, d_out, p.N), dtype=torch.int32, device="cuda")
for _ in range(a.launches):
    phe.matmul_clear_ntt(p, wn, op, T, out_mask=out, out_body=phe.SKIP)
torch.cuda.synchronize()
print("ok")
