"""Ad-hoc probe: time the packed primitive RLWE(Wx) = Eq. 6 + Eq. 7/8 for one linear."""
import argparse, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2505_07329_b200 as phe
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--d_out", type=int, default=2048)
ap.add_argument("--d_in", type=int, default=2048)
ap.add_argument("--T", type=int, default=256)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
p = phe.params(phe.PRESET_PAPER)
W = synth.weights_int8_torch(a.d_out, a.d_in, device="cuda")
w = phe.Weights(p, W)
S = phe.keygen(p, 1)
x = torch.from_numpy(synth.activations_int8(a.T, a.d_in)).cuda()
seeds, body = phe.encrypt_pack(p, S, x, 5)
op = phe.ct_prepare(p, seeds, body)
K = phe.KeySwitchKey(p, phe.ksk_gen(p, S, 9))
out = phe.matmul_clear_packed(p, w, op, a.T, K)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); phe.matmul_clear_packed(p, w, op, a.T, K, out=out); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
pack_ops = 2.0 * 2 * p.ell * phe.KS_LEVELS * p.N * p.N * a.d_out * a.T
hot_ops = 2.0 * p.ell * a.d_out * a.d_in * (p.N + 1) * a.T
print(f"{a.d_out}x{a.d_in} T={a.T}: packed primitive {ms:.2f} ms, {a.T / ms * 1e3:.1f} tok/s, "
      f"int8 TOP/s (pack+hot) {(pack_ops + hot_ops) / ms / 1e9:.0f}")
y = phe.decrypt_packed(p, S, out, a.d_out)
wx = (x.double() @ W.double().T)
print("max |dec - Wx|:", (y.double() - wx).abs().max().item())
