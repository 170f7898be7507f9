"""One packed-path step (q_proj, T tokens) for ncu: digits GEMM + pack GEMM."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2505_07329_b200 as phe  # noqa: E402
import synth  # noqa: E402
T = int(sys.argv[1]) if len(sys.argv) > 1 else 102
p = phe.params(phe.PRESET_PAPER)
S = phe.keygen(p, 1)
K = phe.KeySwitchKey(p, phe.ksk_gen(p, S, 2))
w = phe.Weights(p, synth.weights_int8_torch(2048, 2048, device="cuda"))
x = torch.from_numpy(synth.activations_int8(T, 2048)).cuda()
seeds, body = phe.encrypt_pack(p, S, x, 9)
op = phe.ct_prepare(p, seeds, body)
for _ in range(2):
    phe.matmul_clear_packed(p, w, op, T, K)
torch.cuda.synchronize()
print("ok")
