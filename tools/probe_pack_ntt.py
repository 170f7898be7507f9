"""Times stage 2 of the packed primitive: tensor-core packing GEMM (phe_pack) vs the NTT-domain
KeySwitch (phe_pack_ntt) on q_proj-shaped digits (Table 1, rows = 2048), CUDA events."""
import sys
import torch
import os
import paper_2505_07329_b200 as phe
if os.environ.get("PHE_LIB"):
    phe.load(os.environ["PHE_LIB"])
import synth

T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
p = phe.params(phe.PRESET_PAPER)
W = synth.weights_int8(rows, 2048)
x = synth.activations_int8(T, 2048)
S = phe.keygen(p, 5)
seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).cuda(), 77)
w = phe.Weights(p, torch.from_numpy(W).cuda())
opnd = phe.ct_prepare(p, seeds, body)
ksk = phe.ksk_gen(p, S, 1234)
K, NK = phe.KeySwitchKey(p, ksk), phe.NttKeySwitchKey(p, ksk)
dig, bod = phe.matmul_clear_digits(p, w, opnd, T)
out_a = phe.pack(p, dig, bod, K)
out_b = phe.pack_ntt(p, dig, bod, NK)
torch.cuda.synchronize()
print("identical:", torch.equal(out_a, out_b))
for name, fn in [("pack_gemm", lambda: phe.pack(p, dig, bod, K, out=out_a)),
                 ("pack_ntt", lambda: phe.pack_ntt(p, dig, bod, NK, out=out_b))]:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); n = 3
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{name}: T={T} rows={rows}: {ms:.2f} ms  ({ms / T * 2048:.1f} ms per 2048 tokens)")
