"""C-ABI boundary checks that need no GPU (-m "not gpu"): the library loads, exports every
symbol include/phe.h declares, and its host-only calls (parameters, sizes, errors) behave."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "phe.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2505_07329_b200 import build
    build.build()
    import paper_2505_07329_b200 as phe
    return phe.load()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(phe_[a-z_0-9A-Z]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ["phe_params_init", "phe_keygen", "phe_encrypt_pack", "phe_matmul_clear",
                 "phe_matmul_clear_T", "phe_modswitch", "phe_decrypt_unpack"]:
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    import paper_2505_07329_b200 as phe
    syms = declared_symbols()
    assert set(syms) == set(phe.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_params_presets(lib):
    import paper_2505_07329_b200 as phe
    p = phe.params(phe.PRESET_PAPER)
    assert (p.N, p.q_in, p.q_out, p.beta, p.gamma) == (2048, 39, 26, 27, 12)  # Table 1
    assert phe.num_limbs(p) == 5 and phe.num_blocks(p, 8192) == 4 and phe.num_blocks(p, 768) == 1
    t = phe.params(phe.PRESET_TOY)
    assert (t.N, t.q_in, t.q_out, t.beta) == (1024, 32, 28, 21) and phe.num_limbs(t) == 4


def test_params_validation(lib):
    import paper_2505_07329_b200 as phe
    bad = [dict(N=1000), dict(q_out=40), dict(beta=10, gamma=12), dict(q_in=65), dict(noise_eta=40)]
    for b in bad:
        with pytest.raises(phe.PheError):
            phe.params(phe.PRESET_PAPER, **b)


def test_sizes(lib):
    import paper_2505_07329_b200 as phe
    p = phe.params(phe.PRESET_PAPER)
    P = ctypes.byref(p)
    # 16-shift expansion + padded plain copy
    assert lib.phe_weights_bytes(P, 2048, 2048) == 2048 * 1 * 4096 * 16 + 2048 * 2048
    assert lib.phe_weights_bytes(P, 40, 3000) == 40 * 2 * 4096 * 16 + 128 * 4096
    # two limb-plane matrices, rows padded to a multiple of 256
    assert lib.phe_ct_operand_bytes(P, 2048, 1) == 2 * 10240 * 2048
    assert lib.phe_ct_operand_bytes(P, 1, 4) == 2 * 256 * 4 * 2048
    assert lib.phe_weights_bytes(P, 0, 10) == 0


def test_strerror(lib):
    assert lib.phe_strerror(0) == b"ok"
    assert lib.phe_strerror(3) == b"modulus mismatch"


def test_validation_errors_without_launch(lib):
    """Argument validation is synchronous and enqueues nothing: safe without a GPU."""
    import paper_2505_07329_b200 as phe
    p = phe.params(phe.PRESET_PAPER)
    P = ctypes.byref(p)
    # out_bits neither q_in nor q_out -> EMODULUS
    assert lib.phe_matmul_clear(P, None, 8, 8, 0, 8, None, 4, 30, None, None, None) == phe.PHE_EMODULUS
    # bad row range -> EINVAL
    assert lib.phe_matmul_clear(P, None, 8, 8, 4, 9, None, 4, 26, None, None, None) == phe.PHE_EINVAL
    # T == 0 is a no-op
    assert lib.phe_matmul_clear(P, None, 8, 8, 0, 8, None, 0, 26, None, None, None) == phe.PHE_OK
    # modswitch to_bits > 32 -> EINVAL
    assert lib.phe_modswitch(None, None, 4, 39, 33, None) == phe.PHE_EINVAL
    # too-small prepared-weight buffer -> ENOMEM
    assert lib.phe_weights_prepare(P, ctypes.c_void_p(16), 8, 8, 0, ctypes.c_void_p(16), 10, None) == phe.PHE_ENOMEM
    # N < 128 unsupported on the GPU path
    q = phe.params(phe.PRESET_PAPER, N=64)
    assert lib.phe_keygen(ctypes.byref(q), 1, ctypes.c_void_p(16), None) == phe.PHE_EUNSUPPORTED


def test_product_package_does_not_import_oracle():
    """The CUDA path shares no code with oracle/ and never imports it."""
    pkg = os.path.join(ROOT, "paper_2505_07329_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(dirpath, f)).read()
                code = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
                code = re.sub(r"#.*|//.*", "", code)
                for bad in ("import oracle", "from oracle", "phe_oracle", "c_oracle"):
                    assert bad not in code, (f, bad)


def test_wire_sizes_match_paper(lib):
    """P:223-224 print 9992 B per seeded input block and 13312 B per packed output ciphertext."""
    import paper_2505_07329_b200 as phe
    p = phe.params(phe.PRESET_PAPER)
    assert phe.wire_input_bytes(p) == 9992
    assert phe.wire_output_bytes(p) == 13312


def test_ntt_keyswitch_sizes_and_support(lib):
    """NEXT #1 stage 2 in the NTT domain (R24): buffer sizes and the CRT-range support rule are
    host-side; unsupported parameter sets report 0 bytes / EUNSUPPORTED without a launch."""
    import paper_2505_07329_b200 as phe
    p = phe.params(phe.PRESET_PAPER)
    P = ctypes.byref(p)
    N = 2048
    tables = (2 * 2 * N + 2 * 7 * (N // 8)) * 8           # fwd + inv + last-phase twiddles, 2 primes
    tables = (tables + 255) // 256 * 256
    khat = 2 * 4 * N * 4 * N * 4                          # [2 primes][4N rows][4 parts][N] u32
    assert lib.phe_ntt_ksk_bytes(P) == tables + khat
    # T = 2048, one ciphertext group: one K-split (the grid fills its waves), partials + accumulator
    assert lib.phe_pack_ntt_ws_bytes(P, 2048, 2048) == 2048 * 2 * 4 * N * 4 + 2048 * 2 * N * 8
    ws_small = lib.phe_pack_ntt_ws_bytes(P, 2048, 16)      # small T: K-split partials
    assert ws_small > 16 * 2 * 4 * N * 4 and (ws_small - 16 * 2 * N * 8) % (16 * 2 * 4 * N * 4) == 0
    assert lib.phe_packed_ntt_ws_bytes(P, 2048, 16) >= ws_small + 16 * 2048 * 4 * N
    # q_in = 24 < 32 bits of the 4-level gadget (R18): not supported
    q = phe.params(phe.PRESET_PAPER, q_in=24, q_out=20, beta=20, gamma=8)
    assert lib.phe_ntt_ksk_bytes(ctypes.byref(q)) == 0
    assert lib.phe_ntt_ksk_prepare(ctypes.byref(q), ctypes.c_void_p(16), ctypes.c_void_p(16), 1 << 30,
                                   None) == phe.PHE_EUNSUPPORTED
    # too-small buffers -> ENOMEM, T == 0 -> no-op, all before any launch
    assert lib.phe_ntt_ksk_prepare(P, ctypes.c_void_p(16), ctypes.c_void_p(16), 16, None) == phe.PHE_ENOMEM
    assert lib.phe_pack_ntt(P, ctypes.c_void_p(16), ctypes.c_void_p(16), 4, 2048, ctypes.c_void_p(16),
                            ctypes.c_void_p(16), 16, ctypes.c_void_p(16), None) == phe.PHE_ENOMEM
    assert lib.phe_pack_ntt(P, None, None, 0, 2048, None, None, 0, None, None) == phe.PHE_OK
