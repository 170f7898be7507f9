"""Python binding of libphe (include/phe.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libphe.so; this module allocates
torch device tensors for the outputs, passes raw pointers and the current CUDA stream, and
raises on any non-zero return code.  There is no CPU fallback: if libphe.so is missing or
no GPU is present, `load()` raises.

Storage convention: uint64 ciphertext words live in torch.int64 tensors and uint32 words in
torch.int32 tensors (same bits; every value the path produces is < 2^63 / < 2^31 except the
public seeds, which are opaque 64-bit patterns).
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libphe.so")

PHE_OK, PHE_EINVAL, PHE_ERANGE, PHE_EMODULUS, PHE_ENOMEM, PHE_ECUDA, PHE_EUNSUPPORTED = range(7)
PRESET_PAPER, PRESET_TOY = 0, 1
KS_LEVELS = 4  # KeySwitch gadget levels (base 2^8), R18

# every symbol include/phe.h declares (checked by tests/test_boundary.py)
EXPORTS = [
    "phe_strerror", "phe_last_cuda_error", "phe_params_init", "phe_params_validate",
    "phe_num_limbs", "phe_num_blocks", "phe_keygen", "phe_encrypt_pack", "phe_weights_bytes",
    "phe_weights_prepare", "phe_ct_operand_bytes", "phe_ct_prepare", "phe_matmul_clear",
    "phe_matmul_clear_T", "phe_modswitch", "phe_decrypt_unpack", "phe_server_matvec_host",
    "phe_last_launch_count", "phe_matmul_clear_simt",
    "phe_ksk_bytes", "phe_ksk_gen", "phe_ksk_prep_bytes", "phe_ksk_prepare", "phe_packed_ws_bytes",
    "phe_matmul_clear_packed", "phe_decrypt_packed", "phe_matmul_clear_digits", "phe_pack_acc_bytes",
    "phe_pack", "phe_server_matvec_packed_host",
    "phe_wire_input_bytes", "phe_wire_output_bytes", "phe_wire_serialize_inputs", "phe_wire_deserialize_inputs",
    "phe_wire_serialize_packed", "phe_wire_deserialize_packed", "phe_server_wire_host",
    "phe_ntt_primes", "phe_ntt_max_blocks", "phe_ntt_tables_bytes", "phe_ntt_tables_init",
    "phe_ntt_weights_bytes", "phe_ntt_weights_prepare", "phe_ntt_operand_bytes", "phe_ntt_ct_prepare",
    "phe_matmul_clear_ntt", "phe_matmul_clear_ntt_T", "phe_matmul_clear_ct", "phe_encrypt_pack_ntt",
    "phe_ntt_ksk_bytes", "phe_ntt_ksk_prepare", "phe_pack_ntt_ws_bytes", "phe_pack_ntt",
    "phe_packed_ntt_ws_bytes", "phe_matmul_clear_packed_ntt", "phe_server_wire_host_ntt",
    "phe_matmul_clear_packed_nttw", "phe_server_wire_host_nttw",
    "phe_wire_lwe_bytes", "phe_wire_serialize_lwe", "phe_wire_deserialize_lwe", "phe_server_matvec_wire_host",
    "phe_matmul_clear_digits_ntt", "phe_matmul_clear_into", "phe_matmul_clear_ntt_into",
    "phe_server_matvec_host_ws_bytes", "phe_server_matvec_packed_host_ws_bytes", "phe_server_wire_host_ws_bytes",
    "phe_server_wire_host_ntt_ws_bytes", "phe_server_wire_host_nttw_ws_bytes",
    "phe_server_matvec_wire_host_ws_bytes", "phe_matmul_clear_wire_ws_bytes", "phe_wire_lwe_direct_supported",
    "phe_matmul_clear_wire",
]


class Params(ctypes.Structure):
    """phe_params (Table 1)."""
    _fields_ = [("N", ctypes.c_int32), ("q_in", ctypes.c_int32), ("q_out", ctypes.c_int32),
                ("beta", ctypes.c_int32), ("gamma", ctypes.c_int32), ("noise_eta", ctypes.c_int32)]

    def __repr__(self):
        return (f"Params(N={self.N}, q_in={self.q_in}, q_out={self.q_out}, beta={self.beta}, "
                f"gamma={self.gamma}, noise_eta={self.noise_eta})")

    @property
    def ell(self) -> int:
        return (self.q_in + 7) // 8

    def L(self, d: int) -> int:
        return (d + self.N - 1) // self.N


class PheError(RuntimeError):
    pass


_lib = None
_P = ctypes.POINTER(Params)
_vp, _i64, _i32, _u64, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_size_t


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libphe.so (raises if missing: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise PheError(f"libphe.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    sig = {
        "phe_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "phe_last_cuda_error": ([], ctypes.c_int),
        "phe_last_launch_count": ([], ctypes.c_int),
        "phe_params_init": ([_P, ctypes.c_int], ctypes.c_int),
        "phe_params_validate": ([_P], ctypes.c_int),
        "phe_num_limbs": ([_P], ctypes.c_int),
        "phe_num_blocks": ([_P, _i64], _i64),
        "phe_keygen": ([_P, _u64, _vp, _vp], ctypes.c_int),
        "phe_encrypt_pack": ([_P, _vp, _vp, _i64, _i64, _u64, _u64, _vp, _vp, _vp], ctypes.c_int),
        "phe_weights_bytes": ([_P, _i64, _i64], _sz),
        "phe_weights_prepare": ([_P, _vp, _i64, _i64, ctypes.c_int, _vp, _sz, _vp], ctypes.c_int),
        "phe_ct_operand_bytes": ([_P, _i64, _i64], _sz),
        "phe_ct_prepare": ([_P, _vp, _vp, _i64, _i64, _vp, _sz, _vp], ctypes.c_int),
        "phe_matmul_clear": ([_P, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _i32, _vp, _vp, _vp], ctypes.c_int),
        "phe_matmul_clear_T": ([_P, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _i32, _vp, _vp, _vp], ctypes.c_int),
        "phe_matmul_clear_simt": ([_P, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _i32, _vp, _vp, _vp], ctypes.c_int),
        "phe_modswitch": ([_vp, _vp, _i64, _i32, _i32, _vp], ctypes.c_int),
        "phe_decrypt_unpack": ([_P, _vp, _vp, _vp, _i64, _i64, _i32, _vp, _vp], ctypes.c_int),
        "phe_server_matvec_host": ([_P, _vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp, _vp, _i64,
                                    _i64, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
        "phe_server_matvec_host_ws_bytes": ([_P, _i64, _i64, ctypes.c_int, _i64, _i64, _i64, _i64], _sz),
        "phe_matmul_clear_wire_ws_bytes": ([_P, _i64, _i64], _sz),
        "phe_wire_lwe_direct_supported": ([_P, _i64], ctypes.c_int),
        "phe_matmul_clear_wire": ([_P, _vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp, _i64, _vp, _vp, _sz, _vp],
                                  ctypes.c_int),
        "phe_server_matvec_wire_host_ws_bytes": ([_P, _i64, _i64, ctypes.c_int, _i64, _i64, _i64, _i64], _sz),
        "phe_server_matvec_packed_host_ws_bytes": ([_P, _i64, _i64, ctypes.c_int, _i64, _i64], _sz),
        "phe_server_wire_host_ws_bytes": ([_P, _i64, _i64, ctypes.c_int, _i64, _i64], _sz),
        "phe_server_wire_host_ntt_ws_bytes": ([_P, _i64, _i64, ctypes.c_int, _i64, _i64], _sz),
        "phe_server_wire_host_nttw_ws_bytes": ([_P, _i64, _i64, ctypes.c_int, _i64, _i64], _sz),
        "phe_ksk_bytes": ([_P], _sz),
        "phe_ksk_gen": ([_P, _vp, _u64, _vp, _sz, _vp], ctypes.c_int),
        "phe_ksk_prep_bytes": ([_P], _sz),
        "phe_ksk_prepare": ([_P, _vp, _vp, _sz, _vp], ctypes.c_int),
        "phe_packed_ws_bytes": ([_P, _i64, _i64], _sz),
        "phe_matmul_clear_packed": ([_P, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, _vp, _vp, _sz, _vp, _vp],
                                    ctypes.c_int),
        "phe_decrypt_packed": ([_P, _vp, _vp, _i64, _i64, _i32, _vp, _vp], ctypes.c_int),
        "phe_matmul_clear_digits": ([_P, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, _vp, _vp, _vp], ctypes.c_int),
        "phe_pack_acc_bytes": ([_P, _i64, _i64], _sz),
        "phe_pack": ([_P, _vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp, _vp], ctypes.c_int),
        "phe_server_matvec_packed_host": ([_P, _vp, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _i64, _i64, _vp,
                                           _vp, _sz, _vp], ctypes.c_int),
        "phe_wire_input_bytes": ([_P], _sz),
        "phe_wire_output_bytes": ([_P], _sz),
        "phe_wire_serialize_inputs": ([_P, _vp, _vp, _i64, _i64, _vp, _vp], ctypes.c_int),
        "phe_wire_deserialize_inputs": ([_P, _vp, _i64, _i64, _vp, _vp, _vp], ctypes.c_int),
        "phe_wire_serialize_packed": ([_P, _vp, _i64, _vp, _vp], ctypes.c_int),
        "phe_wire_deserialize_packed": ([_P, _vp, _i64, _vp, _vp], ctypes.c_int),
        "phe_server_wire_host": ([_P, _vp, _i64, _i64, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp],
                                 ctypes.c_int),
        "phe_matmul_clear_ct": ([_P, _vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp, _vp, _i64, _i32, _vp, _sz,
                                 _vp, _vp, _vp], ctypes.c_int),
        "phe_ntt_primes": ([_vp], ctypes.c_int),
        "phe_matmul_clear_into": ([_P, _vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp, _i64, _i32, _vp, _vp, _i64,
                                   _vp], ctypes.c_int),
        "phe_matmul_clear_ntt_into": ([_P, _vp, _vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp, _i64, _i32, _vp, _vp,
                                       _i64, _vp], ctypes.c_int),
        "phe_matmul_clear_digits_ntt": ([_P, _vp, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, _vp, _vp, _vp],
                                        ctypes.c_int),
        "phe_wire_lwe_bytes": ([_P, _i64], _sz),
        "phe_wire_serialize_lwe": ([_P, _vp, _vp, _i64, _i64, _vp, _vp], ctypes.c_int),
        "phe_wire_deserialize_lwe": ([_P, _vp, _i64, _i64, _vp, _vp, _vp], ctypes.c_int),
        "phe_server_matvec_wire_host": ([_P, _vp, _i64, _i64, ctypes.c_int, _i64, _i64, _vp, _i64, _i64, _vp, _vp,
                                         _sz, _vp], ctypes.c_int),
        "phe_encrypt_pack_ntt": ([_P, _vp, _vp, _vp, _i64, _i64, _u64, _u64, _vp, _vp, _vp], ctypes.c_int),
        "phe_ntt_max_blocks": ([_P], _i64),
        "phe_ntt_tables_bytes": ([_P], _sz),
        "phe_ntt_tables_init": ([_P, _vp, _sz, _vp], ctypes.c_int),
        "phe_ntt_weights_bytes": ([_P, _i64, _i64], _sz),
        "phe_ntt_weights_prepare": ([_P, _vp, _vp, _i64, _i64, ctypes.c_int, _vp, _sz, _vp], ctypes.c_int),
        "phe_ntt_operand_bytes": ([_P, _i64, _i64], _sz),
        "phe_ntt_ct_prepare": ([_P, _vp, _vp, _vp, _i64, _i64, _vp, _sz, _vp], ctypes.c_int),
        "phe_matmul_clear_ntt": ([_P, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _i32, _vp, _vp, _vp],
                                 ctypes.c_int),
        "phe_matmul_clear_ntt_T": ([_P, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _i32, _vp, _vp, _vp],
                                   ctypes.c_int),
        "phe_ntt_ksk_bytes": ([_P], _sz),
        "phe_ntt_ksk_prepare": ([_P, _vp, _vp, _sz, _vp], ctypes.c_int),
        "phe_pack_ntt_ws_bytes": ([_P, _i64, _i64], _sz),
        "phe_pack_ntt": ([_P, _vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp, _vp], ctypes.c_int),
        "phe_packed_ntt_ws_bytes": ([_P, _i64, _i64], _sz),
        "phe_matmul_clear_packed_ntt": ([_P, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, _vp, _vp, _sz, _vp, _vp],
                                        ctypes.c_int),
        "phe_server_wire_host_ntt": ([_P, _vp, _i64, _i64, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp],
                                     ctypes.c_int),
        "phe_matmul_clear_packed_nttw": ([_P, _vp, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, _vp, _vp, _sz, _vp,
                                          _vp], ctypes.c_int),
        "phe_server_wire_host_nttw": ([_P, _vp, _vp, _i64, _i64, ctypes.c_int, _vp, _vp, _i64, _i64, _vp, _vp,
                                       _sz, _vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(rc: int, what: str) -> None:
    if rc != PHE_OK:
        lib = load()
        msg = lib.phe_strerror(rc).decode()
        if rc == PHE_ECUDA:
            msg += f" (cudaError {lib.phe_last_cuda_error()})"
        raise PheError(f"{what}: {msg} [code {rc}]")


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor, dtype=None, name="tensor"):
    if not t.is_cuda:
        raise PheError(f"{name} must be a CUDA tensor (no CPU path)")
    if dtype is not None and t.dtype != dtype:
        raise PheError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise PheError(f"{name} must be contiguous")
    return t


# ------------------------------------------------------------------ params
def _need(t: torch.Tensor, dtype, shape, name: str) -> torch.Tensor:
    """A caller-supplied device tensor the C ABI reads or writes without a size argument:
    CUDA, `dtype`, contiguous, exactly `shape` (no silent out-of-bounds access)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise PheError(f"{name} must be a contiguous CUDA {dtype} tensor")
    if tuple(t.shape) != tuple(shape):
        raise PheError(f"{name} has shape {tuple(t.shape)}, the call needs {tuple(shape)}")
    return t


def _need_bytes(t: torch.Tensor, nbytes: int, name: str) -> torch.Tensor:
    """A caller-supplied device buffer of at least `nbytes` bytes (operands, workspaces)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous():
        raise PheError(f"{name} must be a contiguous CUDA tensor")
    if t.numel() * t.element_size() < nbytes:
        raise PheError(f"{name} holds {t.numel() * t.element_size()} bytes, the call reads {nbytes}")
    return t


def params(preset: int = PRESET_PAPER, **override) -> Params:
    p = Params()
    _check(load().phe_params_init(ctypes.byref(p), preset), "phe_params_init")
    for k, v in override.items():
        setattr(p, k, v)
    _check(load().phe_params_validate(ctypes.byref(p)), "phe_params_validate")
    return p


def num_limbs(p: Params) -> int:
    return load().phe_num_limbs(ctypes.byref(p))


def num_blocks(p: Params, d: int) -> int:
    return load().phe_num_blocks(ctypes.byref(p), d)


# ------------------------------------------------------------------ client ops
def keygen(p: Params, master_seed: int, device="cuda") -> torch.Tensor:
    S = torch.empty(p.N, dtype=torch.uint8, device=device)
    _check(load().phe_keygen(ctypes.byref(p), master_seed & (2**64 - 1), _ptr(S), _stream()), "phe_keygen")
    return S


def encrypt_pack(p: Params, S: torch.Tensor, x: torch.Tensor, seed_base: int, noise_seed: int = 0):
    """x int8 [T][d_in] -> (seeds int64[T][L] (u64 bits), body int64[T][L][N])."""
    _dev(S, torch.uint8, "S"); _dev(x, torch.int8, "x")
    T, d_in = x.shape
    L = p.L(d_in)
    seeds = torch.empty((T, L), dtype=torch.int64, device=x.device)
    body = torch.empty((T, L, p.N), dtype=torch.int64, device=x.device)
    _check(load().phe_encrypt_pack(ctypes.byref(p), _ptr(S), _ptr(x), T, d_in, seed_base & (2**64 - 1),
                                   noise_seed & (2**64 - 1), _ptr(seeds), _ptr(body), _stream()),
           "phe_encrypt_pack")
    return seeds, body


def decrypt_unpack(p: Params, S: torch.Tensor, mask: torch.Tensor, body: torch.Tensor, q_bits: int):
    """mask [T][rows][N], body [T][rows] (int64 if q_bits == q_in else int32) -> int32 [T][rows]."""
    _dev(S, torch.uint8, "S"); _dev(mask, None, "mask"); _dev(body, None, "body")
    T, rows = body.shape
    y = torch.empty((T, rows), dtype=torch.int32, device=body.device)
    _check(load().phe_decrypt_unpack(ctypes.byref(p), _ptr(S), _ptr(mask), _ptr(body), T, rows, q_bits,
                                     _ptr(y), _stream()), "phe_decrypt_unpack")
    return y


# ------------------------------------------------------------------ server ops
class Weights:
    """A weight matrix registered for the limb GEMM (phe_weights_prepare, P:182 absorbed).
    transpose=True registers M = W^T for the backward matmul_clear_T."""

    def __init__(self, p: Params, W: torch.Tensor, transpose: bool = False):
        _dev(W, torch.int8, "W")
        self.p = p
        self.d_out, self.d_in = W.shape
        self.transpose = bool(transpose)
        self.rows, self.cols = (self.d_in, self.d_out) if transpose else (self.d_out, self.d_in)
        nbytes = load().phe_weights_bytes(ctypes.byref(p), self.rows, self.cols)
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=W.device)
        _check(load().phe_weights_prepare(ctypes.byref(p), _ptr(W), self.d_out, self.d_in, int(transpose),
                                          _ptr(self.buf), nbytes, _stream()), "phe_weights_prepare")


def ct_prepare(p: Params, seeds: torch.Tensor, body: torch.Tensor, out: torch.Tensor | None = None):
    _dev(seeds, torch.int64, "seeds"); _dev(body, torch.int64, "body")
    T, L = seeds.shape
    nbytes = load().phe_ct_operand_bytes(ctypes.byref(p), T, L)
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=seeds.device)
    _check(load().phe_ct_prepare(ctypes.byref(p), _ptr(seeds), _ptr(body), T, L, _ptr(out),
                                 out.numel(), _stream()), "phe_ct_prepare")
    return out


SKIP = "skip"  # pass as out_mask / out_body to skip that contraction (NULL in the C ABI)


def _outputs(p, T, R, out_bits, device, out_mask, out_body):
    dt = torch.int64 if out_bits == p.q_in else torch.int32
    if out_mask is None:
        out_mask = torch.empty((T, R, p.N), dtype=dt, device=device)
    if out_body is None:
        out_body = torch.empty((T, R), dtype=dt, device=device)
    return (None if isinstance(out_mask, str) else out_mask), (None if isinstance(out_body, str) else out_body)


def matmul_clear(p: Params, w: Weights, operand: torch.Tensor, T: int, out_bits: int | None = None,
                 row_begin: int = 0, row_end: int | None = None, out_mask=None, out_body=None):
    """LWE(x_tau . w_j) for j in [row_begin, row_end) (Eq. 6), modulus-switched to
    q_out when out_bits == q_out (default).  Returns (mask [T][R][N], body [T][R])."""
    if w.transpose:
        raise PheError("matmul_clear needs weights registered with transpose=False")
    out_bits = p.q_out if out_bits is None else out_bits
    row_end = w.rows if row_end is None else row_end
    out_mask, out_body = _outputs(p, T, row_end - row_begin, out_bits, operand.device, out_mask, out_body)
    _check(load().phe_matmul_clear(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, row_begin, row_end,
                                   _ptr(operand), T, out_bits, _ptr(out_mask), _ptr(out_body), _stream()),
           "phe_matmul_clear")
    return out_mask, out_body


def matmul_clear_T(p: Params, w: Weights, operand: torch.Tensor, T: int, out_bits: int | None = None,
                   row_begin: int = 0, row_end: int | None = None, out_mask=None, out_body=None):
    """Backward W^T . [g]: rows index d_in."""
    if not w.transpose:
        raise PheError("matmul_clear_T needs weights registered with transpose=True")
    out_bits = p.q_out if out_bits is None else out_bits
    row_end = w.rows if row_end is None else row_end
    out_mask, out_body = _outputs(p, T, row_end - row_begin, out_bits, operand.device, out_mask, out_body)
    _check(load().phe_matmul_clear_T(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, row_begin, row_end,
                                     _ptr(operand), T, out_bits, _ptr(out_mask), _ptr(out_body), _stream()),
           "phe_matmul_clear_T")
    return out_mask, out_body


def matmul_clear_ct(p: Params, w: Weights, seeds: torch.Tensor, body: torch.Tensor, out_bits: int | None = None,
                    row_begin: int = 0, row_end: int | None = None, ws: torch.Tensor | None = None):
    """matmul_clear(W, ct) in one call (phe_matmul_clear_ct): expands the seeded ciphertext into a
    workspace and contracts it; forward or backward by w.transpose."""
    _dev(seeds, torch.int64, "seeds"); _dev(body, torch.int64, "body")
    T, L = seeds.shape
    out_bits = p.q_out if out_bits is None else out_bits
    row_end = w.rows if row_end is None else row_end
    if ws is None:
        ws = torch.empty(load().phe_ct_operand_bytes(ctypes.byref(p), T, L), dtype=torch.uint8, device=seeds.device)
    out_mask, out_body = _outputs(p, T, row_end - row_begin, out_bits, seeds.device, None, None)
    _check(load().phe_matmul_clear_ct(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose), row_begin,
                                      row_end, _ptr(seeds), _ptr(body), T, out_bits, _ptr(ws), ws.numel(),
                                      _ptr(out_mask), _ptr(out_body), _stream()), "phe_matmul_clear_ct")
    return out_mask, out_body


def matmul_clear_simt(p: Params, W: torch.Tensor, operand: torch.Tensor, T: int, out_bits: int | None = None,
                      row_begin: int = 0, row_end: int | None = None):
    """CUDA-core cross-check of matmul_clear (same contract; W raw int8 [rows][cols])."""
    _dev(W, torch.int8, "W")
    out_bits = p.q_out if out_bits is None else out_bits
    row_end = W.shape[0] if row_end is None else row_end
    out_mask, out_body = _outputs(p, T, row_end - row_begin, out_bits, operand.device, None, None)
    _check(load().phe_matmul_clear_simt(ctypes.byref(p), _ptr(W), W.shape[0], W.shape[1], row_begin, row_end,
                                        _ptr(operand), T, out_bits, _ptr(out_mask), _ptr(out_body), _stream()),
           "phe_matmul_clear_simt")
    return out_mask, out_body


def modswitch(x: torch.Tensor, from_bits: int, to_bits: int, out: torch.Tensor | None = None):
    _dev(x, torch.int64, "x")
    if out is None:
        out = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    _check(load().phe_modswitch(_ptr(x), _ptr(out), x.numel(), from_bits, to_bits, _stream()), "phe_modswitch")
    return out


def server_matvec_host(p: Params, w: Weights, h_seeds: torch.Tensor, h_body: torch.Tensor,
                       h_out_mask: torch.Tensor, h_out_body: torch.Tensor, chunk_tokens: int = 256,
                       row_begin: int = 0, row_end: int | None = None) -> None:
    """End-to-end with HOST buffers (pinned CPU tensors): H2D, prepare, GEMM, D2H pipelined.
    The device workspace (two chunk slots, phe_server_matvec_host_ws_bytes) comes from torch's
    allocator on the weights' device; the call is synchronous, so it is free again on return."""
    T = h_seeds.shape[0]
    row_end = w.rows if row_end is None else row_end
    R, L = row_end - row_begin, p.L(w.cols)
    _host(h_seeds, "h_seeds", T * L * 8); _host(h_body, "h_body", T * L * p.N * 8)
    _host(h_out_mask, "h_out_mask", T * R * p.N * 4); _host(h_out_body, "h_out_body", T * R * 4)
    if T == 0 or R == 0:
        return
    ws = _host_ws(load().phe_server_matvec_host_ws_bytes(ctypes.byref(p), w.d_out, w.d_in, int(w.transpose),
                                                         row_begin, row_end, T, chunk_tokens), w.buf.device)
    _check(load().phe_server_matvec_host(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose),
                                         row_begin, row_end, _ptr(h_seeds), _ptr(h_body), T, chunk_tokens,
                                         _ptr(h_out_mask), _ptr(h_out_body), _ptr(ws), ws.numel(), _stream()),
           "phe_server_matvec_host")


def _host(t: torch.Tensor, name: str, nbytes: int) -> None:
    """A host-buffer argument: contiguous CPU memory of exactly `nbytes` bytes."""
    if t.is_cuda or not t.is_contiguous():
        raise PheError(f"{name} must be a contiguous host tensor")
    if t.numel() * t.element_size() != nbytes:
        raise PheError(f"{name} holds {t.numel() * t.element_size()} bytes, the call needs {nbytes}")


def _host_ws(nbytes: int, device) -> torch.Tensor:
    """Device workspace of a host pipeline (its *_ws_bytes query; 0 = arguments it rejects)."""
    if nbytes == 0:
        raise PheError("host pipeline: invalid arguments (workspace query returned 0)")
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def last_launch_count() -> int:
    return load().phe_last_launch_count()


# ------------------------------------------------------------------ NEXT #1: KeySwitch packing
def ksk_gen(p: Params, S: torch.Tensor, ksk_seed: int) -> torch.Tensor:
    """Client: KSK_A, KSK_B as int64 [2][4N][N] (u64 bits), row l*N + i (Eq. 8 matrices)."""
    _dev(S, torch.uint8, "S")
    ksk = torch.empty((2, KS_LEVELS * p.N, p.N), dtype=torch.int64, device=S.device)
    _check(load().phe_ksk_gen(ctypes.byref(p), _ptr(S), ksk_seed & (2**64 - 1), _ptr(ksk), ksk.numel() * 8,
                              _stream()), "phe_ksk_gen")
    return ksk


class KeySwitchKey:
    """Server-side registration of a KSK (limb planes for the packing GEMM)."""

    def __init__(self, p: Params, ksk: torch.Tensor):
        _dev(ksk, torch.int64, "ksk")
        self.p = p
        nbytes = load().phe_ksk_prep_bytes(ctypes.byref(p))
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=ksk.device)
        _check(load().phe_ksk_prepare(ctypes.byref(p), _ptr(ksk), _ptr(self.buf), nbytes, _stream()),
               "phe_ksk_prepare")


_ws_cache = {}


def matmul_clear_packed(p: Params, w: Weights, operand: torch.Tensor, T: int, ksk: KeySwitchKey,
                        out: torch.Tensor | None = None, ws: torch.Tensor | None = None) -> torch.Tensor:
    """RLWE(Wx) (Eq. 7 + Eq. 8): int32 [T][G][2][N] (A', B' at q_out), G = ceil(rows / N)."""
    G = (w.rows + p.N - 1) // p.N
    _need_bytes(operand, load().phe_ct_operand_bytes(ctypes.byref(p), T, p.L(w.cols)), "operand")
    if out is None:
        out = torch.empty((T, G, 2, p.N), dtype=torch.int32, device=operand.device)
    _need(out, torch.int32, (T, G, 2, p.N), "out")
    nbytes = load().phe_packed_ws_bytes(ctypes.byref(p), w.rows, T)
    if ws is None:
        ws = _ws_cache.get(operand.device)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=operand.device)
            _ws_cache[operand.device] = ws
    _check(load().phe_matmul_clear_packed(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose),
                                          _ptr(operand), T, _ptr(ksk.buf), _ptr(ws), ws.numel(), _ptr(out),
                                          _stream()), "phe_matmul_clear_packed")
    return out


def decrypt_packed(p: Params, S: torch.Tensor, packed: torch.Tensor, rows: int, q_bits: int | None = None):
    _dev(S, torch.uint8, "S"); _dev(packed, torch.int32, "packed")
    q_bits = p.q_out if q_bits is None else q_bits
    T = packed.shape[0]
    y = torch.empty((T, rows), dtype=torch.int32, device=packed.device)
    _check(load().phe_decrypt_packed(ctypes.byref(p), _ptr(S), _ptr(packed), T, rows, q_bits, _ptr(y), _stream()),
           "phe_decrypt_packed")
    return y


def matmul_clear_digits(p: Params, w: Weights, operand: torch.Tensor, T: int, digits=None, body=None):
    """Stage 1 of the packed primitive: Eq. 6 with masks as Decomp digits (int8 [T][R256][4][N],
    KS_LEVELS = 4) and bodies uint64 [T][R] (int64 storage)."""
    r256 = (w.rows + 255) // 256 * 256
    _need_bytes(operand, load().phe_ct_operand_bytes(ctypes.byref(p), T, p.L(w.cols)), "operand")
    if digits is None:
        digits = torch.empty((T, r256, KS_LEVELS, p.N), dtype=torch.int8, device=operand.device)
    if body is None:
        body = torch.empty((T, w.rows), dtype=torch.int64, device=operand.device)
    _need(digits, torch.int8, (T, r256, KS_LEVELS, p.N), "digits")
    _need(body, torch.int64, (T, w.rows), "body")
    _check(load().phe_matmul_clear_digits(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose),
                                          _ptr(operand), T, _ptr(digits), _ptr(body), _stream()),
           "phe_matmul_clear_digits")
    return digits, body


def pack(p: Params, digits: torch.Tensor, body: torch.Tensor, ksk: KeySwitchKey, out=None, acc=None):
    """Stage 2: Eq. 8 + Eq. 7 (KeySwitch GEMM, Rotate, sum) + ModulusSwitch."""
    T, rows = body.shape
    G = (rows + p.N - 1) // p.N
    _need(body, torch.int64, (T, rows), "body")
    _need(digits, torch.int8, (T, (rows + 255) // 256 * 256, KS_LEVELS, p.N), "digits")
    if out is None:
        out = torch.empty((T, G, 2, p.N), dtype=torch.int32, device=body.device)
    _need(out, torch.int32, (T, G, 2, p.N), "out")
    nbytes = load().phe_pack_acc_bytes(ctypes.byref(p), rows, T)
    if acc is None:
        acc = torch.empty(nbytes, dtype=torch.uint8, device=body.device)
    _check(load().phe_pack(ctypes.byref(p), _ptr(digits), _ptr(body), T, rows, _ptr(ksk.buf), _ptr(acc),
                           acc.numel(), _ptr(out), _stream()), "phe_pack")
    return out


class NttKeySwitchKey:
    """Server-side registration of a KSK in the NTT domain for stage 2 (phe_ntt_ksk_prepare)."""

    def __init__(self, p: Params, ksk: torch.Tensor):
        _dev(ksk, torch.int64, "ksk")
        self.p = p
        nbytes = load().phe_ntt_ksk_bytes(ctypes.byref(p))
        if nbytes == 0:
            raise PheError("phe_ntt_ksk_bytes: parameters unsupported by the NTT KeySwitch")
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=ksk.device)
        _check(load().phe_ntt_ksk_prepare(ctypes.byref(p), _ptr(ksk), _ptr(self.buf), nbytes, _stream()),
               "phe_ntt_ksk_prepare")


def pack_ntt(p: Params, digits: torch.Tensor, body: torch.Tensor, nksk: NttKeySwitchKey, out=None, ws=None):
    """Stage 2 in the NTT domain: same contract and bit-identical output as pack()."""
    T, rows = body.shape
    G = (rows + p.N - 1) // p.N
    _need(body, torch.int64, (T, rows), "body")
    _need(digits, torch.int8, (T, (rows + 255) // 256 * 256, KS_LEVELS, p.N), "digits")
    if out is None:
        out = torch.empty((T, G, 2, p.N), dtype=torch.int32, device=body.device)
    _need(out, torch.int32, (T, G, 2, p.N), "out")
    nbytes = load().phe_pack_ntt_ws_bytes(ctypes.byref(p), rows, T)
    if ws is None:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=body.device)
    _check(load().phe_pack_ntt(ctypes.byref(p), _ptr(digits), _ptr(body), T, rows, _ptr(nksk.buf), _ptr(ws),
                               ws.numel(), _ptr(out), _stream()), "phe_pack_ntt")
    return out


def server_matvec_packed_host(p: Params, w: Weights, ksk: KeySwitchKey, h_seeds: torch.Tensor,
                              h_body: torch.Tensor, h_out: torch.Tensor, chunk_tokens: int = 256) -> None:
    """End to end with HOST buffers for the packed primitive: h_out int32 [T][G][2][N]."""
    T, L, G = h_seeds.shape[0], p.L(w.cols), (w.rows + p.N - 1) // p.N
    _host(h_seeds, "h_seeds", T * L * 8); _host(h_body, "h_body", T * L * p.N * 8)
    _host(h_out, "h_out", T * G * 2 * p.N * 4)
    if T == 0:
        return
    ws = _host_ws(load().phe_server_matvec_packed_host_ws_bytes(ctypes.byref(p), w.d_out, w.d_in, int(w.transpose),
                                                                T, chunk_tokens), w.buf.device)
    _check(load().phe_server_matvec_packed_host(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose),
                                                _ptr(ksk.buf), _ptr(h_seeds), _ptr(h_body), T,
                                                chunk_tokens, _ptr(h_out), _ptr(ws), ws.numel(), _stream()),
           "phe_server_matvec_packed_host")


# ------------------------------------------------------------------ NEXT #2: wire format
def wire_input_bytes(p: Params) -> int:
    return load().phe_wire_input_bytes(ctypes.byref(p))


def wire_output_bytes(p: Params) -> int:
    return load().phe_wire_output_bytes(ctypes.byref(p))


def wire_serialize_inputs(p: Params, seeds: torch.Tensor, body: torch.Tensor) -> torch.Tensor:
    T, L = seeds.shape
    out = torch.empty((T, L, wire_input_bytes(p)), dtype=torch.uint8, device=seeds.device)
    _check(load().phe_wire_serialize_inputs(ctypes.byref(p), _ptr(seeds), _ptr(body), T, L, _ptr(out), _stream()),
           "phe_wire_serialize_inputs")
    return out


def wire_deserialize_inputs(p: Params, wire: torch.Tensor):
    T, L, _ = wire.shape
    seeds = torch.empty((T, L), dtype=torch.int64, device=wire.device)
    body = torch.empty((T, L, p.N), dtype=torch.int64, device=wire.device)
    _check(load().phe_wire_deserialize_inputs(ctypes.byref(p), _ptr(wire), T, L, _ptr(seeds), _ptr(body),
                                              _stream()), "phe_wire_deserialize_inputs")
    return seeds, body


def wire_serialize_packed(p: Params, packed: torch.Tensor) -> torch.Tensor:
    T, G = packed.shape[:2]
    out = torch.empty((T, G, wire_output_bytes(p)), dtype=torch.uint8, device=packed.device)
    _check(load().phe_wire_serialize_packed(ctypes.byref(p), _ptr(packed), T * G, _ptr(out), _stream()),
           "phe_wire_serialize_packed")
    return out


def wire_deserialize_packed(p: Params, wire: torch.Tensor) -> torch.Tensor:
    T, G = wire.shape[:2]
    out = torch.empty((T, G, 2, p.N), dtype=torch.int32, device=wire.device)
    _check(load().phe_wire_deserialize_packed(ctypes.byref(p), _ptr(wire), T * G, _ptr(out), _stream()),
           "phe_wire_deserialize_packed")
    return out


def server_wire_host(p: Params, w: Weights, ksk: KeySwitchKey, h_wire_in: torch.Tensor, h_wire_out: torch.Tensor,
                     chunk_tokens: int = 255) -> None:
    """The server step on wire bytes (host buffers): [T][L][9992] in -> [T][G][13312] out."""
    _wire_host(p, w, ksk, h_wire_in, h_wire_out, chunk_tokens, "phe_server_wire_host")


def _wire_host(p, w, key, h_wire_in, h_wire_out, chunk_tokens, api):
    T, L, G = h_wire_in.shape[0], p.L(w.cols), (w.rows + p.N - 1) // p.N
    _host(h_wire_in, "h_wire_in", T * L * wire_input_bytes(p))
    _host(h_wire_out, "h_wire_out", T * G * wire_output_bytes(p))
    if T == 0:
        return
    lib = load()
    ws = _host_ws(getattr(lib, api + "_ws_bytes")(ctypes.byref(p), w.d_out, w.d_in, int(w.transpose), T,
                                                  chunk_tokens), w.buf.device)
    head = [ctypes.byref(p)] + ([_ptr(w.tables.buf)] if api.endswith("_nttw") else [])
    _check(getattr(lib, api)(*head, _ptr(w.buf), w.d_out, w.d_in, int(w.transpose), _ptr(key.buf), _ptr(h_wire_in),
                             T, chunk_tokens, _ptr(h_wire_out), _ptr(ws), ws.numel(), _stream()), api)


def matmul_clear_packed_ntt(p: Params, w: Weights, operand: torch.Tensor, T: int, nksk: "NttKeySwitchKey",
                            out: torch.Tensor | None = None, ws: torch.Tensor | None = None) -> torch.Tensor:
    """matmul_clear_packed with stage 2 (Eq. 7/8) in the NTT domain: same output."""
    G = (w.rows + p.N - 1) // p.N
    _need_bytes(operand, load().phe_ct_operand_bytes(ctypes.byref(p), T, p.L(w.cols)), "operand")
    if out is None:
        out = torch.empty((T, G, 2, p.N), dtype=torch.int32, device=operand.device)
    _need(out, torch.int32, (T, G, 2, p.N), "out")
    nbytes = load().phe_packed_ntt_ws_bytes(ctypes.byref(p), w.rows, T)
    if ws is None:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=operand.device)
    _check(load().phe_matmul_clear_packed_ntt(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose),
                                              _ptr(operand), T, _ptr(nksk.buf), _ptr(ws), ws.numel(), _ptr(out),
                                              _stream()), "phe_matmul_clear_packed_ntt")
    return out


def server_wire_host_ntt(p: Params, w: Weights, nksk: "NttKeySwitchKey", h_wire_in: torch.Tensor,
                         h_wire_out: torch.Tensor, chunk_tokens: int = 255) -> None:
    """server_wire_host with the packing stage in the NTT domain (phe_server_wire_host_ntt)."""
    _wire_host(p, w, nksk, h_wire_in, h_wire_out, chunk_tokens, "phe_server_wire_host_ntt")


def matmul_clear_packed_nttw(p: Params, w: "NttWeights", operand: torch.Tensor, T: int, nksk: "NttKeySwitchKey",
                             out: torch.Tensor | None = None, ws: torch.Tensor | None = None) -> torch.Tensor:
    """matmul_clear_packed with both stages in the NTT domain (operand from ntt_ct_prepare): same
    output (phe_matmul_clear_packed_nttw)."""
    G = (w.rows + p.N - 1) // p.N
    _need_bytes(operand, load().phe_ntt_operand_bytes(ctypes.byref(p), T, p.L(w.cols)), "operand")
    if out is None:
        out = torch.empty((T, G, 2, p.N), dtype=torch.int32, device=operand.device)
    _need(out, torch.int32, (T, G, 2, p.N), "out")
    nbytes = load().phe_packed_ntt_ws_bytes(ctypes.byref(p), w.rows, T)
    if ws is None:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=operand.device)
    _check(load().phe_matmul_clear_packed_nttw(ctypes.byref(p), _ptr(w.tables.buf), _ptr(w.buf), w.d_out, w.d_in,
                                               int(w.transpose), _ptr(operand), T, _ptr(nksk.buf), _ptr(ws),
                                               ws.numel(), _ptr(out), _stream()), "phe_matmul_clear_packed_nttw")
    return out


def server_wire_host_nttw(p: Params, w: "NttWeights", nksk: "NttKeySwitchKey", h_wire_in: torch.Tensor,
                          h_wire_out: torch.Tensor, chunk_tokens: int = 255) -> None:
    """server_wire_host with both stages in the NTT domain (phe_server_wire_host_nttw)."""
    _wire_host(p, w, nksk, h_wire_in, h_wire_out, chunk_tokens, "phe_server_wire_host_nttw")


# ------------------------------------------------------------------ NEXT #4: NTT-domain contraction
def ntt_primes() -> tuple[int, int]:
    """The two NTT primes (p0, p1) of the NTT path (host query, no GPU needed)."""
    out = (ctypes.c_uint32 * 2)()
    _check(load().phe_ntt_primes(ctypes.cast(out, ctypes.c_void_p)), "phe_ntt_primes")
    return int(out[0]), int(out[1])


def ntt_max_blocks(p: Params) -> int:
    """Largest L = ceil(cols/N) for which the two-prime CRT recovers Eq. 6's integers exactly."""
    return int(load().phe_ntt_max_blocks(ctypes.byref(p)))


class NttTables:
    """Twiddle tables for params p (phe_ntt_tables_init); shared by every NTT-path call."""

    def __init__(self, p: Params, device="cuda"):
        self.p = p
        nbytes = load().phe_ntt_tables_bytes(ctypes.byref(p))
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _check(load().phe_ntt_tables_init(ctypes.byref(p), _ptr(self.buf), nbytes, _stream()),
               "phe_ntt_tables_init")


class NttWeights:
    """W (or W^T) registered in the NTT domain (phe_ntt_weights_prepare)."""

    def __init__(self, p: Params, tables: NttTables, W: torch.Tensor, transpose: bool = False):
        _dev(W, torch.int8, "W")
        self.p, self.tables = p, tables
        self.d_out, self.d_in = W.shape
        self.transpose = bool(transpose)
        self.rows, self.cols = (self.d_in, self.d_out) if transpose else (self.d_out, self.d_in)
        nbytes = load().phe_ntt_weights_bytes(ctypes.byref(p), self.rows, self.cols)
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=W.device)
        _check(load().phe_ntt_weights_prepare(ctypes.byref(p), _ptr(tables.buf), _ptr(W), self.d_out, self.d_in,
                                              int(transpose), _ptr(self.buf), nbytes, _stream()),
               "phe_ntt_weights_prepare")


def ntt_ct_prepare(p: Params, tables: NttTables, seeds: torch.Tensor, body: torch.Tensor,
                   out: torch.Tensor | None = None):
    """Forward NTTs of the expanded masks + body limb planes (phe_ntt_ct_prepare)."""
    _dev(seeds, torch.int64, "seeds"); _dev(body, torch.int64, "body")
    T, L = seeds.shape
    nbytes = load().phe_ntt_operand_bytes(ctypes.byref(p), T, L)
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=seeds.device)
    _check(load().phe_ntt_ct_prepare(ctypes.byref(p), _ptr(tables.buf), _ptr(seeds), _ptr(body), T, L,
                                     _ptr(out), out.numel(), _stream()), "phe_ntt_ct_prepare")
    return out


def matmul_clear_ntt(p: Params, w: NttWeights, operand: torch.Tensor, T: int, out_bits: int | None = None,
                     row_begin: int = 0, row_end: int | None = None, out_mask=None, out_body=None):
    """Same contract and bit-identical result as matmul_clear / matmul_clear_T (by w.transpose),
    mask contraction in the NTT domain (NEXT #4)."""
    out_bits = p.q_out if out_bits is None else out_bits
    row_end = w.rows if row_end is None else row_end
    out_mask, out_body = _outputs(p, T, row_end - row_begin, out_bits, operand.device, out_mask, out_body)
    fn = load().phe_matmul_clear_ntt_T if w.transpose else load().phe_matmul_clear_ntt
    _check(fn(ctypes.byref(p), _ptr(w.tables.buf), _ptr(w.buf), w.d_out, w.d_in, row_begin, row_end,
              _ptr(operand), T, out_bits, _ptr(out_mask), _ptr(out_body), _stream()), "phe_matmul_clear_ntt")
    return out_mask, out_body


def encrypt_pack_ntt(p: Params, tables: NttTables, S: torch.Tensor, x: torch.Tensor, seed_base: int,
                     noise_seed: int = 0):
    """encrypt_pack with A*S through the NTT (phe_encrypt_pack_ntt); bit-identical output."""
    _dev(S, torch.uint8, "S"); _dev(x, torch.int8, "x")
    T, d_in = x.shape
    L = p.L(d_in)
    seeds = torch.empty((T, L), dtype=torch.int64, device=x.device)
    body = torch.empty((T, L, p.N), dtype=torch.int64, device=x.device)
    _check(load().phe_encrypt_pack_ntt(ctypes.byref(p), _ptr(tables.buf), _ptr(S), _ptr(x), T, d_in,
                                       seed_base & (2**64 - 1), noise_seed & (2**64 - 1), _ptr(seeds), _ptr(body),
                                       _stream()), "phe_encrypt_pack_ntt")
    return seeds, body


# ------------------------------------------------------------------ LWE outputs on the wire
def wire_lwe_bytes(p: Params, R: int) -> int:
    return int(load().phe_wire_lwe_bytes(ctypes.byref(p), R))


def wire_serialize_lwe(p: Params, mask: torch.Tensor, body: torch.Tensor, out: torch.Tensor | None = None
                       ) -> torch.Tensor:
    """uint32 LWE outputs [T][R][N], [T][R] -> bytes [T][wire_lwe_bytes(p, R)] at q_out bits
    (`out`: a contiguous uint8 CUDA tensor of exactly that shape, 8-byte aligned)."""
    _dev(mask, torch.int32, "mask"); _dev(body, torch.int32, "body")
    T, R = body.shape
    if tuple(mask.shape) != (T, R, p.N):
        raise PheError("mask must be [T][R][N] matching body [T][R]")
    nb = wire_lwe_bytes(p, R)
    if out is None:
        out = torch.empty((T, nb), dtype=torch.uint8, device=mask.device)
    elif (not out.is_cuda or out.dtype != torch.uint8 or not out.is_contiguous() or tuple(out.shape) != (T, nb)
          or out.data_ptr() % 8):
        raise PheError(f"out must be a contiguous, 8-byte aligned uint8 CUDA tensor of shape {(T, nb)}")
    _check(load().phe_wire_serialize_lwe(ctypes.byref(p), _ptr(mask), _ptr(body), T, R, _ptr(out), _stream()),
           "phe_wire_serialize_lwe")
    return out


def wire_lwe_direct_supported(p: Params, R: int) -> bool:
    return bool(load().phe_wire_lwe_direct_supported(ctypes.byref(p), R))


def matmul_clear_wire(p: Params, w, operand: torch.Tensor, T: int, row_begin: int = 0, row_end: int | None = None,
                      out: torch.Tensor | None = None, ws: torch.Tensor | None = None) -> torch.Tensor:
    """matmul_clear / matmul_clear_T (by w.transpose) writing the switched LWE outputs straight into
    wire records uint8 [T][wire_lwe_bytes(p, R)] (the mask epilogue bit-packs at q_out;
    phe_matmul_clear_wire).  Byte-identical to wire_serialize_lwe(matmul_clear(...))."""
    row_end = w.rows if row_end is None else row_end
    R = row_end - row_begin
    _need_bytes(operand, load().phe_ct_operand_bytes(ctypes.byref(p), T, p.L(w.cols)), "operand")
    nb = wire_lwe_bytes(p, R) if R > 0 else 0
    if out is None:
        out = torch.empty((T, nb), dtype=torch.uint8, device=operand.device)
    _need(out, torch.uint8, (T, nb), "out")
    need = load().phe_matmul_clear_wire_ws_bytes(ctypes.byref(p), T, max(R, 1))
    if ws is None:
        ws = torch.empty(need, dtype=torch.uint8, device=operand.device)
    _need_bytes(ws, need, "ws")
    _check(load().phe_matmul_clear_wire(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose), row_begin,
                                        row_end, _ptr(operand), T, _ptr(out), _ptr(ws), ws.numel(), _stream()),
           "phe_matmul_clear_wire")
    return out


def wire_deserialize_lwe(p: Params, wire: torch.Tensor, R: int):
    _dev(wire, torch.uint8, "wire")
    T = wire.shape[0]
    mask = torch.empty((T, R, p.N), dtype=torch.int32, device=wire.device)
    body = torch.empty((T, R), dtype=torch.int32, device=wire.device)
    _check(load().phe_wire_deserialize_lwe(ctypes.byref(p), _ptr(wire), T, R, _ptr(mask), _ptr(body), _stream()),
           "phe_wire_deserialize_lwe")
    return mask, body


def server_matvec_wire_host(p: Params, w: Weights, h_wire_in: torch.Tensor, h_wire_out: torch.Tensor,
                            chunk_tokens: int = 256, row_begin: int = 0, row_end: int | None = None) -> None:
    """End to end on wire bytes with HOST buffers: input blocks [T][L][9992] -> switched LWE outputs
    at q_out bits [T][wire_lwe_bytes(p, R)] (phe_server_matvec_wire_host)."""
    T = h_wire_in.shape[0]
    row_end = w.rows if row_end is None else row_end
    R, L = row_end - row_begin, p.L(w.cols)
    _host(h_wire_in, "h_wire_in", T * L * wire_input_bytes(p))
    _host(h_wire_out, "h_wire_out", T * (wire_lwe_bytes(p, R) if R > 0 else 0))
    if T == 0 or R == 0:
        return
    ws = _host_ws(load().phe_server_matvec_wire_host_ws_bytes(ctypes.byref(p), w.d_out, w.d_in, int(w.transpose),
                                                              row_begin, row_end, T, chunk_tokens), w.buf.device)
    _check(load().phe_server_matvec_wire_host(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose),
                                              row_begin, row_end, _ptr(h_wire_in), T, chunk_tokens,
                                              _ptr(h_wire_out), _ptr(ws), ws.numel(), _stream()),
           "phe_server_matvec_wire_host")


def matmul_clear_digits_ntt(p: Params, w: "NttWeights", operand: torch.Tensor, T: int, digits=None, body=None):
    """matmul_clear_digits through the NTT-domain contraction (bit-identical); feeds phe.pack."""
    r256 = (w.rows + 255) // 256 * 256
    _need_bytes(operand, load().phe_ntt_operand_bytes(ctypes.byref(p), T, p.L(w.cols)), "operand")
    if digits is None:
        digits = torch.empty((T, r256, KS_LEVELS, p.N), dtype=torch.int8, device=operand.device)
    if body is None:
        body = torch.empty((T, w.rows), dtype=torch.int64, device=operand.device)
    _need(digits, torch.int8, (T, r256, KS_LEVELS, p.N), "digits")
    _need(body, torch.int64, (T, w.rows), "body")
    _check(load().phe_matmul_clear_digits_ntt(ctypes.byref(p), _ptr(w.tables.buf), _ptr(w.buf), w.d_out, w.d_in,
                                              int(w.transpose), _ptr(operand), T, _ptr(digits), _ptr(body),
                                              _stream()), "phe_matmul_clear_digits_ntt")
    return digits, body


def matmul_clear_into(p: Params, w, operand: torch.Tensor, T: int, mask_block: torch.Tensor,
                      body_block: torch.Tensor, row_begin: int, row_end: int, out_bits: int | None = None) -> None:
    """matmul_clear / matmul_clear_T (by w.transpose; Weights or NttWeights) writing rows
    [row_begin, row_end) into row-block views of larger [T][R_total][N] / [T][R_total] tensors --
    also peer-mapped ones (dist.PeerGather): the fused gather (phe_matmul_clear_into)."""
    out_bits = p.q_out if out_bits is None else out_bits
    R = row_end - row_begin
    dt = torch.int64 if out_bits == p.q_in else torch.int32
    for t, n in [(mask_block, "mask_block"), (body_block, "body_block")]:
        if not t.is_cuda or t.dtype != dt:
            raise PheError(f"{n} must be a CUDA {dt} tensor")
    if (tuple(mask_block.shape) != (T, R, p.N) or mask_block.stride(2) != 1 or mask_block.stride(1) != p.N
            or tuple(body_block.shape) != (T, R) or body_block.stride(1) != 1
            or mask_block.stride(0) != body_block.stride(0) * p.N):
        raise PheError("mask_block/body_block must be row blocks [T][R][N] / [T][R] of [T][R_total][N] / [T][R_total]")
    out_rows = body_block.stride(0)
    if isinstance(w, NttWeights):
        _check(load().phe_matmul_clear_ntt_into(ctypes.byref(p), _ptr(w.tables.buf), _ptr(w.buf), w.d_out, w.d_in,
                                                int(w.transpose), row_begin, row_end, _ptr(operand), T, out_bits,
                                                _ptr(mask_block), _ptr(body_block), out_rows, _stream()),
               "phe_matmul_clear_ntt_into")
    else:
        _check(load().phe_matmul_clear_into(ctypes.byref(p), _ptr(w.buf), w.d_out, w.d_in, int(w.transpose),
                                            row_begin, row_end, _ptr(operand), T, out_bits, _ptr(mask_block),
                                            _ptr(body_block), out_rows, _stream()), "phe_matmul_clear_into")

