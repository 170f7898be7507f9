"""ctypes loader for the C oracle (oracle/phe_oracle.c).  TEST INFRASTRUCTURE ONLY.

`build()` compiles it with plain gcc (-O2 -fopenmp); `load()` builds on demand.  The
library is the same literal Eq. 6 path as phe_oracle.py (see that file's header).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "phe_oracle.c")
LIB = os.path.join(_HERE, "_build", "libphe_oracle.so")

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i8p = ctypes.POINTER(ctypes.c_int8)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", LIB, SRC])
    return LIB


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class COracle:
    def __init__(self, path: str):
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.oracle_chacha20_block.argtypes = [_u8p, ctypes.c_uint32, _u8p, _u8p]
        L.oracle_expand_mask.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _u64p]
        L.oracle_matmul_clear_literal.argtypes = [
            ctypes.c_int, ctypes.c_int, _i8p, ctypes.c_int64, ctypes.c_int64, _u64p, _u64p,
            _u64p, _u64p, ctypes.c_int]
        L.oracle_matmul_clear_literal.restype = ctypes.c_int
        L.oracle_mask_entries.argtypes = [ctypes.c_int, ctypes.c_int, _i8p, ctypes.c_int64,
                                          _u64p, _i64p, _i64p, ctypes.c_int64, _u64p]
        L.oracle_modswitch.argtypes = [_u64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _u64p]
        L.oracle_mask_projection.argtypes = [ctypes.c_int, ctypes.c_int, _i8p, ctypes.c_int64, ctypes.c_int64,
                                             _u64p, ctypes.c_int64, _u64p, ctypes.c_int, _u64p, ctypes.c_int]
        L.oracle_ksk_gen.argtypes = [ctypes.c_int, ctypes.c_int, _u8p, ctypes.c_uint64, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, _u64p, _u64p, ctypes.c_int]
        L.oracle_decompose.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int32)]
        L.oracle_pack.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, _u64p, ctypes.c_int64, _u64p, _u64p,
                                  ctypes.c_int, ctypes.c_int, _u64p, _u64p, ctypes.c_int]

    def chacha20_block(self, key: bytes, counter: int, nonce: bytes) -> bytes:
        k = np.frombuffer(key, np.uint8).copy()
        n = np.frombuffer(nonce, np.uint8).copy()
        out = np.zeros(64, np.uint8)
        self.lib.oracle_chacha20_block(_p(k, _u8p), counter, _p(n, _u8p), _p(out, _u8p))
        return out.tobytes()

    def expand_mask(self, seed: int, N: int, q_in: int) -> np.ndarray:
        A = np.zeros(N, np.uint64)
        self.lib.oracle_expand_mask(seed, N, q_in, _p(A, _u64p))
        return A

    def matmul_clear_literal(self, params, W: np.ndarray, A: np.ndarray, B: np.ndarray,
                             nthreads: int = 1):
        W = np.ascontiguousarray(W, dtype=np.int8)
        A = np.ascontiguousarray(A, dtype=np.uint64)
        B = np.ascontiguousarray(B, dtype=np.uint64)
        d_out, d_in = W.shape
        mask = np.zeros((d_out, params.N), np.uint64)
        body = np.zeros(d_out, np.uint64)
        self.lib.oracle_matmul_clear_literal(params.N, params.q_in, _p(W, _i8p), d_out, d_in,
                                             _p(A, _u64p), _p(B, _u64p), _p(mask, _u64p),
                                             _p(body, _u64p), nthreads)
        return mask, body

    def mask_entries(self, params, W: np.ndarray, A: np.ndarray, js, ts) -> np.ndarray:
        W = np.ascontiguousarray(W, dtype=np.int8)
        A = np.ascontiguousarray(A, dtype=np.uint64)
        js = np.ascontiguousarray(js, dtype=np.int64)
        ts = np.ascontiguousarray(ts, dtype=np.int64)
        out = np.zeros(len(js), np.uint64)
        self.lib.oracle_mask_entries(params.N, params.q_in, _p(W, _i8p), W.shape[1],
                                     _p(A, _u64p), _p(js, _i64p), _p(ts, _i64p), len(js),
                                     _p(out, _u64p))
        return out

    def mask_projection(self, params, W: np.ndarray, A: np.ndarray, r: np.ndarray, nthreads: int = 1):
        """Freivalds projections sum_t a_{tau,j}[t] r_e[t] mod 2^q_in of Eq. 6's masks for matrix W,
        masks A [T][L][N], vectors r [nr][N]: returns [T][d_out][nr] (see phe_oracle.c)."""
        W = np.ascontiguousarray(W, dtype=np.int8)
        A = np.ascontiguousarray(A, dtype=np.uint64)
        r = np.ascontiguousarray(r, dtype=np.uint64)
        d_out, d_in = W.shape
        T = A.shape[0]
        assert A.shape == (T, params.L(d_in), params.N) and r.shape[1] == params.N
        out = np.zeros((T, d_out, r.shape[0]), np.uint64)
        self.lib.oracle_mask_projection(params.N, params.q_in, _p(W, _i8p), d_out, d_in, _p(A, _u64p), T,
                                        _p(r, _u64p), r.shape[0], _p(out, _u64p), nthreads)
        return out

    def modswitch(self, v: np.ndarray, q_from: int, q_to: int) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.uint64)
        out = np.zeros_like(v)
        self.lib.oracle_modswitch(_p(v, _u64p), v.size, q_from, q_to, _p(out, _u64p))
        return out


    def ksk_gen(self, params, S, ksk_seed: int, eta: int = 0, base_log: int = 8, levels: int = 4,
                nthreads: int = 1):
        N = params.N
        S = np.ascontiguousarray(S, dtype=np.uint8)
        KA = np.zeros((levels * N, N), np.uint64)
        KB = np.zeros((levels * N, N), np.uint64)
        self.lib.oracle_ksk_gen(N, params.q_in, _p(S, _u8p), ksk_seed, eta, base_log, levels,
                                _p(KA, _u64p), _p(KB, _u64p), nthreads)
        return KA, KB

    def pack(self, params, A_lwe, b_lwe, KA, KB, base_log: int = 8, levels: int = 4, nthreads: int = 1):
        N = params.N
        A_lwe = np.ascontiguousarray(A_lwe, dtype=np.uint64)
        b_lwe = np.ascontiguousarray(b_lwe, dtype=np.uint64)
        d_out = A_lwe.shape[0]
        G = (d_out + N - 1) // N
        PA = np.zeros((G, N), np.uint64)
        PB = np.zeros((G, N), np.uint64)
        self.lib.oracle_pack(N, params.q_in, _p(A_lwe, _u64p), _p(b_lwe, _u64p), d_out,
                             _p(np.ascontiguousarray(KA), _u64p), _p(np.ascontiguousarray(KB), _u64p),
                             base_log, levels, _p(PA, _u64p), _p(PB, _u64p), nthreads)
        return PA, PB


_cached = None


def load() -> COracle:
    global _cached
    if _cached is None:
        _cached = COracle(build())
    return _cached
