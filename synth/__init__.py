"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no ChaCha20, no encryption, no
negacyclic products, no modulus switching).  It only draws the *cleartext* inputs the
paper's workloads have: quantized int8 weights W and int8 activations x / gradients g,
plus the public integers (seed bases, master seeds) both sides are fed.  Everything the
method itself draws (masks from seeds, the secret key, the noise) is derived from these
integers independently by each side (oracle/ and the CUDA library) with its own
ChaCha20 (reading R6).

Distributions:
  * W: Llama-like N(0, 0.02^2) floats, symmetric per-output-channel int8 in [-127, 127]
    ("SC"; symmetric => zero-point 0).
  * x: per-token dynamic symmetric int8 ("DTok") of N(0,1) rows
    with 1% outlier channels scaled x20.
  * g: per-token dynamic symmetric int8 of Laplace rows (gradients).
"""
from __future__ import annotations

import numpy as np

MASTER_SEED = 250507329


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _sym_quant_rows(f: np.ndarray) -> np.ndarray:
    """Symmetric int8 quantization with one scale per row (zero-point 0)."""
    amax = np.abs(f).max(axis=1, keepdims=True)
    amax[amax == 0] = 1.0
    q = np.rint(f / amax * 127.0)
    return np.clip(q, -127, 127).astype(np.int8)


def weights_int8(d_out: int, d_in: int, seed: int = MASTER_SEED) -> np.ndarray:
    """int8 W [d_out][d_in] (nn.Linear layout), per-output-channel symmetric."""
    f = _rng(seed ^ 0x5757).normal(0.0, 0.02, size=(d_out, d_in)).astype(np.float32)
    return _sym_quant_rows(f)


def activations_int8(T: int, d_in: int, seed: int = MASTER_SEED + 1,
                     outlier_frac: float = 0.01, outlier_scale: float = 20.0) -> np.ndarray:
    """int8 x [T][d_in], per-token dynamic symmetric, with outlier channels."""
    r = _rng(seed ^ 0xA11C)
    f = r.normal(0.0, 1.0, size=(T, d_in)).astype(np.float32)
    n_out = max(1, int(round(outlier_frac * d_in))) if d_in > 0 else 0
    if n_out and T:
        ch = r.choice(d_in, size=n_out, replace=False)
        f[:, ch] *= outlier_scale
    return _sym_quant_rows(f) if T else np.zeros((0, d_in), np.int8)


def gradients_int8(T: int, d: int, seed: int = MASTER_SEED + 2) -> np.ndarray:
    """int8 g [T][d], per-token dynamic symmetric of Laplace rows."""
    f = _rng(seed ^ 0x9AD).laplace(0.0, 1.0, size=(T, d)).astype(np.float32)
    return _sym_quant_rows(f) if T else np.zeros((0, d), np.int8)


def uniform_int8(shape, seed: int, lo: int = -127, hi: int = 127) -> np.ndarray:
    """Uniform int8 in [lo, hi] (for edge-case and extreme-value tests)."""
    return _rng(seed).integers(lo, hi + 1, size=shape, dtype=np.int64).astype(np.int8)


def uniform_u64(shape, seed: int, bits: int) -> np.ndarray:
    """Uniform integers in [0, 2^bits) as uint64 (raw ciphertext words for tests)."""
    r = _rng(seed)
    hi = r.integers(0, 1 << 32, size=shape, dtype=np.uint64)
    lo = r.integers(0, 1 << 32, size=shape, dtype=np.uint64)
    v = (hi << np.uint64(32)) | lo
    if bits < 64:
        v &= np.uint64((1 << bits) - 1)
    return v


def seed_base(tag: int = 0) -> int:
    """Public per-call seed base (an integer; the expansion is each side's own)."""
    return (MASTER_SEED * 1000003 + tag * 7919) & ((1 << 63) - 1)


def weights_int8_torch(d_out: int, d_in: int, seed: int = MASTER_SEED, device="cuda"):
    """Same recipe as weights_int8 (N(0, 0.02^2), per-row symmetric int8), drawn with torch on
    `device` so the 16-layer stack (973M weights) is generated in seconds.  Not bitwise equal
    to weights_int8 (different RNG); used only where no oracle comparison is made."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed ^ 0x5757)
    f = torch.randn((d_out, d_in), generator=g, device=device, dtype=torch.float32) * 0.02
    amax = f.abs().amax(dim=1, keepdim=True).clamp_min(1e-30)
    return torch.clamp(torch.round(f / amax * 127.0), -127, 127).to(torch.int8)
