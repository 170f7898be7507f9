"""Test helper: Freivalds projections of CUDA-path LWE masks (test arithmetic on the outputs under
test; the expected values come from oracle.mask_projection / oracle.body_projection)."""
import numpy as np
import torch

NR = 4  # independent random vectors per (tau, j)


def r_limbs(r: np.ndarray, device) -> torch.Tensor:
    """r [NR][N] residues < 2^39 -> int64 [NR][3][N] 13-bit limbs."""
    return torch.stack([torch.from_numpy(((r >> np.uint64(13 * l)) & np.uint64(8191)).astype(np.int64))
                        for l in range(3)], 1).to(device)


def projections(m39, r_limbs):
    """sum_t a[tau, j, t] r_e[t] mod 2^64 for each e, exactly: r = r0 + 2^13 r1 + 2^26 r2 with
    13-bit limbs, so each int64 partial sum (< 2^39 * 2^13 * N <= 2^63) cannot overflow.
    Returns uint64 [T][R][NR]."""
    T, R, N = m39.shape
    out = np.zeros((T, R, NR), np.uint64)
    step = max(1, (1 << 28) // (R * N))
    for t0 in range(0, T, step):
        blk = m39[t0:t0 + step]
        acc = np.zeros((blk.shape[0], R, NR), np.uint64)
        for e in range(NR):
            for l in range(3):
                s = (blk * r_limbs[e, l]).sum(-1)                 # int64 [t][R], exact
                with np.errstate(over="ignore"):
                    acc[:, :, e] += s.cpu().numpy().view(np.uint64) << np.uint64(13 * l)
        out[t0:t0 + step] = acc
    return out
