"""Chunk attention over the dequantized cache, float64 (TEST INFRASTRUCTURE).

For query token i of the current chunk and head h (
softmax form standard, reading Z13: scale 1/sqrt(d), no bias or dropout,
Q and K arrive post-RoPE):

    sigma_ij = (sum_u Q[i,h,u] * K^[j,h,u]) * scale,        j in K_eff(t)
    O[i,h,:] = sum_j exp(sigma_ij - m_i) V^[j,h,:] / sum_j exp(sigma_ij - m_i)

with m_i = max_j sigma_ij.  Q is the exact input value widened to float64 and
K^, V^ are the exact dequantized values (Eq. 2).  A matmul is the
only library primitive used (allowed as a step); nothing is blocked, fused or
reordered beyond the definition.
"""
from __future__ import annotations

import numpy as np


def attention(Q, K, V, softmax_scale=None, rows=None):
    """O = softmax(Q K^T * scale) V per head, float64.

    Q: [Tq, H, d]; K, V: [Nk, H, d]; rows: optional query-row indices to
    evaluate (sampled parity at full size).  Returns [len(rows) or Tq, H, d].
    """
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    if rows is not None:
        Q = Q[np.asarray(rows)]
    Tq, H, d = Q.shape
    scale = 1.0 / np.sqrt(d) if softmax_scale is None or softmax_scale <= 0 else float(softmax_scale)
    O = np.empty((Tq, H, d), dtype=np.float64)
    for h in range(H):
        S = (Q[:, h, :] @ K[:, h, :].T) * scale          # [Tq, Nk]
        m = S.max(axis=1, keepdims=True)
        P = np.exp(S - m)
        O[:, h, :] = (P @ V[:, h, :]) / P.sum(axis=1, keepdims=True)
    return O


def softmax_rows(Q, K, softmax_scale=None):
    """The probability rows themselves (for the rows-sum-to-1 pin), [H, Tq, Nk]."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    Tq, H, d = Q.shape
    scale = 1.0 / np.sqrt(d) if softmax_scale is None or softmax_scale <= 0 else float(softmax_scale)
    out = []
    for h in range(H):
        S = (Q[:, h, :] @ K[:, h, :].T) * scale
        P = np.exp(S - S.max(axis=1, keepdims=True))
        out.append(P / P.sum(axis=1, keepdims=True))
    return np.stack(out)
