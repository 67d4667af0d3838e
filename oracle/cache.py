"""Chunkwise NVFP4 KV cache driven step by step, float64 (TEST INFRASTRUCTURE).

PAPER.md:134-139 (§3.2): each layer's cached KV chunk c, K_{l,c}, V_{l,c} in
R^{T_c x H x d}, is quantized independently as (T_c H) x d with NVFP4.
PAPER.md:246-249 (§4.2): attention at chunk step t reads K_eff(t).
Reading Z9: the current chunk is appended first and attended in
quantized form; re-appending the newest chunk overwrites it (denoising step).

The oracle keeps every chunk (it has no memory budget); which chunks the
device cache may evict is a property of the device path, tested there.
"""
from __future__ import annotations

import numpy as np

from . import nvfp4
from .attention import attention
from .keyset import key_token_ranges


class OracleKVCache:
    """``scale_search`` = Four-Over-Six block scales for K and V;
    ``k_smoothing`` = keys mean-centred per (t, h) row, mean restored on dequantization
    (readings Z20-Z22)."""

    def __init__(self, num_layers, num_heads, head_dim, tokens_per_frame, frames_per_chunk,
                 scale_search=False, k_smoothing=False):
        self.scale_search, self.k_smoothing = bool(scale_search), bool(k_smoothing)
        self.L, self.H, self.d = num_layers, num_heads, head_dim
        self.tpf, self.fc = tokens_per_frame, frames_per_chunk
        self.Tc = tokens_per_frame * frames_per_chunk
        self.chunks = [dict() for _ in range(num_layers)]   # layer -> {chunk: (qK, qV)}

    def append(self, layer, chunk_index, K, V):
        """kv_quantize_append: quantize K and V of one chunk."""
        self.chunks[layer][int(chunk_index)] = (
            nvfp4.quantize_kv_chunk(K, self.scale_search, smooth=self.k_smoothing),
            nvfp4.quantize_kv_chunk(V, self.scale_search))

    def export(self, layer, chunk_index):
        qk, qv = self.chunks[layer][int(chunk_index)]
        return qk, qv

    def dequantized_chunk(self, layer, chunk_index):
        qk, qv = self.chunks[layer][int(chunk_index)]
        return (nvfp4.dequantize_kv_chunk(qk, self.Tc, self.H, self.d),
                nvfp4.dequantize_kv_chunk(qv, self.Tc, self.H, self.d))

    def keys(self, layer, chunk_index, sink_frames, window_frames, shot_start=0, shot_len=0):
        """Dequantized K^, V^ over K_eff(t) in ascending logical token order, [Nk, H, d]."""
        ranges = key_token_ranges(chunk_index, self.fc, self.tpf, sink_frames, window_frames,
                                  shot_start, shot_len)
        Ks, Vs, deq = [], [], {}
        for a, b in ranges:
            tok = a
            while tok < b:
                c = tok // self.Tc
                end = min(b, (c + 1) * self.Tc)
                if c not in deq:
                    deq[c] = self.dequantized_chunk(layer, c)
                Kc, Vc = deq[c]
                Ks.append(Kc[tok - c * self.Tc:end - c * self.Tc])
                Vs.append(Vc[tok - c * self.Tc:end - c * self.Tc])
                tok = end
        return np.concatenate(Ks), np.concatenate(Vs)

    def attend(self, layer, chunk_index, Q, sink_frames, window_frames, shot_start=0, shot_len=0,
               softmax_scale=None, rows=None, q_nvfp4=False):
        """chunk_attention: softmax(Q K^T/sqrt(d)) V over K_eff(t).
        q_nvfp4: the queries are NVFP4-quantized first, as one (T_c H) x d tensor with the plain
        encoding ("cast the runtime Q to NVFP4" before the all-to-all; reading Z24),
        and attention uses the exact dequantized Q^ = dec(c) dec(s) g_Q."""
        K, V = self.keys(layer, chunk_index, sink_frames, window_frames, shot_start, shot_len)
        if q_nvfp4:
            Q = np.asarray(Q, dtype=np.float64)
            T, H, d = Q.shape
            Q = nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(Q), T, H, d)
        return attention(Q, K, V, softmax_scale, rows)
