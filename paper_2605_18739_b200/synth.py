"""Seeded synthetic inputs shared by the tests, the bench and smoke().

This module holds NO arithmetic of the method (no quantization, no attention):
it only draws reproducible Q/K/V tensors shaped like the paper's workloads
(DESIGN.md §4 "input recipe").  Both the CUDA path and the float64 oracle
consume exactly the bytes produced here.

Recipe: SplitMix64 counter stream -> Box-Muller in float64 -> N(0, 1) ->
variant transform in float64 -> round-to-nearest-even to the input dtype
(bf16 for the Wan-shaped configs, fp32 for ``tiny``).  Per-tensor seed =
0x4C4C32 ^ (layer << 40 | chunk << 8 | tensor_id), tensor_id 0/1/2 = Q/K/V.

Variants (the paper prints no activation statistics):
  iid     -- N(0, 1) for Q, K, V
  peaked  -- Q * 3 (score std ~3)
  outlier -- K + per-channel offsets of +-8 on 4 of the d channels
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """n outputs of SplitMix64 started at ``seed`` (uint64, wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (np.arange(1, n + 1, dtype=np.uint64)
                                                    * np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def normal(seed: int, n: int) -> np.ndarray:
    """n standard normals (float64) via Box-Muller on a SplitMix64 stream."""
    m = (n + 1) // 2
    r = splitmix64(seed, 2 * m)
    u1 = ((r[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53   # (0, 1]
    u2 = (r[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53           # [0, 1)
    rad = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * m, dtype=np.float64)
    z[0::2] = rad * np.cos(2.0 * np.pi * u2)
    z[1::2] = rad * np.sin(2.0 * np.pi * u2)
    return z[:n]


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float64 -> float32 -> bf16 (RNE) and return the uint16 bit patterns."""
    f = np.asarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return b.astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def tensor_seed(layer: int, chunk: int, tensor_id: int, base: int = 0x4C4C32) -> int:
    return base ^ ((layer << 40) | (chunk << 8) | tensor_id)


class Tensor:
    """A generated tensor: exact float64 values plus the raw bytes in its dtype."""

    def __init__(self, values: np.ndarray, dtype: str):
        self.dtype = dtype
        if dtype == "bf16":
            self.raw = to_bf16_bits(values)
            self.f64 = bf16_bits_to_f64(self.raw)
        elif dtype == "fp32":
            self.raw = np.asarray(values, dtype=np.float32)
            self.f64 = self.raw.astype(np.float64)
        else:
            raise ValueError(dtype)
        self.shape = self.f64.shape

    def torch(self, device="cpu"):
        import torch
        if self.dtype == "bf16":
            t = torch.from_numpy(self.raw.view(np.int16).copy()).view(torch.bfloat16)
        else:
            t = torch.from_numpy(self.raw.copy())
        return t.to(device)


def make_qkv(T: int, H: int, d: int, dtype: str = "bf16", layer: int = 0, chunk: int = 0,
             variant: str = "iid", base_seed: int = 0x4C4C32):
    """(Q, K, V) for one (layer, chunk): each a Tensor of shape [T, H, d]."""
    n = T * H * d
    out = []
    for tid in range(3):
        x = normal(tensor_seed(layer, chunk, tid, base_seed), n).reshape(T, H, d)
        if variant == "peaked" and tid == 0:
            x = x * 3.0
        elif variant == "outlier" and tid == 1:
            off = np.zeros(d)
            ch = [d // 8, 3 * d // 8, 5 * d // 8, 7 * d // 8]
            off[ch] = [8.0, -8.0, 8.0, -8.0]
            x = x + off
        elif variant not in ("iid", "peaked", "outlier"):
            raise ValueError(variant)
        out.append(Tensor(x, dtype))
    return tuple(out)


def make_tensor(shape, dtype="bf16", seed=1, scale=1.0):
    n = int(np.prod(shape))
    return Tensor(normal(seed, n).reshape(shape) * scale, dtype)
