"""BASELINE.json configs[2] and [3] at full Wan shape (-m gpu): the 30-layer rollout with the 3-frame
sink + 21-frame window (W30), parity against the oracle (every row and head at t = 0, 6, 7), and the long-rollout cache
footprint (L240: NVFP4 vs bf16 KV).  Inputs come from a pool of 4 seeded chunks (as in
SURVEY.md §8(d)), so the oracle quantizes each distinct tensor once."""
import numpy as np
import pytest
import torch

from oracle import nvfp4
from oracle.attention import attention
from oracle.keyset import key_token_ranges
from paper_2605_18739_b200 import kvq, synth

from gpu_util import check_bf16_out, check_fp32_out

pytestmark = pytest.mark.gpu
DEV = "cuda"
T, H, D, TPF, FC, SINK, WIN, SLOTS = 4680, 12, 128, 1560, 3, 3, 21, 8
POOL = 4


def _pool_index(layer, chunk):
    return (layer * 7 + chunk) % POOL


@pytest.fixture(scope="module")
def pool():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = []
    for i in range(POOL):
        q, k, v = synth.make_qkv(T, H, D, "bf16", 0, 100 + i)
        out.append((q, k, v))
    return out


@pytest.fixture(scope="module")
def pool_dequant(pool):
    return [(nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(k.f64), T, H, D),
             nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(v.f64), T, H, D)) for _, k, v in pool]


def _oracle_keys(layer, t, deq):
    Ks, Vs = [], []
    for a, b in key_token_ranges(t, FC, TPF, SINK, WIN):
        tok = a
        while tok < b:
            ch = tok // T
            end = min(b, (ch + 1) * T)
            Kc, Vc = deq[_pool_index(layer, ch)]
            Ks.append(Kc[tok - ch * T:end - ch * T])
            Vs.append(Vc[tok - ch * T:end - ch * T])
            tok = end
    return np.concatenate(Ks), np.concatenate(Vs)


ROWS = np.array([0, 127, 128, 2500, 4607, 4679])
FULL_T = (0, 6, 7)          # every row and head at the first chunk, the last ramp chunk and the first steady one


def test_w30_rollout_parity(pool, pool_dequant):
    L = 30
    cache = kvq.KVCache(L, H, D, TPF, FC, sink_frames=SINK, window_frames=WIN, max_chunk_slots=SLOTS, device=DEV)
    dev_pool = [tuple(x.torch(DEV) for x in qkv) for qkv in pool]
    for t in range(9):
        for layer in range(L):
            q, k, v = dev_pool[_pool_index(layer, t)]
            cache.append(layer, t, k, v)
            m = kvq.Mask(t, SINK, WIN)
            O = cache.attention(layer, q, m, torch.float32)
            if layer in (0, 29) and t in (0, 6, 7, 8):
                n_keys = sum(b - a for a, b in key_token_ranges(t, FC, TPF, SINK, WIN))
                assert cache.n_keys(layer, m) == n_keys
                assert n_keys == (37440 if t >= 7 else 4680 * (t + 1))
                Kk, Vk = _oracle_keys(layer, t, pool_dequant)
                rows = None if t in FULL_T else ROWS
                ref = attention(pool[_pool_index(layer, t)][0].f64, Kk, Vk, rows=rows)
                O32 = O.cpu().numpy()
                check_fp32_out(O32 if rows is None else O32[rows], ref)
                if layer == 0 and rows is None:
                    Ob = cache.attention(layer, q, m, torch.bfloat16).float().cpu().numpy()
                    check_bf16_out(Ob, ref, O32)
        for layer in (0, 29):
            assert cache.resident_chunks(layer) == min(t + 1, 8)   # sink chunk 0 + 7-chunk window


def test_l240_footprint_nvfp4_vs_bf16(pool):
    # long rollout: the cache footprint stays at sink + window chunks per layer, 32/9 of bf16 payload
    L = 30
    cache = kvq.KVCache(L, H, D, TPF, FC, sink_frames=SINK, window_frames=WIN, max_chunk_slots=SLOTS, device=DEV)
    k, v = pool[0][1].torch(DEV), pool[0][2].torch(DEV)
    for t in range(12):
        for layer in range(L):
            cache.append(layer, t, k, v)
    per_chunk = nvfp4.storage_bytes(T, H, D)
    assert cache.resident_bytes() == L * SLOTS * per_chunk
    bf16_bytes = L * SLOTS * 2 * T * H * D * 2
    ratio = bf16_bytes / (cache.resident_bytes() - L * SLOTS * 8)
    assert abs(ratio - 32 / 9) < 1e-12
    # 1.94 GB NVFP4 vs 6.90 GB bf16 for 8 slots x 30 layers
    assert abs(cache.resident_bytes() / 1e9 - 1.94) < 0.01 and abs(bf16_bytes / 1e9 - 6.90) < 0.01
    assert cache.arena_bytes < 2.05e9
