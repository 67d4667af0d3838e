"""Pins for oracle/keyset.py, oracle/attention.py and oracle/cache.py (-m "not gpu")."""
import math

import mpmath
import numpy as np
import pytest

from oracle import nvfp4
from oracle.attention import attention, softmax_rows
from oracle.cache import OracleKVCache
from oracle.keyset import key_frames, key_token_ranges
from paper_2605_18739_b200 import synth


# --------------------------------------------------------------------------- K_eff
def _chunks(frames, fc):
    return sorted({f // fc for f in frames})


@pytest.mark.parametrize("fc", [1, 3])
def test_keyset_spec_example(fc):
    # A_g = {0}, shot at 5, W = 4 history chunks, t = 10 -> {0,5,6,7,8,9} (+ current 10,
    # reading Z9/Z10: window_frames counts the current chunk)
    fr = key_frames(10, fc, sink_frames=fc, window_frames=5 * fc, shot_start_frame=5 * fc,
                    shot_len_frames=fc)
    assert _chunks(fr, fc) == [0, 5, 6, 7, 8, 9, 10]


def test_keyset_dedup_when_window_covers_sinks():
    # t = 2, W = 4, A_g = {0}, shot at 0 -> {0, 1} (+ current 2)
    assert _chunks(key_frames(2, 3, 3, 15, 0, 3), 3) == [0, 1, 2]


def test_keyset_prompt_switch_example():
    # switch at 7, query t = 12, W = 3 -> {7} + {9,10,11} + A_g (+ current 12)
    assert _chunks(key_frames(12, 2, 2, 8, 14, 2), 2) == [0, 7, 9, 10, 11, 12]


def test_keyset_g2_w30_ranges():
    # F_c = 3, 1560 tokens/frame, S_g = 3 frames, window 21 frames incl. current
    R = lambda t: key_token_ranges(t, 3, 1560, 3, 21)
    assert R(0) == [(0, 4680)]
    assert R(1) == [(0, 9360)]
    assert R(5) == [(0, 28080)]
    assert R(6) == [(0, 32760)]
    assert R(7) == [(0, 37440)]
    assert R(8) == [(0, 4680), (9360, 42120)]
    assert R(9) == [(0, 4680), (14040, 46800)]
    for t in range(7, 40):
        assert sum(b - a for a, b in R(t)) == 37440


def test_keyset_bound_and_shot_pointer_zero_copy():
    # PAPER.md:187 / SPEC.md:315: |K_eff| <= (S_g + S_s + W) L_f for all t
    for t in range(0, 50):
        for (sg, w, s0, sl) in [(3, 21, 0, 0), (3, 21, 30, 6), (0, 9, 12, 3), (6, 6, 3, 9)]:
            n = sum(b - a for a, b in key_token_ranges(t, 3, 10, sg, w, s0, sl))
            assert n <= (sg + sl + w) * 10
            assert n >= min((t + 1) * 3, 3) * 10       # the current chunk is always there


# --------------------------------------------------------------------------- attention
def _rand(shape, seed):
    return synth.make_tensor(shape, "fp32", seed=seed).f64


def test_softmax_rows_sum_to_one():
    Q, K = _rand((17, 2, 64), 1), _rand((50, 2, 64), 2)
    P = softmax_rows(Q * 4, K)
    assert np.max(np.abs(P.sum(-1) - 1.0)) < 1e-12


def test_constant_v_gives_o_equal_v():
    # north_star pin "constant V giving O = V": V = c everywhere -> V^ = 2688 g sign(c) = O
    T, H, d = 64, 2, 64
    Q, K = _rand((T, H, d), 3), _rand((T, H, d), 4)
    V = np.full((T, H, d), 0.7)
    cache = OracleKVCache(1, H, d, 64, 1)
    cache.append(0, 0, K, V)
    O = cache.attend(0, 0, Q, 0, 10)
    g = nvfp4.tensor_scale(V)
    assert np.allclose(O, 2688.0 * g, rtol=1e-14, atol=0)
    assert float(np.float32(O[0, 0, 0])) == np.float32(0.70000004)


def test_zero_q_gives_mean_of_v():
    Q = np.zeros((5, 2, 32))
    K, V = _rand((40, 2, 32), 5), _rand((40, 2, 32), 6)
    O = attention(Q, K, V)
    assert np.allclose(O, V.mean(0)[None], atol=1e-14, rtol=0)


def test_single_key_gives_that_value():
    Q, K, V = _rand((7, 3, 16), 7), _rand((1, 3, 16), 8), _rand((1, 3, 16), 9)
    assert np.array_equal(attention(Q, K, V), np.broadcast_to(V, (7, 3, 16)))


def test_key_permutation_invariance():
    Q, K, V = _rand((9, 2, 32), 10), _rand((30, 2, 32), 11), _rand((30, 2, 32), 12)
    p = np.random.default_rng(0).permutation(30)
    assert np.allclose(attention(Q, K, V), attention(Q, K[p], V[p]), atol=1e-13, rtol=0)


def test_attention_vs_mpmath_bruteforce():
    # brute force at 50 digits with plain loops (no matmul) on 2 heads x 3 queries x 16 dims
    Q, K, V = _rand((3, 2, 16), 13), _rand((5, 2, 16), 14), _rand((5, 2, 16), 15)
    O = attention(Q, K, V)
    mpmath.mp.dps = 50
    for i in range(3):
        for h in range(2):
            s = [mpmath.fsum(mpmath.mpf(Q[i, h, u]) * mpmath.mpf(K[j, h, u]) for u in range(16))
                 / mpmath.sqrt(16) for j in range(5)]
            w = [mpmath.exp(x) for x in s]
            z = mpmath.fsum(w)
            for u in range(16):
                ref = mpmath.fsum(w[j] * mpmath.mpf(V[j, h, u]) for j in range(5)) / z
                assert abs(float(ref) - O[i, h, u]) < 1e-14


def test_cache_pipeline_tiny_vs_bruteforce():
    # tiny config: 2 heads x 64 dim, 3 chunks x 64 tokens, fp32, full window; the cached pipeline
    # equals dequant-then-attend written with plain Python sums over the key set
    T, H, d = 64, 2, 64
    cache = OracleKVCache(1, H, d, 64, 1)
    chunks = [synth.make_qkv(T, H, d, "fp32", 0, c) for c in range(3)]
    Ks, Vs = [], []
    for c, (q, k, v) in enumerate(chunks):
        cache.append(0, c, k.f64, v.f64)
        Ks.append(nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(k.f64), T, H, d))
        Vs.append(nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(v.f64), T, H, d))
    Q = chunks[2][0].f64
    O = cache.attend(0, 2, Q, 0, 1 << 20)
    K, V = np.concatenate(Ks), np.concatenate(Vs)
    for i in (0, 31, 63):
        for h in range(H):
            s = [math.fsum(Q[i, h] * K[j, h]) / 8.0 for j in range(3 * T)]
            m = max(s)
            w = [math.exp(x - m) for x in s]
            z = math.fsum(w)
            ref = [math.fsum(w[j] * V[j, h, u] for j in range(3 * T)) / z for u in range(d)]
            assert np.allclose(O[i, h], ref, atol=1e-13, rtol=0)


def test_cache_keys_follow_ranges_across_chunks():
    # sink (first frame of chunk 0) + window covering the tail of chunk 1 and chunk 2
    H, d, tpf, fc = 1, 16, 4, 2
    cache = OracleKVCache(1, H, d, tpf, fc)
    raw = []
    for c in range(3):
        K = np.full((8, H, d), float(c + 1)) + np.arange(8)[:, None, None] * 0.01
        cache.append(0, c, K, K)
        raw.append(nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(K), 8, H, d))
    Kk, _ = cache.keys(0, 2, sink_frames=1, window_frames=3)
    # frames {0} U {3, 4, 5} -> tokens [0,4) U [12,24)
    ref = np.concatenate([raw[0][0:4], raw[1][4:8], raw[2]])
    assert np.array_equal(Kk, ref)


def test_q_nvfp4_mode_is_identity_on_lattice_queries_and_quantizes_otherwise():
    # reading Z24 (NVFP4 Q before the all-to-all): queries already on the NVFP4 lattice
    # (g = 2^-8, a +-6 in every block so the scale is recovered) pass through unchanged; other queries
    # are replaced by their exact dequantized NVFP4 values
    T, H, d = 16, 2, 32
    rng = np.random.default_rng(7)
    c = OracleKVCache(1, H, d, T, 1)
    k = synth.make_tensor((T, H, d), "fp32", seed=11).f64
    v = synth.make_tensor((T, H, d), "fp32", seed=12).f64
    c.append(0, 0, k, v)
    mags = np.array([0, 0.5, 1, 1.5, 2, 3, 4, 6])
    e = rng.choice(mags, size=(T * H, d // 16, 16)) * rng.choice([-1, 1], size=(T * H, d // 16, 16))
    e[:, :, 0] = 6.0
    s = nvfp4.e4m3_decode(rng.integers(40, 110, size=(T * H, d // 16)).astype(np.uint8))
    s[0, 0] = 448.0
    q_lat = (e * s[..., None] * 2.0 ** -8).reshape(T, H, d)
    np.testing.assert_array_equal(c.attend(0, 0, q_lat, 0, 1, q_nvfp4=True), c.attend(0, 0, q_lat, 0, 1))
    q = synth.make_tensor((T, H, d), "fp32", seed=13).f64
    q_hat = nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(q), T, H, d)
    assert not np.array_equal(q_hat, q)
    np.testing.assert_array_equal(c.attend(0, 0, q, 0, 1, q_nvfp4=True), attention(q_hat, *c.keys(0, 0, 0, 1)))
