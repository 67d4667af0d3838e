"""Pins for the oracle's §8(f) modes (-m "not gpu"): Four-Over-Six block-scale search
(App. F Eq. 4o6) and K-smoothing with mean restitution
(§3.2), plus the exact float32 FMA helper both rely on.

Each pin is something the paper, SPEC.md or arithmetic fixes independently of the oracle's own
code: SPEC's worked 4/6 examples, exact-rational brute force, hand-computed float32 sums, the
4-target analogue of the "block max codes to 6" invariant, argmin dominance, lattice round trips
(which make the reconstruction exact, so attention over the cache equals attention over the raw
keys), constant-row and shift properties of a mean subtraction, and SPEC.md:277/320's "smoothing
does not lose to plain quantization" check.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import nvfp4
from oracle.attention import attention
from oracle.cache import OracleKVCache
from paper_2605_18739_b200 import synth


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def rn32_fraction(q: Fraction) -> float:
    """Correctly rounded float32 of an exact rational (brute force on the two neighbours)."""
    x = np.float32(float(q))          # within an ulp or so
    cands = {float(x), float(np.nextafter(x, np.float32(np.inf))), float(np.nextafter(x, np.float32(-np.inf)))}
    best = sorted(cands, key=lambda c: (abs(Fraction(c) - q), int(np.float32(c).view(np.uint32)) & 1))
    return best[0]


# ----------------------------------------------------------------------------- exact FMA
def test_rn32_fma_against_fractions():
    rng = np.random.default_rng(7)
    n = 4000
    a = f32(rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n)))
    b = f32(rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n)))
    c = f32(rng.standard_normal(n) * np.exp2(rng.integers(-40, 40, n)))
    # constructed near-midpoint cases: c = -(a*b) + a half-ulp-ish perturbation
    m = 1000
    c[:m] = f32(-(a[:m] * b[:m]) + np.ldexp(1.0, -60))
    got = nvfp4._rn32_fma(a, b, c)
    for i in range(n):
        want = rn32_fraction(Fraction(float(a[i])) * Fraction(float(b[i])) + Fraction(float(c[i])))
        assert got[i] == want, (i, a[i], b[i], c[i], got[i], want)


def test_rn32_fma_exact_midpoints():
    # p + c rounds in float64 exactly onto a float32 midpoint; the TwoSum error must decide,
    # and here ties-to-even of the float64 sum would pick the wrong neighbour.
    #  c = 2^24, p = (1 + 2^-12)(1 - 2^-12 + 2^-24) = 1 + 2^-36 -> exact 2^24 + 1 + 2^-36 -> 2^24 + 2
    #  c = 2^24 + 2, p = (1 + 2^-23)(1 - 2^-23) = 1 - 2^-46 -> exact 2^24 + 3 - 2^-46 -> 2^24 + 2
    a = np.array([1 + 2.0 ** -12, 1 + 2.0 ** -23])
    b = np.array([1 - 2.0 ** -12 + 2.0 ** -24, 1 - 2.0 ** -23])
    c = np.array([2.0 ** 24, 2.0 ** 24 + 2])
    assert np.array_equal(f32(a), a) and np.array_equal(f32(b), b)
    np.testing.assert_array_equal(nvfp4._rn32_fma(a, b, c), [2.0 ** 24 + 2, 2.0 ** 24 + 2])
    assert np.array_equal(f32(a * b + c), [2.0 ** 24, 2.0 ** 24 + 4])   # the naive double rounding


# ----------------------------------------------------------------------------- K-smoothing
def test_row_sum_tree_order_hand_example():
    # [2^24, 1 x 15]: y_0 = RN32(2^24 + 1) = 2^24 (tie to even), y_1..7 = 2; z_0 = 2^24 + 2,
    # z_1..3 = 4; w_0 = 2^24 + 6, w_1 = 8; S = 2^24 + 14 (the exact sum is 2^24 + 15; a
    # left-to-right float32 sum would give 2^24).
    x = np.ones((1, 16))
    x[0, 0] = 2.0 ** 24
    assert nvfp4.row_sum_fp32(x)[0] == 2.0 ** 24 + 14
    # blocks are combined as adjacent pairs: ((S0+S1)+(S2+S3)) for d = 64
    y = np.zeros((1, 64))
    y[0, 0], y[0, 16], y[0, 32], y[0, 48] = 2.0 ** 24, 1.0, 1.0, 1.0
    # S0 + S1 = 2^24 + 1 -> 2^24; S2 + S3 = 2; total 2^24 + 2
    assert nvfp4.row_sum_fp32(y)[0] == 2.0 ** 24 + 2


def test_row_sum_exact_on_grid():
    rng = np.random.default_rng(3)
    x = rng.integers(-512, 512, size=(50, 128)) / 64.0          # dyadic, sums exact in float32
    np.testing.assert_array_equal(nvfp4.row_sum_fp32(x), x.sum(axis=1))


def test_k_smooth_constant_rows_and_zero():
    # constant key rows -> smoothed rows zero, means = c, zero blocks
    c = np.array([0.75, -3.5, 0.0, 1e-3])
    x = np.repeat(f32(c)[:, None], 128, axis=1)
    xb, m = nvfp4.k_smooth(x)
    assert np.all(xb == 0) and np.array_equal(m, f32(c))
    q = nvfp4.quantize_kv_chunk(x.reshape(4, 1, 128), smooth=True)
    assert q["g"] == 1.0 and np.all(q["scales"] == 0) and np.all(q["codes"] == 0)
    np.testing.assert_array_equal(nvfp4.dequantize_kv_chunk(q, 4, 1, 128).reshape(4, 128), x)


def test_k_smooth_shift_invariance_on_grid():
    rng = np.random.default_rng(5)
    x = rng.integers(-64, 64, size=(40, 64)) / 16.0
    shift = rng.integers(-40, 40, size=(40, 1)) / 8.0
    xb0, m0 = nvfp4.k_smooth(x)
    xb1, m1 = nvfp4.k_smooth(x + shift)
    np.testing.assert_array_equal(xb0, xb1)
    np.testing.assert_array_equal(m1 - m0, shift[:, 0])
    np.testing.assert_allclose(xb0.mean(axis=1), 0.0, atol=1e-12)


def test_smoothing_not_worse_than_plain_on_offset_keys():
    # dequantized-plus-mean keys vs plain quantization, >= 100 seeded chunks
    # with per-row offsets (the structure smoothing targets); MSE of the smoothed path is lower
    # on every chunk.
    for seed in range(100):
        k = synth.make_tensor((64, 2, 64), "bf16", seed=9000 + seed).f64
        off = synth.make_tensor((64, 2, 1), "bf16", seed=19000 + seed).f64 * 2.0
        K = f32(k + off)
        plain = nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(K), 64, 2, 64)
        smooth = nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(K, smooth=True), 64, 2, 64)
        assert np.mean((smooth - K) ** 2) < np.mean((plain - K) ** 2), seed


def _lattice_zero_mean_rows(rows, d, rng):
    """Rows of exact NVFP4 lattice values (g = 2^-8) with every block holding +-6 at scale 448 in
    row 0 and pairs (+v, -v) so each row sums to zero exactly."""
    g = 2.0 ** -8
    half = rng.integers(0, 8, size=(rows, d // 16, 8))
    mags = nvfp4.E2M1_MAGNITUDES[half]
    sc = nvfp4.e4m3_decode(rng.integers(0x30, 0x70, size=(rows, d // 16)))
    mags[:, :, 0] = 6.0
    sc[0, 0] = 448.0
    blk = np.concatenate([mags, -mags], axis=-1) * sc[..., None] * g
    return blk.reshape(rows, d)


def test_smoothing_lattice_round_trip_makes_attention_exact():
    rng = np.random.default_rng(11)
    T, H, d = 32, 2, 64
    L = _lattice_zero_mean_rows(T * H, d, rng)
    mean = rng.integers(-16, 16, size=(T * H, 1)) / 4.0
    K = (L + mean).reshape(T, H, d)
    assert np.array_equal(f32(K), K)
    q = nvfp4.quantize_kv_chunk(K, smooth=True)
    np.testing.assert_array_equal(q["mean"], mean[:, 0])
    assert q["g"] == 2.0 ** -8
    Kh = nvfp4.dequantize_kv_chunk(q, T, H, d)
    np.testing.assert_array_equal(Kh, K)
    Q = synth.make_tensor((T, H, d), "fp32", seed=1).f64
    V = synth.make_tensor((T, H, d), "fp32", seed=2).f64
    cache = OracleKVCache(1, H, d, T, 1, k_smoothing=True)
    cache.append(0, 0, K, V)
    Vh = cache.dequantized_chunk(0, 0)[1]
    np.testing.assert_allclose(cache.attend(0, 0, Q, 0, 1), attention(Q, K, Vh), atol=1e-12)


def test_dequantize_rn32_with_mean_is_one_rounding():
    rng = np.random.default_rng(2)
    K = synth.make_tensor((16, 2, 64), "bf16", seed=77).f64 + 3.0
    q = nvfp4.quantize_kv_chunk(K, smooth=True)
    got = nvfp4.dequantize_kv_chunk_rn32(q, 16, 2, 64).reshape(32, 64)
    codes = nvfp4.unpack_codes(q["codes"])
    v = nvfp4.e2m1_decode(codes) * np.repeat(nvfp4.e4m3_decode(q["scales"]), 16, axis=1)
    for i in rng.integers(0, 32 * 64, 300):
        r, c = divmod(int(i), 64)
        want = rn32_fraction(Fraction(float(v[r, c])) * Fraction(q["g"]) + Fraction(float(q["mean"][r])))
        assert got[r, c] == want


# ----------------------------------------------------------------------------- Four-Over-Six
def _with_unit_g(block):
    """Tensor whose first block holds 2688 (so g = RN32(2688/2688) = 1) followed by `block`."""
    x = np.zeros((2, 16))
    x[0, 0] = 2688.0
    x[1, :len(block)] = block
    return x


def test_four_over_six_spec_examples():
    # [6, 4.5, 0 x 14], g = 1 -> 4-target scale 1.5 (codes 4 and 3), MSE 0
    c, s, g = nvfp4.quantize(_with_unit_g([6.0, 4.5]), scale_search=True)
    assert g == 1.0 and nvfp4.e4m3_decode(s[1, 0]) == 1.5
    assert list(nvfp4.e2m1_decode(c[1, :2])) == [4.0, 3.0]
    assert np.array_equal(nvfp4.dequantize(c, s, g)[1], _with_unit_g([6.0, 4.5])[1])
    # the standard scale 1.0 rounds 4.5 to 4 (MSE > 0)
    c6, s6, _ = nvfp4.quantize(_with_unit_g([6.0, 4.5]))
    assert nvfp4.e4m3_decode(s6[1, 0]) == 1.0 and list(nvfp4.e2m1_decode(c6[1, :2])) == [6.0, 4.0]
    # [6, 0...] -> both exact, tie -> 6-target
    _, s, _ = nvfp4.quantize(_with_unit_g([6.0]), scale_search=True)
    assert nvfp4.e4m3_decode(s[1, 0]) == 1.0
    # sixteen 6.0 -> 6-target scale 1.0, codes 6
    c, s, _ = nvfp4.quantize(_with_unit_g([6.0] * 16), scale_search=True)
    assert nvfp4.e4m3_decode(s[1, 0]) == 1.0 and np.all(nvfp4.e2m1_decode(c[1]) == 6.0)
    # [6, 5.9, 0...] -> both reconstruct 5.9 as 6.0 (equal error) -> 6-target
    _, s, _ = nvfp4.quantize(_with_unit_g([6.0, float(f32(5.9))]), scale_search=True)
    assert nvfp4.e4m3_decode(s[1, 0]) == 1.0
    # zero block: scale 0, codes 0 in both modes
    c, s, _ = nvfp4.quantize(_with_unit_g([]), scale_search=True)
    assert s[1, 0] == 0 and np.all(c[1] == 0)


def _exact_sse(x, c, s, g):
    xb = x.reshape(x.shape[0], -1, 16)
    v = nvfp4.dequantize(c, s, g).reshape(xb.shape)
    return ((xb - v) ** 2).sum(axis=-1)   # f64: differences exact, squares/sums within 2^-50


@pytest.mark.parametrize("variant", ["iid", "outlier"])
def test_four_over_six_dominance_and_argmin(variant):
    x = synth.make_qkv(64, 4, 128, "bf16", 0, 4242, variant=variant)[1].f64.reshape(256, 128)
    c6, s6, g = nvfp4.quantize(x)
    cs, ss, gs = nvfp4.quantize(x, scale_search=True)
    assert gs == g
    e6, es = _exact_sse(x, c6, s6, g), _exact_sse(x, cs, ss, g)
    # dominance (up to float32 rounding of the compared errors)
    assert np.all(es <= e6 * (1 + 2.0 ** -20) + 1e-300)
    # the choice is the exact argmin except at float32 near-ties
    x4 = x.reshape(256, 8, 16)
    bmax = np.abs(x4).max(axis=-1)
    s4, d4 = nvfp4._block_scales(bmax, f32(bmax / g), g, 4.0)
    c4 = nvfp4._block_codes(x4, bmax, d4).reshape(256, 128)
    e4 = _exact_sse(x, c4, s4, g)
    picked4 = (ss == s4) & (ss != s6)
    clear = np.abs(e4 - e6) > 2.0 ** -18 * np.maximum(e4, e6)
    assert np.all((e4 < e6)[clear] == picked4[clear])
    assert 0.05 < picked4.mean() < 0.95        # both candidates win a real share of blocks


def test_four_over_six_block_max_codes_to_four():
    # analogue of the "scale = amax/6" invariant: a block that takes a normal 4-target scale
    # has its max-magnitude element at code +-4 (bmax/d_b in [4/(1+2^-4), 4/(1-2^-4)] rounds to 4)
    x = synth.make_tensor((256, 128), "bf16", seed=99).f64
    c, s, g = nvfp4.quantize(x, scale_search=True)
    c6, s6, _ = nvfp4.quantize(x)
    xb = x.reshape(256, 8, 16)
    cb = c.reshape(256, 8, 16)
    arg = np.abs(xb).argmax(axis=-1)
    top = np.abs(nvfp4.e2m1_decode(np.take_along_axis(cb, arg[..., None], -1)[..., 0]))
    took4 = (s != s6) & (s >= 0x08) & (s < 0x7E)      # a normal, unsaturated 4-target scale
    assert took4.any()
    assert np.all(top[took4] == 4.0)
    assert np.all(top[(s == s6) & (s6 >= 0x08) & (s6 < 0x7E)] == 6.0)   # the standard invariant


def test_four_over_six_lattice_and_value_idempotence():
    # a lattice built on 4-target scales (block max code 4) is recovered exactly
    rng = np.random.default_rng(8)
    g = 2.0 ** -8
    codes = rng.integers(0, 7, size=(64, 8, 16))            # magnitudes up to 4
    codes[:, :, 0] = 6                                       # code 6 = value 4 (block max)
    sc = nvfp4.e4m3_decode(rng.integers(0x30, 0x60, size=(64, 8)))
    x = nvfp4.E2M1_MAGNITUDES[codes] * sc[..., None] * g * np.where(rng.random((64, 8, 16)) < 0.5, -1, 1)
    x[0, 0, :] = 0.0
    x[0, 0, 0] = 6.0 * 448.0 * g                             # amax = 2688 g -> g recovered
    x = x.reshape(64, 128)
    c, s, gg = nvfp4.quantize(x, scale_search=True)
    assert gg == g
    np.testing.assert_array_equal(nvfp4.dequantize(c, s, gg), x)
    # Q(D(Q(x))) reproduces the values (bytes may differ only where both candidates are exact)
    y = synth.make_tensor((128, 128), "bf16", seed=5).f64
    c1, s1, g1 = nvfp4.quantize(y, scale_search=True)
    d1 = nvfp4.dequantize(c1, s1, g1)
    c2, s2, g2 = nvfp4.quantize(d1, scale_search=True)
    assert g2 == g1
    np.testing.assert_array_equal(nvfp4.dequantize(c2, s2, g2), d1)


def test_block_sse_fp32_is_float32_fma_chain():
    # E = RN32(A + B), A/B float32 FMA chains over even/odd elements, r_i one rounding;
    # compared with an exact-rational evaluation of the same sequence on a few blocks
    x = synth.make_tensor((4, 4, 16), "bf16", seed=3).f64
    c, s, g = nvfp4.quantize(x.reshape(4, 64))
    cb = c.reshape(4, 4, 16)
    got = nvfp4.block_sse_fp32(x, cb, s, g)
    for r in range(4):
        for b in range(4):
            acc = [0.0, 0.0]
            for i in range(16):
                v = Fraction(float(nvfp4.e2m1_decode(cb[r, b, i]))) * Fraction(float(nvfp4.e4m3_decode(s[r, b])))
                ri = rn32_fraction(Fraction(float(x[r, b, i])) - v * Fraction(g))
                acc[i & 1] = rn32_fraction(Fraction(ri) * Fraction(ri) + Fraction(acc[i & 1]))
            assert got[r, b] == rn32_fraction(Fraction(acc[0]) + Fraction(acc[1]))
