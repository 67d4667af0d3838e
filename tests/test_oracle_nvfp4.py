"""Pins for oracle/nvfp4.py against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins.  None re-types the oracle's own formula:
the checks use printed values, an independent library
(ml_dtypes, a different rounding implementation), exact rational arithmetic
(fractions.Fraction), constructed lattices, and invariants.
"""
import json
import math
import os
from fractions import Fraction

import ml_dtypes
import numpy as np
import pytest

from oracle import nvfp4
from paper_2605_18739_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------- E2M1
def test_e2m1_value_set_is_papers():
    # PAPER.md:719 prints the E2M1 set {0, +-0.5, +-1, +-1.5, +-2, +-3, +-4, +-6}
    vals = set(nvfp4.e2m1_decode(np.arange(16)).tolist())
    assert vals == {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0, -0.5, -1.0, -1.5, -2.0, -3.0, -4.0, -6.0}
    assert nvfp4.e2m1_decode(8) == 0.0          # negative zero decodes to 0.0
    assert nvfp4.M_FP4 == 6.0


@pytest.mark.parametrize("x,want", [
    (2.5, 2.0), (0.74, 0.5), (6.0, 6.0), (0.0, 0.0),            # SPEC.md:47-51 examples
    (0.25, 0.0), (0.75, 1.0), (1.25, 1.0), (1.75, 2.0),         # ties -> even mantissa (Z3)
    (3.5, 4.0), (5.0, 4.0), (7.0, 6.0), (1e30, 6.0),            # ties + saturation (Z7)
    (-2.5, -2.0), (-5.5, -6.0), (0.2499, 0.0), (0.2501, 0.5),
])
def test_e2m1_encode_examples(x, want):
    assert nvfp4.e2m1_decode(nvfp4.e2m1_encode(x)) == want


def test_e2m1_negative_zero_code():
    # reading Z6: sign-preserving, -0.0 and tiny negatives give code 0x8
    assert int(nvfp4.e2m1_encode(-0.0)) == 8
    assert int(nvfp4.e2m1_encode(-0.1)) == 8
    assert int(nvfp4.e2m1_encode(0.1)) == 0


def test_e2m1_roundtrip_all_codes():
    codes = np.arange(16, dtype=np.uint8)
    vals = nvfp4.e2m1_decode(codes)
    vals = np.where(codes == 8, -0.0, vals)
    assert np.array_equal(nvfp4.e2m1_encode(vals), codes)


def test_e2m1_matches_ml_dtypes_dense_sweep():
    # independent library (RNE, saturating float4_e2m1fn) on a dense fp32 sweep incl. every tie
    x = np.concatenate([np.linspace(-8, 8, 200001), np.arange(-7, 7.01, 0.25)]).astype(np.float32)
    ref = x.astype(ml_dtypes.float4_e2m1fn).view(np.uint8) & 0xF
    assert np.array_equal(nvfp4.e2m1_encode(x.astype(np.float64)), ref)


# --------------------------------------------------------------------------- E4M3
def test_e4m3_table_matches_ml_dtypes():
    # all 256 patterns; 0x7F/0xFF are NaN in E4M3 (no inf); max 448
    ours = nvfp4.e4m3_decode(np.arange(256))
    ref = np.arange(256, dtype=np.uint8).view(ml_dtypes.float8_e4m3fn).astype(np.float64)
    assert np.array_equal(np.isnan(ours), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert np.array_equal(ours[ok], ref[ok])
    assert np.nanmax(ours) == nvfp4.M_FP8 == 448.0
    assert nvfp4.e4m3_decode(1) == 2.0 ** -9


@pytest.mark.parametrize("x,want", [(500.0, 448.0), (1.5, 1.5), (0.0, 0.0), (464.0, 448.0),
                                    (17.0, 16.0), (19.0, 20.0), (2.0 ** -10, 0.0), (1e9, 448.0),
                                    (3 * 2.0 ** -10, 2.0 ** -8), (3 * 2.0 ** -11, 2.0 ** -9)])
def test_e4m3_encode_examples(x, want):
    # SPEC.md:66-69 (500 -> 448, 1.5 -> 1.5); RNE ties; saturation at M^FP8
    assert nvfp4.e4m3_decode(nvfp4.e4m3_encode_nonneg(x)) == want


def test_e4m3_encode_matches_ml_dtypes_in_range():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(0, 448, 100000), np.exp2(rng.uniform(-12, 8.8, 100000)),
                        nvfp4.e4m3_decode(np.arange(0x7F))]).astype(np.float32)
    # midpoints between consecutive finite codes exercise every tie
    v = nvfp4.e4m3_decode(np.arange(0x7F))
    x = np.concatenate([x, ((v[1:] + v[:-1]) / 2).astype(np.float32)])
    x = x[x <= 448]
    ref = x.astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
    assert np.array_equal(nvfp4.e4m3_encode_nonneg(x.astype(np.float64)), ref)


# --------------------------------------------------------------------------- quantize
def _gold():
    with open(os.path.join(GOLD, "g1_nvfp4.json")) as f:
        return json.load(f)


def test_golden_g1():
    G = _gold()
    x = np.array(G["input_rows"], dtype=np.float64)
    x[0, 9] = -0.0
    codes, scales, g = nvfp4.quantize(x)
    assert np.float32(g).view(np.uint32) == int(G["g_bits"], 16)
    assert scales.tolist() == [[int(v, 16) for v in r] for r in G["scales_hex"]]
    assert codes.tolist() == G["codes"]
    packed = nvfp4.pack_codes(codes)
    assert [bytes(r).hex() for r in packed] == G["packed_hex"]
    deq = nvfp4.dequantize(codes, scales, g)
    assert deq[1, :4].tolist() == G["dequant_row1_first4"]


def _exact_rne(value: Fraction, grid):
    """Nearest point of a sorted list of Fractions, ties to the even index (RNE)."""
    best = min(range(len(grid)), key=lambda i: (abs(grid[i] - value), i % 2))
    return best


def _exact_quantize_pow2(x_rows):
    """Exact-real NVFP4 (reading Z4's R3) with rationals -- equals R1 when g is a power of two."""
    flat = [Fraction(v) for row in x_rows for v in row]
    amax = max(abs(v) for v in flat)
    g = amax / 2688
    assert g.numerator == 1 and (g.denominator & (g.denominator - 1)) == 0   # power of two
    e4 = [Fraction(float(v)) for v in nvfp4.e4m3_decode(np.arange(0x7F))]
    e2 = [Fraction(v) for v in [0, 0.5, 1, 1.5, 2, 3, 4, 6]]
    codes, scales = [], []
    for row in x_rows:
        crow, srow = [], []
        for b in range(0, len(row), 16):
            blk = [Fraction(v) for v in row[b:b + 16]]
            bmax = max(abs(v) for v in blk)
            if bmax == 0:
                srow.append(0)
                crow.extend([0] * 16)
                continue
            s = _exact_rne(bmax / (6 * g), e4)
            s = max(s, 1)
            db = e4[s] * g
            srow.append(s)
            for v in blk:
                m = min(abs(v / db), Fraction(6))
                c = _exact_rne(m, e2)
                crow.append(c + (8 if (v < 0 or (v == 0 and math.copysign(1, float(v)) < 0)) else 0))
        codes.append(crow)
        scales.append(srow)
    return np.array(codes, dtype=np.uint8), np.array(scales, dtype=np.uint8), float(g)


def test_quantize_matches_exact_rationals_pow2_scale():
    # definition-agnostic pin (Z4): power-of-two g makes every decode scale exact
    t = synth.make_tensor((48, 64), "bf16", seed=11, scale=2.0)
    x = np.clip(t.f64, -10.0, 10.0)
    x[5, 7] = -10.5                     # amax = 2688 * 2^-8 exactly
    x[9, 16:32] = 0.0                   # a zero block
    x[11, 32:48] = x[11, 32:48] * 1e-3  # a small-scale block
    x = synth.bf16_bits_to_f64(synth.to_bf16_bits(x))
    c, s, g = nvfp4.quantize(x)
    ce, se, ge = _exact_quantize_pow2(x.tolist())
    assert g == ge == 2.0 ** -8
    assert np.array_equal(s, se)
    assert np.array_equal(c, ce)


def test_quantize_matches_float32_ml_dtypes_implementation():
    # the same R1 sequence computed independently: IEEE float32 numpy arithmetic + ml_dtypes casts
    for seed, scale in [(3, 1.0), (5, 0.37), (7, 45.0), (9, 0.01)]:
        t = synth.make_tensor((64, 12, 128), "bf16", seed=seed, scale=scale)
        x = t.f64.reshape(-1, 128)
        c, s, g = nvfp4.quantize(x)
        x32 = x.astype(np.float32)
        g32 = np.float32(np.abs(x32).max()) / np.float32(2688.0)
        xb = x32.reshape(x.shape[0], 8, 16)
        bmax = np.abs(xb).max(-1)
        u = (bmax / g32) / np.float32(6.0)
        s_ref = u.astype(ml_dtypes.float8_e4m3fn).view(np.uint8).copy()
        s_ref[(s_ref == 0) & (bmax > 0)] = 1
        s_ref[bmax == 0] = 0
        db = s_ref.view(ml_dtypes.float8_e4m3fn).astype(np.float32) * g32
        q = xb / db[..., None]
        c_ref = (q.astype(ml_dtypes.float4_e2m1fn).view(np.uint8) & 0xF).reshape(x.shape)
        assert np.float32(g) == g32
        assert np.array_equal(s, s_ref), seed
        assert np.array_equal(c, c_ref), seed


def test_scale_is_amax_over_6_invariant():
    # PAPER.md:726 alpha_i(6) = cast(max|U_bar|/6): every normal-scale block's max element codes to +-6
    t = synth.make_tensor((4680 // 10, 12, 128), "bf16", seed=3)
    c, s, g = nvfp4.quantize(t.f64.reshape(-1, 128))
    x = t.f64.reshape(-1, 8, 16)
    arg = np.abs(x).argmax(-1)
    cmax = np.take_along_axis(c.reshape(-1, 8, 16), arg[..., None], -1)[..., 0]
    normal = s >= 8                          # E4M3 exponent field != 0
    assert normal.mean() > 0.99
    assert np.all((cmax[normal] & 7) == 7)
    # the block holding amax gets the max scale 448 (u = 2688/6 up to one fp32 rounding)
    r, b = np.unravel_index(np.abs(x).max(-1).argmax(), s.shape)
    assert s[r, b] == 0x7E


def test_lattice_roundtrip():
    # x = e * s * g on the NVFP4 lattice (g = 2^-8, normal E4M3 s, +-6 in every block,
    # one block at s = 448) is recovered exactly: g, s and codes (Eq. 2 inverted)
    rng = np.random.default_rng(1)
    rows, nb = 40, 4
    s = rng.integers(8, 0x7E, size=(rows, nb)).astype(np.uint8)
    s[0, 0] = 0x7E
    e = rng.integers(0, 16, size=(rows, nb, 16)).astype(np.uint8)
    e[..., 3] = np.where(rng.random((rows, nb)) < 0.5, 7, 15)     # a +-6 in every block
    e = np.where(e == 8, 0, e)
    x = nvfp4.e2m1_decode(e) * nvfp4.e4m3_decode(s)[..., None] * 2.0 ** -8
    c, s2, g = nvfp4.quantize(x.reshape(rows, nb * 16))
    assert g == 2.0 ** -8
    assert np.array_equal(s2, s)
    assert np.array_equal(c.reshape(rows, nb, 16), e)


def test_idempotence():
    # Q(D(Q(x))) = Q(x): quantization is a projection onto the lattice
    for seed in (1, 2, 3):
        t = synth.make_tensor((256, 128), "bf16", seed=seed)
        c, s, g = nvfp4.quantize(t.f64)
        c2, s2, g2 = nvfp4.quantize(nvfp4.dequantize(c, s, g))
        assert g2 == g and np.array_equal(s2, s) and np.array_equal(c2, c)


def test_dequant_fp32_keeps_sign_of_zero_and_is_idempotent():
    # kv_dequantize's fp32 value RN32(dec(c) dec(s) g): Eq. 2 is a product, so code 0x8
    # (-0, reading Z6) must come back as -0.0, and re-quantizing the fp32 dequantized chunk gives the
    # same bytes (a sign-dropping +0 addend would turn every -0 code into 0x0)
    for seed in (3, 7):
        x = synth.make_tensor((64, 4, 128), "bf16", seed=seed).f64
        q = nvfp4.quantize_kv_chunk(x)
        codes = nvfp4.unpack_codes(q["codes"])
        assert (codes == 8).any()
        d32 = nvfp4.dequantize_kv_chunk_rn32(q, 64, 4, 128).reshape(256, 128)
        assert np.all(np.signbit(d32[codes == 8])) and not np.any(np.signbit(d32[codes == 0]))
        q2 = nvfp4.quantize_kv_chunk(d32.reshape(64, 4, 128))
        assert np.array_equal(q2["codes"], q["codes"]) and np.array_equal(q2["scales"], q["scales"])


def test_zero_and_underflow_conventions():
    z = np.zeros((3, 32))
    c, s, g = nvfp4.quantize(z)
    assert g == 1.0 and not c.any() and not s.any()          # Z5: zero tensor -> g = 1
    x = np.zeros((2, 32))
    x[0, 0] = 2688.0                                          # g = 1
    x[1, 16] = 1e-4                                           # bmax/6 = 1.7e-5 < 2^-10 -> E4M3 0
    x[1, 17] = -0.0
    c, s, g = nvfp4.quantize(x)
    assert g == 1.0
    assert s[1, 1] == 0x01                                    # promoted to 2^-9
    assert s[0, 1] == 0 and not c[0, 16:].any()               # zero block: scale 0, codes 0x00
    assert c[1, 17] == 8                                      # -0 in a non-zero block keeps its sign


def test_nonfinite_rejected_with_index():
    x = np.ones((4, 16))
    x[2, 5] = np.inf
    with pytest.raises(ValueError, match="index 37"):
        nvfp4.quantize(x)


def test_dequant_eq2_against_library_decoders():
    # Eq. 2 with independent decoders: ml_dtypes float4/float8 values times g
    t = synth.make_tensor((64, 128), "bf16", seed=4)
    c, s, g = nvfp4.quantize(t.f64)
    e = c.astype(np.uint8).view(ml_dtypes.float4_e2m1fn).astype(np.float64)
    sc = s.view(ml_dtypes.float8_e4m3fn).astype(np.float64)
    ref = (e.reshape(64, 8, 16) * sc[..., None] * g).reshape(64, 128)
    assert np.array_equal(nvfp4.dequantize(c, s, g), ref)


def test_storage_ratio_32_over_9():
    # 4 T_c H d bytes (bf16 K+V) -> 9/8 T_c H d bytes, "close to 3.6x"
    T, H, d = 4680, 12, 128
    nv = nvfp4.storage_bytes(T, H, d) - 8                     # ignore the two tensor scales
    assert Fraction(4 * T * H * d, nv) == Fraction(32, 9)
    assert abs(4 * T * H * d / nv - 3.6) < 0.05


def test_pack_roundtrip_and_order():
    codes = np.array([[1, 2, 3, 4]], dtype=np.uint8)
    assert nvfp4.pack_codes(codes).tolist() == [[0x21, 0x43]]  # element 2k in the low nibble
    r = np.random.default_rng(0).integers(0, 16, (7, 64)).astype(np.uint8)
    assert np.array_equal(nvfp4.unpack_codes(nvfp4.pack_codes(r)), r)
