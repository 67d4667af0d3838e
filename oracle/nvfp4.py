"""NVFP4 codecs and quantize / dequantize, float64 reference (TEST INFRASTRUCTURE).

Paper passages followed (PAPER.md = /root/reference/PAPER.md, LaTeX of
arxiv 2605.18739):

* PAPER.md:81-86 (§2.2, Eq. 2): ``X^ = X^FP4 * alpha^FP8 * alpha^FP32`` with
  X^FP4 in E2M1, alpha^FP8 an E4M3 scale per 16-element block, alpha^FP32 a
  tensor-wise FP32 scale.
* ``M^FP8 = 448`` (max E4M3), ``M^FP4 = 6`` (max E2M1).
  Eq. 3 itself is missing from the text (reading Z1 in DESIGN.md):
  alpha^FP32 = amax / (M^FP8 * M^FP4) = amax / 2688.
* PAPER.md:719 (App. F): the E2M1 value set {0, +-0.5, +-1, +-1.5, +-2, +-3,
  +-4, +-6}.
* PAPER.md:723-727 (App. F): U_bar = U / alpha^FP32 and the standard block
  scale alpha_i(6) = cast_E4M3(max|U_bar_Bi| / 6).
* PAPER.md:134-139 (§3.2): a KV chunk K_{l,c} in R^{T_c x H x d} is reshaped
  to (T_c H) x d and quantized independently (one alpha^FP32 per tensor,
  blocks of 16 along d).

Readings where the paper is silent: rounding is
round-to-nearest-even everywhere (Z3); the fp32 operation order is
definition R1 (Z4):

    g    = RN32(amax / 2688)                 (amax = 0 -> g = 1)
    t    = RN32(bmax / g)                    (= max|U_bar_Bi| materialised in fp32)
    u    = RN32(t / 6)
    s    = E4M3_RNE_SAT(u)                   (zero block -> 0; s = 0 with bmax > 0 -> 2^-9)
    d_b  = RN32(dec(s) * g)                  (the decode scale Eq. 2 multiplies by)
    c    = E2M1_RNE_SAT(RN32(x / d_b))       (sign from x; zero block -> code 0)

RN32(a op b) is evaluated as an IEEE float64 operation on float32 operands
followed by one rounding to float32.  For + - * / this equals the correctly
rounded float32 result because 53 >= 2*24 + 2 (double rounding is innocuous).
A fused multiply-add RN32(a*b + c) is evaluated exactly (``_rn32_fma``: the
product is exact in float64, TwoSum gives the exact sum as s + e, and the one
rounding to float32 is decided from s and the sign of e).

Optional modes of §8(f) (off on the north_star path):

* Four-Over-Six block-scale search (App. F Eq. 4o6; applied
  to KV by PAPER.md:146 "the same adaptive scale selection"): both candidates
  alpha_i(6) and alpha_i(4) = cast_E4M3(max|U_bar|/4) are formed as in R1
  (u_k = RN32(t / k)); each block is quantized and dequantized with both and
  the one with the lower squared reconstruction error wins, ties to 6
  (SPEC.md:155, 192).  Reading Z21: the error is the float32 quantity the
  kernel computes -- r_i = RN32(x_i - dec(c_i) dec(s) g) (one rounding, an
  FMA), E = RN32(A + B) with A (B) the FMA chain a <- RN32(r_i^2 + a) over the
  even (odd) elements in ascending order -- so both sides take the decision
  in the same precision.
* K-smoothing (§3.2): K_bar[t,h,:] = K[t,h,:] - mean_u
  K[t,h,u], keys only.  Reading Z20: the mean is the float32 sum in a fixed
  tree order (``row_sum_fp32``) times 1/d, K_bar = RN32(K - m), and the mean
  is stored per (t, h) row as float32 and restored on dequantization
  (K^ = dequant(K_bar) + m; the paper is silent on restitution).

Parity pins: tests/test_oracle_nvfp4.py.
"""
from __future__ import annotations

import numpy as np

# magnitudes of E2M1 codes 0..7 (bits S E1 E0 M; code 8+k = -value(k)).
E2M1_MAGNITUDES = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0], dtype=np.float64)
M_FP8 = 448.0
M_FP4 = 6.0
BLOCK = 16      # PAPER.md:84 "block-wise (16 elements) scale"


def _rn32(x):
    """Round float64 values to the nearest float32 (ties to even), keep subnormals."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def _rn32_fma(a, b, c):
    """RN32(a * b + c) with one rounding (an IEEE float32 FMA), for float32-valued inputs
    whose product a*b is exact in float64 (<= 53 significant bits).

    s = RN64(p + c) and e = (p + c) - s exactly (TwoSum); RN32(s + e) = RN32(s) unless s is
    exactly halfway between two float32 neighbours, in which case the sign of e decides.
    """
    a, b, c = (np.asarray(v, dtype=np.float64) for v in (a, b, c))
    p = a * b
    s = p + c
    bb = s - p
    e = (p - (s - bb)) + (c - bb)
    r = s.astype(np.float32)
    rf = r.astype(np.float64)
    # neighbour on the other side of s
    toward = np.where(s > rf, np.float32(np.inf), np.float32(-np.inf)).astype(np.float32)
    other = np.nextafter(r, toward).astype(np.float64)
    mid = (rf + other) * 0.5
    is_mid = (s != rf) & (s == mid) & (e != 0)
    # at a midpoint s + e lies on the side of e: pick the neighbour in that direction
    up = e > 0
    pick_other = is_mid & (up == (other > rf))
    out = np.where(pick_other, other, rf)
    # exact midpoint with e == 0: float64 -> float32 conversion already rounds ties to even
    return out


# ----------------------------------------------------------------------------- E2M1
def e2m1_decode(codes):
    """Decode 4-bit E2M1 codes to float64 (code 8 = -0 decodes to 0.0)."""
    codes = np.asarray(codes, dtype=np.int64)
    mag = E2M1_MAGNITUDES[codes & 7]
    return np.where(codes & 8, -mag, mag)


def e2m1_encode(x):
    """Round-to-nearest-even onto the E2M1 set with saturation at +-6 (reading Z3, Z7).

    Brute force: distance to each of the 8 magnitudes; among equally near
    magnitudes the one whose code has mantissa bit 0 (even code) wins.  Values
    beyond 6 are nearer to 6 than to any other magnitude, so saturation falls
    out of the nearest rule (clamped first so huge inputs keep exact distances).  Sign bit = signbit(x) (reading Z6: -0.0 and
    negatives that round to 0 give code 8).
    """
    x = np.asarray(x, dtype=np.float64)
    flat = x.reshape(-1)
    out = np.empty(flat.shape, dtype=np.uint8)
    even = (np.arange(8) % 2) == 0
    step = 1 << 20                                           # bounds memory only
    for i in range(0, flat.size, step):
        xs = flat[i:i + step]
        a = np.minimum(np.abs(xs), M_FP4)[:, None]           # saturation: RNE(|x| > 6) -> 6
        dist = np.abs(a - E2M1_MAGNITUDES)                   # [n, 8], exact in f64
        is_best = dist == dist.min(axis=-1, keepdims=True)
        # prefer the even code among ties; otherwise the unique nearest
        choose_even = (is_best & even).any(axis=-1)
        mag_code = np.where(choose_even, np.argmax(is_best & even, axis=-1), np.argmax(is_best, axis=-1))
        out[i:i + step] = mag_code + 8 * np.signbit(xs)
    return out.reshape(x.shape)


# ----------------------------------------------------------------------------- E4M3
def _e4m3_table():
    """Values of the 256 E4M3 bit patterns (bias 7, subnormals m*2^-9, 0x7F/0xFF NaN)."""
    vals = np.empty(256, dtype=np.float64)
    for b in range(256):
        s, e, m = b >> 7, (b >> 3) & 0xF, b & 7
        if e == 0xF and m == 7:
            v = np.nan
        elif e == 0:
            v = m * 2.0 ** -9
        else:
            v = (1.0 + m / 8.0) * 2.0 ** (e - 7)
        vals[b] = -v if s else v
    return vals


E4M3_VALUES = _e4m3_table()
_E4M3_POS = E4M3_VALUES[:0x7F]          # codes 0x00..0x7E: the 127 finite non-negative values


def e4m3_decode(codes):
    """Decode E4M3 bytes to float64 (max 448 = 0x7E)."""
    return E4M3_VALUES[np.asarray(codes, dtype=np.int64)]


def e4m3_encode_nonneg(u):
    """RNE of non-negative values onto the finite E4M3 grid, saturating at 448 (0x7E).

    Brute force over the 127 finite non-negative codes; ties go to the code
    with mantissa LSB 0 (the even code).  Values above 448 are nearest to 448.
    """
    u = np.minimum(np.asarray(u, dtype=np.float64), M_FP8)   # saturation: RNE(u > 448) -> 448
    flat = u.reshape(-1)
    out = np.empty(flat.shape, dtype=np.uint8)
    # chunked to bound memory: distance matrix [n, 127]
    step = 1 << 16
    for i in range(0, flat.size, step):
        a = flat[i:i + step, None]
        dist = np.abs(a - _E4M3_POS)
        best = dist.min(axis=-1, keepdims=True)
        is_best = dist == best
        even = (np.arange(0x7F) % 2) == 0
        choose_even = (is_best & even).any(axis=-1)
        idx = np.where(choose_even, np.argmax(is_best & even, axis=-1), np.argmax(is_best, axis=-1))
        out[i:i + step] = idx
    return out.reshape(u.shape)


# ----------------------------------------------------------------------------- quantize
def tensor_scale(x):
    """alpha^FP32 = RN32(amax / (M^FP8 * M^FP4)); amax = 0 -> 1 (readings Z1, Z5).

    ``x`` holds the exact input values (bf16 or fp32 widened to float64).
    Raises ValueError on non-finite input (SPEC.md:138 convention).
    """
    x = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(x)):
        bad = int(np.flatnonzero(~np.isfinite(x.reshape(-1)))[0])
        raise ValueError(f"non-finite input at flat index {bad}")
    amax = float(np.max(np.abs(x))) if x.size else 0.0
    if amax == 0.0:
        return 1.0
    return float(_rn32(amax / (M_FP8 * M_FP4)))


def _block_scales(bmax, t, g, target):
    """R1 block scale for max target `target` (6 standard, 4 the Four-Over-Six candidate):
    s = E4M3_RNE_SAT(RN32(t / target)), zero block -> 0, underflow -> 2^-9; d_b = RN32(dec(s) g)."""
    u = _rn32(t / target)
    s = e4m3_encode_nonneg(u)                            # cast_E4M3 (RNE, saturating)
    s = np.where((s == 0) & (bmax > 0), np.uint8(1), s)  # underflow promotion (Z5)
    s = np.where(bmax == 0, np.uint8(0), s)              # zero block (Z5)
    d_b = _rn32(e4m3_decode(s) * g)                      # decode scale of Eq. 2 (exact product, one rounding)
    return s.astype(np.uint8), d_b


def _block_codes(xb, bmax, d_b):
    """c = E2M1_RNE_SAT(RN32(x / d_b)); zero block -> 0x00 (Z6 exception)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        q = _rn32(xb / d_b[..., None])
    q = np.where(bmax[..., None] == 0, 0.0, q)
    c = e2m1_encode(q)
    return np.where(bmax[..., None] == 0, np.uint8(0), c).astype(np.uint8)


def block_sse_fp32(xb, c, s, g):
    """Squared reconstruction error of each 16-element block in float32 (reading Z21):
    r_i = RN32(x_i - dec(c_i) dec(s) g); A = FMA chain over even i, B over odd i (ascending),
    E = RN32(A + B).  dec(c) dec(s) is exact (<= 6 significant bits) and its product with g
    is exact in float64, so r_i is one FMA rounding."""
    v = e2m1_decode(c) * e4m3_decode(s)[..., None]            # exact
    r = _rn32_fma(-v, g, xb)                                  # [..., 16]
    acc = [np.zeros(xb.shape[:-1]), np.zeros(xb.shape[:-1])]
    for i in range(BLOCK):
        acc[i & 1] = _rn32_fma(r[..., i], r[..., i], acc[i & 1])
    return _rn32(acc[0] + acc[1])


def quantize(x, scale_search=False):
    """NVFP4-quantize a (rows, d) tensor along its last axis.

    Returns (codes uint8 [rows, d] of 4-bit values, scales uint8 [rows, d/16]
    of E4M3 bytes, g float) following definition R1 (module docstring).  With
    ``scale_search`` each block takes the Four-Over-Six choice (Eq. 4o6,
    PAPER.md:728-739): the 4-target scale when its float32 error is strictly lower.
    """
    x = np.asarray(x, dtype=np.float64)
    rows, d = x.shape
    assert d % BLOCK == 0
    g = tensor_scale(x)
    xb = x.reshape(rows, d // BLOCK, BLOCK)
    bmax = np.abs(xb).max(axis=-1)                       # [rows, nb], exact
    t = _rn32(bmax / g)                                  # U_bar block max in fp32
    s, d_b = _block_scales(bmax, t, g, M_FP4)            # alpha_i(6)
    c = _block_codes(xb, bmax, d_b)
    if scale_search:
        s4, d_b4 = _block_scales(bmax, t, g, 4.0)        # alpha_i(4)
        c4 = _block_codes(xb, bmax, d_b4)
        pick4 = block_sse_fp32(xb, c4, s4, g) < block_sse_fp32(xb, c, s, g)   # ties -> 6
        s = np.where(pick4, s4, s)
        c = np.where(pick4[..., None], c4, c)
    return c.reshape(rows, d).astype(np.uint8), s.astype(np.uint8), g


def row_sum_fp32(x):
    """float32 sum of each row of a (rows, d) float32-valued array in the fixed tree order of
    reading Z20: per 16-element block, y_k = x_k + x_{k+8} (k < 8), z_k = y_k + y_{k+4} (k < 4),
    w_k = z_k + z_{k+2} (k < 2), S = w_0 + w_1; then over the d/16 block sums, adjacent pairs
    level by level: ((S_0 + S_1) + (S_2 + S_3)) + ((S_4 + S_5) + (S_6 + S_7)).  Every + is RN32."""
    x = np.asarray(x, dtype=np.float64)
    rows, d = x.shape
    v = x.reshape(rows, d // BLOCK, BLOCK)
    n = BLOCK
    while n > 1:                                          # halves: element k + element k + n/2
        n //= 2
        v = _rn32(v[..., :n] + v[..., n:2 * n])
    S = v[..., 0]                                         # [rows, nb]
    while S.shape[-1] > 1:                                # adjacent pairs
        S = _rn32(S[..., 0::2] + S[..., 1::2])
    return S[..., 0]


def k_smooth(x):
    """K-smoothing: K_bar = K - (1/d) sum_u K[., u] per row.
    Returns (K_bar, mean) with mean = RN32(row_sum_fp32 / d) and K_bar = RN32(K - mean)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[1]
    mean = _rn32(row_sum_fp32(x) / d)
    return _rn32(x - mean[:, None]), mean


def dequantize(codes, scales, g):
    """Eq. 2: x^ = dec(c) * dec(s) * g, exact in float64 (<= 30 significant bits)."""
    codes = np.asarray(codes)
    rows, d = codes.shape
    blk = e4m3_decode(scales).reshape(rows, d // BLOCK, 1)
    val = e2m1_decode(codes).reshape(rows, d // BLOCK, BLOCK)
    return (val * blk * np.float64(g)).reshape(rows, d)


def pack_codes(codes):
    """Two codes per byte, element 2k in the low nibble (reading Z8)."""
    codes = np.asarray(codes, dtype=np.uint8)
    return (codes[..., 0::2] | (codes[..., 1::2] << 4)).astype(np.uint8)


def unpack_codes(packed):
    packed = np.asarray(packed, dtype=np.uint8)
    out = np.empty(packed.shape[:-1] + (packed.shape[-1] * 2,), dtype=np.uint8)
    out[..., 0::2] = packed & 0xF
    out[..., 1::2] = packed >> 4
    return out


def quantize_kv_chunk(kv, scale_search=False, smooth=False):
    """Quantize one KV chunk tensor [T_c, H, d] as (T_c H) x d.

    Returns dict(codes=[T_c*H, d/2] packed bytes, scales=[T_c*H, d/16], g=float),
    rows in (t, h) t-major order -- the canonical export layout.  ``smooth`` (keys,
    PAPER.md:139-145) quantizes K_bar and adds mean=[T_c*H] float32 row means;
    ``scale_search`` selects Four-Over-Six block scales.
    """
    kv = np.asarray(kv, dtype=np.float64)
    T, H, d = kv.shape
    x = kv.reshape(T * H, d)
    out = {}
    if smooth:
        x, out["mean"] = k_smooth(x)
    c, s, g = quantize(x, scale_search)
    out.update(codes=pack_codes(c), scales=s, g=g)
    return out


def dequantize_kv_chunk(q, T, H, d):
    """Inverse of quantize_kv_chunk in float64: [T_c, H, d] (exact values; with a stored
    K-smoothing mean, K^ = dequant(K_bar) + mean)."""
    x = dequantize(unpack_codes(q["codes"]), q["scales"], q["g"])
    if "mean" in q:
        x = x + np.asarray(q["mean"], dtype=np.float64)[:, None]
    return x.reshape(T, H, d)


def dequantize_kv_chunk_rn32(q, T, H, d):
    """The float32 value kv_dequantize returns: RN32(dec(c) dec(s) g [+ mean]) with one rounding."""
    codes = unpack_codes(q["codes"])
    rows = T * H
    v = (e2m1_decode(codes).reshape(rows, d // BLOCK, BLOCK) * e4m3_decode(q["scales"])[..., None]).reshape(rows, d)
    # without a mean the addend is -0.0, the additive identity: RN32(v g + -0) = RN32(v g) keeps Eq. 2's
    # sign of zero (code 0x8 decodes to -0.0 * s * g = -0.0, reading Z6)
    mean = np.asarray(q["mean"], dtype=np.float64)[:, None] if "mean" in q else np.full((rows, 1), -0.0)
    return _rn32_fma(v, q["g"], mean).reshape(T, H, d)


def storage_bytes(T, H, d):
    """NVFP4 bytes of one K+V chunk: codes d/2 + scales d/16 per row, + 4 B g per tensor
    (4 T_c H d -> 9/8 T_c H d bytes, ignoring the tensor scale)."""
    rows = T * H
    return 2 * (rows * d // 2 + rows * d // BLOCK + 4)
