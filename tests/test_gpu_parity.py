"""CUDA path vs the float64 oracle, through the C ABI (-m gpu).

Bar (BASELINE.json north_star): codes, scales and tensor scales bit-exact; attention in the
fp32-out parity mode within max-abs 2e-3 and rel-L2 1e-3; bf16 output within 1 bf16 ulp of
RN_bf16(oracle) (reading Z17).  Inputs come from paper_2605_18739_b200.synth (seeded; the
oracle and the GPU consume the same bytes).
"""
import numpy as np
import pytest
import torch

from oracle import nvfp4
from oracle.cache import OracleKVCache
from oracle.keyset import key_token_ranges
from paper_2605_18739_b200 import kvq, synth

from gpu_util import assert_chunk_bytes_equal, check_bf16_out, check_fp32_out

pytestmark = pytest.mark.gpu

DEV = "cuda"


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


# --------------------------------------------------------------------------- codec probes
def test_probe_e2m1_encode_matches_oracle():
    _gpu()
    base = np.concatenate([np.linspace(-8, 8, 400001), np.arange(-7, 7.01, 0.25), [-0.0, 0.0, -1e-30, 1e30, -1e30,
                                                                                   2.0 ** -149, -(2.0 ** -149)]])
    # all fp32 neighbours of every midpoint
    mids = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])
    nb = np.concatenate([np.nextafter(mids.astype(np.float32), np.float32(0)), np.nextafter(mids.astype(np.float32), np.float32(9))])
    x = np.concatenate([base, nb, -nb]).astype(np.float32)
    if x.size % 2:
        x = np.append(x, np.float32(0))
    got = kvq.probe(0, torch.from_numpy(x).to(DEV), x.size // 2).cpu().numpy()
    want = nvfp4.e2m1_encode(x.astype(np.float64))
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]


def test_probe_e4m3_encode_matches_oracle():
    _gpu()
    v = nvfp4.e4m3_decode(np.arange(0x7F))
    mids = (v[1:] + v[:-1]) / 2
    x = np.concatenate([np.linspace(0, 464, 300001), np.exp2(np.linspace(-14, 8.9, 100001)), v, mids,
                        np.nextafter(mids.astype(np.float32), np.float32(0)),
                        np.nextafter(mids.astype(np.float32), np.float32(1000))]).astype(np.float32)
    got = kvq.probe(1, torch.from_numpy(x).to(DEV), x.size).cpu().numpy()
    want = nvfp4.e4m3_encode_nonneg(x.astype(np.float64))
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]


def test_probe_decoders_exhaustive():
    _gpu()
    b = torch.arange(256, dtype=torch.uint8, device=DEV)
    e2 = kvq.probe(2, b, 256).cpu().numpy().reshape(256, 2)
    ref = np.stack([nvfp4.e2m1_decode(np.arange(256) & 0xF), nvfp4.e2m1_decode(np.arange(256) >> 4)], 1)
    assert np.array_equal(e2, ref)   # low nibble first (reading Z8)
    e4 = kvq.probe(3, b, 256).cpu().numpy()
    ref4 = nvfp4.e4m3_decode(np.arange(256))
    ok = ~np.isnan(ref4)
    assert np.array_equal(e4[ok], ref4[ok])


# --------------------------------------------------------------------------- quantize / append
def _cache(H, d, tpf, fc, sink=0, window=None, slots=8, layers=1):
    return kvq.KVCache(layers, H, d, tpf, fc, sink_frames=sink, window_frames=window or slots * fc,
                       max_chunk_slots=slots, device=DEV)


def test_quantize_tiny_bitexact():
    _gpu()
    T, H, d = 64, 2, 64
    c = _cache(H, d, 64, 1)
    for ch in range(3):
        _, k, v = synth.make_qkv(T, H, d, "fp32", 0, ch)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        assert_chunk_bytes_equal(c.export(0, ch), nvfp4.quantize_kv_chunk(k.f64), nvfp4.quantize_kv_chunk(v.f64))


@pytest.mark.parametrize("variant,scale", [("iid", 1.0), ("outlier", 1.0), ("iid", 0.37), ("iid", 45.0),
                                           ("iid", 0.01)])
def test_quantize_wan_shape_bitexact(variant, scale):
    _gpu()
    T, H, d = 4680, 12, 128
    c = _cache(H, d, 1560, 3)
    _, k, v = synth.make_qkv(T, H, d, "bf16", 3, 7, variant=variant)
    if scale != 1.0:
        k = synth.Tensor(k.f64 * scale, "bf16")
        v = synth.Tensor(v.f64 * scale, "bf16")
    c.append(0, 0, k.torch(DEV), v.torch(DEV))
    assert_chunk_bytes_equal(c.export(0, 0), nvfp4.quantize_kv_chunk(k.f64), nvfp4.quantize_kv_chunk(v.f64))


@pytest.mark.parametrize("two_pass", [False, True])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_quantize_single_and_two_pass_bitexact(two_pass, dtype):
    # the cooperative single-pass kernel and the amax + quantize two-launch path give the oracle's bytes
    _gpu()
    T, H, d = 4680, 12, 128
    c = _cache(H, d, 1560, 3)
    c.force_two_pass(two_pass)
    _, k, v = synth.make_qkv(T, H, d, dtype, 1, 2)
    c.append(0, 0, k.torch(DEV), v.torch(DEV))
    assert_chunk_bytes_equal(c.export(0, 0), nvfp4.quantize_kv_chunk(k.f64), nvfp4.quantize_kv_chunk(v.f64))


def test_quantize_lattice_inputs_take_exact_path():
    # inputs on the NVFP4 lattice make every quotient an exact E2M1 value (the fast-divide guard fires
    # for most blocks); codes must still be bit-exact, and re-quantizing the dequantized chunk is the
    # identity (idempotence)
    _gpu()
    T, H, d = 256, 4, 128
    c = _cache(H, d, 256, 1)
    _, k, v = synth.make_qkv(T, H, d, "bf16", 0, 3)
    c.append(0, 0, k.torch(DEV), v.torch(DEV))
    K32, V32 = c.dequantize(0, 0, torch.float32)
    c.append(0, 0, K32.contiguous(), V32.contiguous())      # overwrite with the lattice values
    qk = nvfp4.quantize_kv_chunk(K32.cpu().numpy().astype(np.float64))
    qv = nvfp4.quantize_kv_chunk(V32.cpu().numpy().astype(np.float64))
    assert_chunk_bytes_equal(c.export(0, 0), qk, qv)
    ref = nvfp4.quantize_kv_chunk(k.f64)
    assert np.array_equal(qk["codes"], ref["codes"]) and np.array_equal(qk["scales"], ref["scales"])


def test_quantize_graph_replay_of_one_append_bitexact():
    # one append captured in a CUDA graph and replayed with new inputs: the single-pass kernel's grid
    # barrier must not pass on a previous replay's tags (the launch epoch lives on the device)
    _gpu()
    T, H, d = 1560, 12, 128
    c = _cache(H, d, 1560, 1)
    _, k0, v0 = synth.make_qkv(T, H, d, "bf16", 0, 0)
    K, V = k0.torch(DEV), v0.torch(DEV)
    c.append(0, 0, K, V)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        c.append(0, 0, K, V)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        c.append(0, 0, K, V)
    for rep in range(1, 5):
        _, k, v = synth.make_qkv(T, H, d, "bf16", 0, rep, variant="outlier" if rep % 2 else "iid")
        K.copy_(k.torch(DEV))
        V.copy_(v.torch(DEV))
        g.replay()
        torch.cuda.synchronize()
        assert_chunk_bytes_equal(c.export(0, 0), nvfp4.quantize_kv_chunk(k.f64), nvfp4.quantize_kv_chunk(v.f64))


def test_quantize_edge_blocks_bitexact():
    # zero tensor (g = 1), zero blocks, underflow-promoted scales, -0.0, ragged T_c (not a multiple of 128)
    _gpu()
    T, H, d = 40, 3, 128
    c = _cache(H, d, 40, 1)
    x = synth.make_tensor((T, H, d), "bf16", seed=5).f64
    x[:, :, 16:32] = 0.0
    x[3, 1, 32:48] = x[3, 1, 32:48] * 1e-6
    x[4, 0, 0] = -0.0
    x[7, 2, 5] = 2688.0 * 4
    x = synth.Tensor(x, "bf16").f64
    z = np.zeros((T, H, d))
    c.append(0, 0, synth.Tensor(x, "bf16").torch(DEV), synth.Tensor(z, "bf16").torch(DEV))
    assert_chunk_bytes_equal(c.export(0, 0), nvfp4.quantize_kv_chunk(x), nvfp4.quantize_kv_chunk(z))


def test_dequantize_bitexact():
    _gpu()
    T, H, d = 120, 4, 128
    c = _cache(H, d, 40, 3)
    _, k, v = synth.make_qkv(T, H, d, "bf16", 0, 0)
    c.append(0, 0, k.torch(DEV), v.torch(DEV))
    K32, V32 = c.dequantize(0, 0, torch.float32)
    refK = nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(k.f64), T, H, d)
    refV = nvfp4.dequantize_kv_chunk(nvfp4.quantize_kv_chunk(v.f64), T, H, d)
    assert np.array_equal(K32.cpu().numpy(), refK.astype(np.float32))
    assert np.array_equal(V32.cpu().numpy(), refV.astype(np.float32))
    Kb, _ = c.dequantize(0, 0, torch.bfloat16)
    assert torch.equal(Kb.cpu(), torch.from_numpy(refK.astype(np.float32)).to(torch.bfloat16))


def test_nonfinite_reported():
    _gpu()
    T, H, d = 64, 2, 64
    c = _cache(H, d, 64, 1)
    _, k, v = synth.make_qkv(T, H, d, "fp32", 0, 0)
    kk = k.torch(DEV)
    kk.view(-1)[1234] = float("inf")
    c.append(0, 0, kk, v.torch(DEV))
    code, idx = c.status()
    assert code == -6 and idx == 1234
    assert c.status() == (0, -1)


# --------------------------------------------------------------------------- attention
def _run_chunks(T, H, d, tpf, fc, n_chunks, dtype, sink, window, slots, variant="iid", layers=1):
    c = _cache(H, d, tpf, fc, sink, window, slots, layers)
    o = OracleKVCache(layers, H, d, tpf, fc)
    data = []
    for ch in range(n_chunks):
        q, k, v = synth.make_qkv(T, H, d, dtype, 0, ch, variant=variant)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        o.append(0, ch, k.f64, v.f64)
        data.append(q)
    return c, o, data


def test_attention_tiny_full_window():
    _gpu()
    T, H, d = 64, 2, 64
    c, o, qs = _run_chunks(T, H, d, 64, 1, 3, "fp32", 0, 1 << 20, 8)
    for variant in ("iid",):
        for ch in range(3):
            m = kvq.Mask(ch, 0, 1 << 20)
            O32 = c.attention(0, qs[ch].torch(DEV), m, torch.float32).cpu().numpy()
            ref = o.attend(0, ch, qs[ch].f64, 0, 1 << 20)
            check_fp32_out(O32, ref)
            Ob = c.attention(0, qs[ch].torch(DEV), m, torch.bfloat16).float().cpu().numpy()
            check_bf16_out(Ob, ref, O32)


@pytest.mark.parametrize("variant", ["iid", "peaked", "outlier"])
def test_attention_tiny_variants(variant):
    _gpu()
    T, H, d = 64, 2, 64
    c, o, qs = _run_chunks(T, H, d, 64, 1, 3, "fp32", 0, 1 << 20, 8, variant=variant)
    O32 = c.attention(0, qs[2].torch(DEV), kvq.Mask(2, 0, 1 << 20), torch.float32).cpu().numpy()
    check_fp32_out(O32, o.attend(0, 2, qs[2].f64, 0, 1 << 20))


def test_attention_sink_window_ragged_d128():
    # W30-like mask at small scale: T_c = 120 (ragged vs 128-key tiles), sink 3 frames, window 9 frames
    _gpu()
    T, H, d, tpf, fc = 120, 3, 128, 40, 3
    sink, window = 3, 9
    c = _cache(H, d, tpf, fc, sink, window, 8)
    o = OracleKVCache(1, H, d, tpf, fc)
    for ch in range(9):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        o.append(0, ch, k.f64, v.f64)
        m = kvq.Mask(ch, sink, window)
        O32 = c.attention(0, q.torch(DEV), m, torch.float32).cpu().numpy()
        check_fp32_out(O32, o.attend(0, ch, q.f64, sink, window))
        assert c.resident_chunks(0) <= 8
    # a mask reaching an evicted chunk is refused
    with pytest.raises(kvq.KVQError) as e:
        c.attention(0, q.torch(DEV), kvq.Mask(8, 0, 27), torch.float32)
    assert e.value.code == -4


def test_attention_shot_sink_and_partial_frames():
    # sink of 1 frame (mid-chunk boundary), a shot sink, window not a multiple of the chunk
    _gpu()
    T, H, d, tpf, fc = 96, 2, 64, 32, 3
    c = _cache(H, d, tpf, fc, sink=1, window=7, slots=8)
    o = OracleKVCache(1, H, d, tpf, fc)
    c.set_shot(12, 4)
    for ch in range(10):
        q, k, v = synth.make_qkv(T, H, d, "fp32", 0, ch)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        o.append(0, ch, k.f64, v.f64)
        if ch >= 4:
            m = kvq.Mask(ch, 1, 7, 12, 4)
            O32 = c.attention(0, q.torch(DEV), m, torch.float32).cpu().numpy()
            check_fp32_out(O32, o.attend(0, ch, q.f64, 1, 7, 12, 4))


def test_overwrite_newest_chunk():
    # a denoising step re-writes the in-progress chunk (chunk_index == newest)
    _gpu()
    T, H, d = 64, 2, 64
    c = _cache(H, d, 64, 1)
    _, k, v = synth.make_qkv(T, H, d, "fp32", 0, 0)
    c.append(0, 0, k.torch(DEV), v.torch(DEV))
    _, k2, v2 = synth.make_qkv(T, H, d, "fp32", 0, 5)
    c.append(0, 0, k2.torch(DEV), v2.torch(DEV))
    assert_chunk_bytes_equal(c.export(0, 0), nvfp4.quantize_kv_chunk(k2.f64), nvfp4.quantize_kv_chunk(v2.f64))
    with pytest.raises(kvq.KVQError):
        c.append(0, 2, k.torch(DEV), v.torch(DEV))


@pytest.fixture(scope="module")
def wan_layer():
    """Wan2.1-1.3B-shaped single layer: 12 heads x 128, T_c = 3 x 1560, window 21 frames (7 chunks)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T, H, d, tpf, fc = 4680, 12, 128, 1560, 3
    c = _cache(H, d, tpf, fc, sink=3, window=21, slots=8)
    o = OracleKVCache(1, H, d, tpf, fc)
    q = None
    for ch in range(7):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        o.append(0, ch, k.f64, v.f64)
    return c, o, q


ROWS = np.array([0, 1, 63, 64, 127, 128, 129, 1000, 2047, 2048, 3333, 4095, 4096, 4500, 4607, 4608, 4609, 4679])


@pytest.fixture(scope="module")
def wan_layer_ref(wan_layer):
    """The oracle's O for EVERY query row and head of the Wan layer (float64 BLAS, one head at a time)."""
    c, o, q = wan_layer
    return o.attend(0, 6, q.f64, 3, 21)


def test_attention_wan_layer_full(wan_layer, wan_layer_ref):
    # every one of the 4,680 x 12 x 128 outputs, in the launch configuration bench.py times
    c, o, q = wan_layer
    m = kvq.Mask(6, 3, 21)
    assert c.n_keys(0, m) == 32760
    O32 = c.attention(0, q.torch(DEV), m, torch.float32).cpu().numpy()
    check_fp32_out(O32, wan_layer_ref)
    Ob = c.attention(0, q.torch(DEV), m, torch.bfloat16).float().cpu().numpy()
    check_bf16_out(Ob, wan_layer_ref, O32)


def test_attention_wan_layer_concurrent_streams(wan_layer, wan_layer_ref):
    # two chunk_attention calls in flight at once on two streams, each with its own split-KV workspace
    # (chunk_attention_ws; kvq.h: concurrent readers), against the oracle -- and the cache-owned
    # workspace call on the default stream afterwards
    c, o, q = wan_layer
    m = kvq.Mask(6, 3, 21)
    Q = q.torch(DEV)
    ws = [c.new_attention_workspace() for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [torch.empty(Q.shape, dtype=torch.float32, device=DEV) for _ in range(2)]
    torch.cuda.synchronize()
    for rep in range(3):
        for i in range(2):
            with torch.cuda.stream(streams[i]):
                c.attention(0, Q, m, torch.float32, out=outs[i], workspace=ws[i])
        torch.cuda.synchronize()
        for i in range(2):
            check_fp32_out(outs[i].cpu().numpy(), wan_layer_ref)
    assert torch.equal(outs[0], outs[1])      # deterministic: same inputs, same bits


def test_attention_q_outside_fp16_range(wan_layer, wan_layer_ref):
    # bf16 queries outside fp16's range (|q| up to ~4e6 and 262144, down to ~1e-21, and 70000): the
    # per-row power-of-two scaling keeps them exact in the fp16 MMA.  (a) With a softmax scale of
    # 2^-16/sqrt(d) their scores stay moderate: the rows match the oracle and nothing is reported.
    # (b) At the default scale the scores of rows 0 (x 2^70), 130, 2047 and 4679 reach 2^12 log2
    # units: KVQ_ERANGE at the first such row's first element (reading Z25); other rows unchanged.
    c, o, q = wan_layer
    m = kvq.Mask(6, 3, 21)
    rows = np.array([5, 130, 2047, 4679])
    f = q.f64.copy()
    f[0] *= 2.0 ** 70
    f[5] *= 2.0 ** -70
    f[130] = f[130] / np.abs(f[130]).max() * 70000.0
    f[2047, :, 0] = 65504.0 * 4
    f[4679] *= 2.0 ** 20
    qq = synth.Tensor(f, "bf16")
    assert c.status() == (0, -1)
    sc = 2.0 ** -16 / np.sqrt(128.0)
    O32 = c.attention(0, qq.torch(DEV), m, torch.float32, softmax_scale=sc).cpu().numpy()
    assert c.status() == (-7, 0)                      # row 0 (x 2^70) is out of range even at this scale
    check_fp32_out(O32[rows], o.attend(0, 6, qq.f64, 3, 21, softmax_scale=sc, rows=rows))
    O32 = c.attention(0, qq.torch(DEV), m, torch.float32).cpu().numpy()
    assert c.status() == (-7, 0)                      # KVQ_ERANGE, row 0 head 0 element 0
    assert c.status() == (0, -1)
    keep = np.setdiff1d(np.arange(4680), np.array([0, 5, 130, 2047, 4679]))[::97]
    check_fp32_out(O32[keep], wan_layer_ref[keep])      # the untouched rows are unchanged


def test_attention_q_nonfinite_and_score_overflow_reported(wan_layer):
    c, o, q = wan_layer
    m = kvq.Mask(6, 3, 21)
    H, d = 12, 128
    Qb = q.torch(DEV).clone()
    Qb[17, 3, 5] = float("inf")
    c.attention(0, Qb, m, torch.float32)
    code, idx = c.status()
    assert code == -6 and idx == (17 * H + 3) * d + 5       # KVQ_ENONFINITE, flat index into Q
    # finite fp32 queries whose scores exceed fp32: KVQ_ERANGE at the row's first element
    Qf = q.torch(DEV).float()
    Qf[40, 7, :] = 3.0e38
    c.attention(0, Qf, m, torch.float32)
    code, idx = c.status()
    assert code == -7 and idx == (40 * H + 7) * d
    assert c.status() == (0, -1)


def test_attention_wan_layer_properties(wan_layer):
    # at full size: every output row is a convex combination of V^ rows -> within [min V^, max V^]
    c, o, q = wan_layer
    O = c.attention(0, q.torch(DEV), kvq.Mask(6, 3, 21), torch.float32)
    assert torch.isfinite(O).all()
    Kw, Vw = c.dequantize_window(0, kvq.Mask(6, 3, 21))
    vmin = Vw.float().amin(0)
    vmax = Vw.float().amax(0)
    assert bool((O >= vmin - 1e-3).all()) and bool((O <= vmax + 1e-3).all())


def test_dequantize_window_matches_oracle(wan_layer):
    c, o, q = wan_layer
    Kw, Vw = c.dequantize_window(0, kvq.Mask(6, 3, 21))
    Kr, Vr = o.keys(0, 6, 3, 21)
    idx = np.arange(0, Kr.shape[0], 997)
    assert torch.equal(Kw[idx].cpu(), torch.from_numpy(Kr[idx].astype(np.float32)).to(torch.bfloat16))
    assert torch.equal(Vw[idx].cpu(), torch.from_numpy(Vr[idx].astype(np.float32)).to(torch.bfloat16))


def test_bf16kv_mode_against_oracle():
    # A12 comparison mode: bf16 K/V, bf16 P (documented looser numerics: rel-L2 <= 4e-3)
    _gpu()
    Tq, H, d, N = 300, 2, 128, 700
    Q = synth.make_tensor((Tq, H, d), "bf16", seed=1)
    K = synth.make_tensor((N, H, d), "bf16", seed=2)
    V = synth.make_tensor((N, H, d), "bf16", seed=3)
    O = kvq.chunk_attention_bf16kv(Q.torch(DEV), K.torch(DEV), V.torch(DEV), torch.float32).cpu().numpy()
    from oracle.attention import attention
    ref = attention(Q.f64, K.f64, V.f64)
    err = np.abs(O - ref).max()
    rel = np.linalg.norm(O - ref) / np.linalg.norm(ref)
    assert err < 1e-2 and rel < 4e-3, (err, rel)


@pytest.mark.parametrize("Tq,H,d,N", [(300, 2, 128, 700), (200, 3, 64, 333), (4680, 12, 128, 640)])
def test_bf16kv_ws_persistent_against_oracle(Tq, H, d, N):
    # A12 on the persistent grid (chunk_attention_bf16kv_ws): TMA-landed tiles, ragged key tails (TMA
    # zero fill), d = 64 and 128; the Wan-width case has 228 units > 148 CTAs -> one wave of whole
    # units, the other 80 units split stream-K and merged by combine_kernel.  Every row and head.
    _gpu()
    Q = synth.make_tensor((Tq, H, d), "bf16", seed=11)
    K = synth.make_tensor((N, H, d), "bf16", seed=12)
    V = synth.make_tensor((N, H, d), "bf16", seed=13)
    ws = kvq.new_bf16kv_workspace(d, DEV)
    Qt, Kt, Vt = Q.torch(DEV), K.torch(DEV), V.torch(DEV)
    O = kvq.chunk_attention_bf16kv(Qt, Kt, Vt, torch.float32, workspace=ws).cpu().numpy()
    from oracle.attention import attention
    ref = attention(Q.f64, K.f64, V.f64)
    err = np.abs(O - ref).max()
    rel = np.linalg.norm(O - ref) / np.linalg.norm(ref)
    assert err < 1e-2 and rel < 4e-3, (err, rel)
    # the data-parallel launch (no workspace) computes the same attention
    O1 = kvq.chunk_attention_bf16kv(Qt, Kt, Vt, torch.float32).cpu().numpy()
    assert np.abs(O1 - ref).max() < 1e-2


def test_resident_footprint_ratio():
    # NVFP4 K+V payload vs bf16 -> 32/9 up to the two fp32 tensor scales per chunk
    _gpu()
    T, H, d = 4680, 12, 128
    c = _cache(H, d, 1560, 3)
    _, k, v = synth.make_qkv(T, H, d, "bf16", 0, 0)
    c.append(0, 0, k.torch(DEV), v.torch(DEV))
    nv = c.resident_bytes()
    assert nv == nvfp4.storage_bytes(T, H, d)
    assert abs((4 * T * H * d) / (nv - 8) - 32 / 9) < 1e-12


def test_probe_e2m1_encode_exhaustive_binades():
    # SURVEY.md §4 item 2 (day-1 codec probe): cvt.rn.satfinite.e2m1x2.f32 against the oracle on EVERY
    # fp32 value in [2^-3, 2^3) and its negative (all E2M1 decision boundaries lie there; below is 0,
    # above saturates), 16M values per call
    _gpu()
    bad = 0
    for e in range(-3, 3):
        m = np.arange(1 << 23, dtype=np.uint32)
        for sign in (0, 1):
            bits = (np.uint32(sign << 31) | np.uint32((e + 127) << 23) | m).view(np.float32)
            got = kvq.probe(0, torch.from_numpy(bits).to(DEV), bits.size // 2).cpu().numpy()
            want = nvfp4.e2m1_encode(bits.astype(np.float64))
            bad += int(np.count_nonzero(got != want))
    assert bad == 0


def test_probe_e4m3_encode_near_every_midpoint_and_strided():
    # cvt.rn.satfinite.e4m3x2.f32 against the oracle: +-64 fp32 ulps around every midpoint between
    # adjacent E4M3 values (the only places rounding can go wrong) plus every 16th fp32 pattern in
    # [2^-12, 2^9)
    _gpu()
    v = nvfp4.e4m3_decode(np.arange(0x7F))
    mids = ((v[1:] + v[:-1]) / 2).astype(np.float32)
    near = (mids.view(np.uint32)[:, None].astype(np.int64) + np.arange(-64, 65)[None, :]).reshape(-1)
    strided = np.arange((127 - 12) << 23, (127 + 9) << 23, 16, dtype=np.int64)
    x = np.concatenate([near, strided]).astype(np.uint32).view(np.float32)
    bad = 0
    for i in range(0, x.size, 1 << 24):
        xs = x[i:i + (1 << 24)]
        got = kvq.probe(1, torch.from_numpy(xs.copy()).to(DEV), xs.size).cpu().numpy()
        bad += int(np.count_nonzero(got != nvfp4.e4m3_encode_nonneg(xs.astype(np.float64))))
    assert bad == 0


def test_attention_v2_64key_tiles_wan_layer_sampled():
    # the opt-in 64-key-tile attention (KVQ_ATTN_V2=1, read once per process): run in a subprocess so
    # the default path of this process is untouched; Wan layer, sampled rows vs the oracle
    _gpu()
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, torch
from oracle.cache import OracleKVCache
from paper_2605_18739_b200 import kvq, synth
import sys
sys.path.insert(0, 'tests')
from gpu_util import check_fp32_out, check_bf16_out
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device='cuda')
o = OracleKVCache(1, H, d, 1560, 3)
for ch in range(7):
    q, k, v = synth.make_qkv(T, H, d, 'bf16', 0, ch)
    c.append(0, ch, k.torch('cuda'), v.torch('cuda'))
    o.append(0, ch, k.f64, v.f64)
rows = np.array([0, 127, 128, 2047, 4095, 4607, 4608, 4679])
m = kvq.Mask(6, 3, 21)
O32 = c.attention(0, q.torch('cuda'), m, torch.float32).cpu().numpy()
ref = o.attend(0, 6, q.f64, 3, 21, rows=rows)
check_fp32_out(O32[rows], ref)
Ob = c.attention(0, q.torch('cuda'), m, torch.bfloat16).float().cpu().numpy()
check_bf16_out(Ob[rows], ref, O32[rows])
print('ok')
"""
    env = dict(os.environ, KVQ_ATTN_V2="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
