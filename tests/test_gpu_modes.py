"""§8(f) modes on the CUDA path vs the float64 oracle, through the C ABI (-m gpu):
Four-Over-Six block-scale search and K-smoothing with mean restitution
(PAPER.md:139-145), separately and together.

Bar: codes, scales, tensor scales and the stored K row means bit-exact (the oracle takes the 4/6
decision in the kernel's float32 order, reading Z21, and the mean in the fixed float32 tree order,
reading Z20); kv_dequantize bit-exact; attention within the north_star tolerance (fp32-out) and
the bf16 check of reading Z17.  Keys carry per-row offsets (the structure smoothing targets).
"""
import numpy as np
import pytest
import torch

from oracle import nvfp4
from oracle.cache import OracleKVCache
from paper_2605_18739_b200 import kvq, synth

from gpu_util import assert_chunk_bytes_equal, check_bf16_out, check_fp32_out

pytestmark = pytest.mark.gpu
DEV = "cuda"
MODES = [(True, False), (False, True), (True, True)]   # (scale_search, k_smoothing)
ATT_MODES = [(False, False)] + MODES                    # attention: the plain path on the same keys too


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _offset_k(k, layer, chunk, scale=1.5):
    """K + a per-(t, h) row offset, re-rounded to the input dtype (the same bytes on both sides)."""
    T, H, _ = k.shape
    off = synth.make_tensor((T, H, 1), "fp32", seed=0x5EED ^ (layer << 20) ^ chunk).f64 * scale
    return synth.Tensor(k.f64 + off, k.dtype)


def _qkv(T, H, d, dtype, layer, chunk, variant="iid"):
    q, k, v = synth.make_qkv(T, H, d, dtype, layer, chunk, variant=variant)
    return q, _offset_k(k, layer, chunk), v


def _cache(H, d, tpf, fc, search, smooth, sink=0, window=None, slots=8, layers=1):
    return kvq.KVCache(layers, H, d, tpf, fc, sink_frames=sink, window_frames=window or slots * fc,
                       max_chunk_slots=slots, device=DEV, scale_search=search, k_smoothing=smooth)


def _check_chunk(c, layer, chunk, k, v, search, smooth):
    T, H, d = k.shape
    qk = nvfp4.quantize_kv_chunk(k.f64, search, smooth=smooth)
    qv = nvfp4.quantize_kv_chunk(v.f64, search)
    assert_chunk_bytes_equal(c.export(layer, chunk), qk, qv)
    if smooth:
        got = c.export_kmean(layer, chunk).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), qk["mean"].astype(np.float32).view(np.uint32))
    return qk, qv


@pytest.mark.parametrize("search,smooth", MODES)
@pytest.mark.parametrize("two_pass", [False, True])
def test_modes_quantize_bitexact(search, smooth, two_pass):
    _gpu()
    T, H, d = 1560, 12, 128
    c = _cache(H, d, 1560, 1, search, smooth)
    c.force_two_pass(two_pass)
    for ch in range(2):
        _, k, v = _qkv(T, H, d, "bf16", 0, ch, variant="outlier" if ch else "iid")
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        _check_chunk(c, 0, ch, k, v, search, smooth)


@pytest.mark.parametrize("search,smooth", MODES)
def test_modes_quantize_fp32_d64_and_scales(search, smooth):
    _gpu()
    T, H, d = 192, 3, 64
    c = _cache(H, d, 64, 3, search, smooth)
    for i, scale in enumerate((1.0, 1e-3, 300.0)):
        _, k, v = _qkv(T, H, d, "fp32", 1, i)
        k = synth.Tensor(k.f64 * scale, "fp32")
        v = synth.Tensor(v.f64 * scale, "fp32")
        c.append(0, i, k.torch(DEV), v.torch(DEV))
        _check_chunk(c, 0, i, k, v, search, smooth)


def test_modes_quantize_wan_chunk_bitexact():
    _gpu()
    T, H, d = 4680, 12, 128
    c = _cache(H, d, 1560, 3, True, True)
    _, k, v = _qkv(T, H, d, "bf16", 5, 9)
    c.append(0, 0, k.torch(DEV), v.torch(DEV))
    _check_chunk(c, 0, 0, k, v, True, True)


def test_smoothing_constant_rows_and_edges():
    # constant key rows -> zero K_bar blocks (scale 0), means = the constants
    _gpu()
    T, H, d = 64, 2, 64
    c = _cache(H, d, 64, 1, True, True)
    k = np.repeat(synth.make_tensor((T, H, 1), "bf16", seed=3).f64, d, axis=2)
    k[5, 1, :] = 0.0
    kt = synth.Tensor(k, "bf16")
    _, _, v = synth.make_qkv(T, H, d, "bf16", 0, 0)
    c.append(0, 0, kt.torch(DEV), v.torch(DEV))
    qk, _ = _check_chunk(c, 0, 0, kt, v, True, True)
    assert qk["g"] == 1.0 and np.all(qk["scales"] == 0)
    K32, _ = c.dequantize(0, 0, torch.float32)
    assert np.array_equal(K32.cpu().numpy(), kt.f64.astype(np.float32))


@pytest.mark.parametrize("search,smooth", MODES)
def test_modes_dequantize_bitexact(search, smooth):
    _gpu()
    T, H, d = 120, 4, 128
    c = _cache(H, d, 40, 3, search, smooth)
    _, k, v = _qkv(T, H, d, "bf16", 0, 4)
    c.append(0, 0, k.torch(DEV), v.torch(DEV))
    K32, V32 = c.dequantize(0, 0, torch.float32)
    refK = nvfp4.dequantize_kv_chunk_rn32(nvfp4.quantize_kv_chunk(k.f64, search, smooth=smooth), T, H, d)
    refV = nvfp4.dequantize_kv_chunk_rn32(nvfp4.quantize_kv_chunk(v.f64, search), T, H, d)
    assert np.array_equal(K32.cpu().numpy(), refK.astype(np.float32))
    assert np.array_equal(V32.cpu().numpy(), refV.astype(np.float32))
    Kb, _ = c.dequantize(0, 0, torch.bfloat16)
    assert torch.equal(Kb.cpu(), torch.from_numpy(refK.astype(np.float32)).to(torch.bfloat16))


def test_smoothing_nonfinite_reported():
    _gpu()
    T, H, d = 64, 2, 64
    c = _cache(H, d, 64, 1, False, True)
    _, k, v = synth.make_qkv(T, H, d, "fp32", 0, 0)
    kk = k.torch(DEV)
    kk.view(-1)[777] = float("nan")
    c.append(0, 0, kk, v.torch(DEV))
    code, idx = c.status()
    assert code == -6 and idx == 777


def _run(T, H, d, tpf, fc, n_chunks, dtype, sink, window, slots, search, smooth, variant="iid"):
    c = _cache(H, d, tpf, fc, search, smooth, sink, window, slots)
    o = OracleKVCache(1, H, d, tpf, fc, scale_search=search, k_smoothing=smooth)
    qs = []
    for ch in range(n_chunks):
        q, k, v = _qkv(T, H, d, dtype, 0, ch, variant=variant)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        o.append(0, ch, k.f64, v.f64)
        qs.append(q)
    return c, o, qs


@pytest.mark.parametrize("search,smooth", ATT_MODES)
@pytest.mark.parametrize("variant", ["iid", "peaked"])
def test_modes_attention_tiny(search, smooth, variant):
    _gpu()
    T, H, d = 64, 2, 64
    c, o, qs = _run(T, H, d, 64, 1, 3, "fp32", 0, 1 << 20, 8, search, smooth, variant)
    for ch in range(3):
        m = kvq.Mask(ch, 0, 1 << 20)
        O32 = c.attention(0, qs[ch].torch(DEV), m, torch.float32).cpu().numpy()
        ref = o.attend(0, ch, qs[ch].f64, 0, 1 << 20)
        check_fp32_out(O32, ref)
        Ob = c.attention(0, qs[ch].torch(DEV), m, torch.bfloat16).float().cpu().numpy()
        check_bf16_out(Ob, ref, O32)


@pytest.mark.parametrize("search,smooth", ATT_MODES)
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_modes_attention_sink_window_ragged_d128(search, smooth, dtype):
    # 50 tokens/frame x 3 -> ragged 150-token chunks; sink 1 frame, window 12 frames (4 chunks); each
    # chunk is attended right after its append (later appends evict the chunks an early mask reaches)
    _gpu()
    T, H, d, tpf, fc = 150, 3, 128, 50, 3
    c = _cache(H, d, tpf, fc, search, smooth, 1, 12, 6)
    o = OracleKVCache(1, H, d, tpf, fc, scale_search=search, k_smoothing=smooth)
    for ch in range(7):
        q, k, v = _qkv(T, H, d, dtype, 0, ch, variant="peaked" if dtype == "fp32" else "iid")
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        o.append(0, ch, k.f64, v.f64)
        if ch in (0, 4, 6):
            m = kvq.Mask(ch, 1, 12)
            O32 = c.attention(0, q.torch(DEV), m, torch.float32).cpu().numpy()
            check_fp32_out(O32, o.attend(0, ch, q.f64, 1, 12))


@pytest.fixture(scope="module")
def wan_layer_modes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    T, H, d, tpf, fc = 4680, 12, 128, 1560, 3
    c = _cache(H, d, tpf, fc, True, True, sink=3, window=21, slots=8)
    o = OracleKVCache(1, H, d, tpf, fc, scale_search=True, k_smoothing=True)
    q = None
    for ch in range(7):
        q, k, v = _qkv(T, H, d, "bf16", 0, ch)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        o.append(0, ch, k.f64, v.f64)
    return c, o, q


ROWS = np.array([0, 127, 128, 2047, 2048, 4095, 4096, 4607, 4608, 4679])


def test_modes_attention_wan_layer_sampled(wan_layer_modes):
    c, o, q = wan_layer_modes
    m = kvq.Mask(6, 3, 21)
    O32 = c.attention(0, q.torch(DEV), m, torch.float32).cpu().numpy()
    ref = o.attend(0, 6, q.f64, 3, 21, rows=ROWS)
    check_fp32_out(O32[ROWS], ref)
    Ob = c.attention(0, q.torch(DEV), m, torch.bfloat16).float().cpu().numpy()
    check_bf16_out(Ob[ROWS], ref, O32[ROWS])


def test_modes_dequantize_window_restores_means(wan_layer_modes):
    c, o, q = wan_layer_modes
    m = kvq.Mask(6, 3, 21)
    Kw, Vw = c.dequantize_window(0, m)
    Kref, Vref = o.keys(0, 6, 3, 21)
    sel = np.array([0, 4679, 4680, 20000, 32759])
    np.testing.assert_allclose(Kw.float().cpu().numpy()[sel], Kref[sel], rtol=2 ** -7, atol=1e-6)
    np.testing.assert_allclose(Vw.float().cpu().numpy()[sel], Vref[sel], rtol=2 ** -7, atol=1e-6)
