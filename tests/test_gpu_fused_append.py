"""chunk_attention_append (the append fused into the attention launch) vs the float64 oracle (-m gpu).

The bar is the same as the separate calls': the cache bytes of every appended chunk bit-exact to the
oracle's quantizer (reading Z4 definition R1), attention in the fp32-out mode within max-abs 2e-3 and
rel-L2 1e-3 of the oracle (north_star).  Cases: a rollout whose early chunks take the fallback (the new
chunk is more than half of K_eff) and whose later ones fuse, a denoising re-write of the newest chunk,
graph replay of one fused call (the device-side launch epoch), fp32 K/V input, the Wan shape in the
bench's launch configuration (every row and head), and a non-finite K element.
"""
import numpy as np
import pytest
import torch

from oracle import nvfp4
from oracle.cache import OracleKVCache
from paper_2605_18739_b200 import kvq, synth

from gpu_util import assert_chunk_bytes_equal, check_fp32_out

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(autouse=True)
def _fused_on(monkeypatch):
    # the fused launch is opt-in (kvq.h): every test here runs it
    monkeypatch.setenv("KVQ_FUSED_APPEND", "1")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_fused_append_rollout_matches_oracle(dtype):
    # H = 4, d = 128, 3 frames x 256 tokens per chunk, 3-frame sink + 12-frame window: chunks 0, 1 fall
    # back (the new chunk is > half of the keys), chunks 2.. are fused; chunk 4 is re-written (a denoising
    # step) before chunk 5.  Every step: codes/scales/g bit-exact, O (fp32) within the oracle bar.
    _need_gpu()
    H, d, tpf, fc = 4, 128, 256, 3
    T = tpf * fc
    c = kvq.KVCache(1, H, d, tpf, fc, sink_frames=3, window_frames=12, max_chunk_slots=6, device=DEV)
    o = OracleKVCache(1, H, d, tpf, fc)
    ws = c.new_attention_workspace()
    steps = [0, 1, 2, 3, 4, 4, 5, 6]
    for i, ch in enumerate(steps):
        q, k, v = synth.make_qkv(T, H, d, dtype, 7, 10 * ch + i, variant="outlier" if i % 3 == 1 else "iid")
        Q = q.torch(DEV).to(torch.bfloat16) if dtype == "fp32" else q.torch(DEV)
        qf = synth.Tensor(Q.float().cpu().numpy().astype(np.float64), "fp32").f64
        m = kvq.Mask(ch, 3, 12)
        O = c.append_attention(0, ch, k.torch(DEV), v.torch(DEV), Q, m, torch.float32,
                               workspace=ws if i % 2 else None).cpu().numpy()
        o.append(0, ch, k.f64, v.f64)
        assert c.status() == (0, -1)
        assert_chunk_bytes_equal(c.export(0, ch), nvfp4.quantize_kv_chunk(k.f64), nvfp4.quantize_kv_chunk(v.f64))
        check_fp32_out(O, o.attend(0, ch, qf, 3, 12))


def test_fused_append_graph_replay():
    # one fused call captured in a CUDA graph and replayed with new K/V: the amax exchange between CTAs
    # is tagged with a launch epoch kept on the device, so a replay never reads a previous launch's tags
    _need_gpu()
    H, d, tpf, fc = 4, 128, 256, 3
    T = tpf * fc
    c = kvq.KVCache(1, H, d, tpf, fc, sink_frames=3, window_frames=12, max_chunk_slots=6, device=DEV)
    for ch in range(3):
        _, k, v = synth.make_qkv(T, H, d, "bf16", 1, ch)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
    q, k, v = synth.make_qkv(T, H, d, "bf16", 1, 3)
    Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
    O = torch.empty((T, H, d), dtype=torch.float32, device=DEV)
    m = kvq.Mask(3, 3, 12)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        c.append_attention(0, 3, K, V, Q, m, out=O)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        c.append_attention(0, 3, K, V, Q, m, out=O)
    ref = kvq.KVCache(1, H, d, tpf, fc, sink_frames=3, window_frames=12, max_chunk_slots=6, device=DEV)
    for ch in range(3):
        _, k0, v0 = synth.make_qkv(T, H, d, "bf16", 1, ch)
        ref.append(0, ch, k0.torch(DEV), v0.torch(DEV))
    for rep in range(4):
        _, k2, v2 = synth.make_qkv(T, H, d, "bf16", 2, rep, variant="outlier" if rep % 2 else "iid")
        K.copy_(k2.torch(DEV))
        V.copy_(v2.torch(DEV))
        g.replay()
        torch.cuda.synchronize()
        assert_chunk_bytes_equal(c.export(0, 3), nvfp4.quantize_kv_chunk(k2.f64), nvfp4.quantize_kv_chunk(v2.f64))
        ref.append(0, 3, K, V)
        O_ref = ref.attention(0, Q, m, torch.float32)
        assert torch.allclose(O, O_ref, rtol=1e-3, atol=2e-4)


def test_fused_append_wan_layer_every_row():
    # the bench's step (chunk 6 of the Wan layer, 32,760 keys, persistent grid of 148 CTAs) as one fused
    # launch: bytes bit-exact, every row and head of O within the oracle bar
    _need_gpu()
    T, H, d, tpf, fc = 4680, 12, 128, 1560, 3
    c = kvq.KVCache(1, H, d, tpf, fc, sink_frames=3, window_frames=21, max_chunk_slots=8, device=DEV)
    o = OracleKVCache(1, H, d, tpf, fc)
    for ch in range(6):
        _, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
        o.append(0, ch, k.f64, v.f64)
    q, k, v = synth.make_qkv(T, H, d, "bf16", 0, 6)
    m = kvq.Mask(6, 3, 21)
    O = c.append_attention(0, 6, k.torch(DEV), v.torch(DEV), q.torch(DEV), m, torch.float32).cpu().numpy()
    o.append(0, 6, k.f64, v.f64)
    assert c.status() == (0, -1)
    assert_chunk_bytes_equal(c.export(0, 6), nvfp4.quantize_kv_chunk(k.f64), nvfp4.quantize_kv_chunk(v.f64))
    check_fp32_out(O, o.attend(0, 6, q.f64, 3, 21))


def test_fused_append_reports_nonfinite():
    _need_gpu()
    H, d, tpf, fc = 4, 128, 256, 3
    T = tpf * fc
    c = kvq.KVCache(1, H, d, tpf, fc, sink_frames=3, window_frames=12, max_chunk_slots=6, device=DEV)
    for ch in range(3):
        _, k, v = synth.make_qkv(T, H, d, "bf16", 3, ch)
        c.append(0, ch, k.torch(DEV), v.torch(DEV))
    q, k, v = synth.make_qkv(T, H, d, "bf16", 3, 3)
    K = k.torch(DEV).clone()
    K[100, 2, 17] = float("nan")
    c.append_attention(0, 3, K, v.torch(DEV), q.torch(DEV), kvq.Mask(3, 3, 12))
    code, idx = c.status()
    assert code == -6 and idx == (100 * H + 2) * d + 17        # KVQ_ENONFINITE, flat index into K


def test_append_attention_default_two_launches(monkeypatch):
    # without the opt-in the call runs kv_quantize_append + chunk_attention: same bytes, same bar
    _need_gpu()
    monkeypatch.delenv("KVQ_FUSED_APPEND", raising=False)
    H, d, tpf, fc = 4, 128, 256, 3
    T = tpf * fc
    c = kvq.KVCache(1, H, d, tpf, fc, sink_frames=3, window_frames=12, max_chunk_slots=6, device=DEV)
    o = OracleKVCache(1, H, d, tpf, fc)
    for ch in range(4):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 4, ch)
        m = kvq.Mask(ch, 3, 12)
        O = c.append_attention(0, ch, k.torch(DEV), v.torch(DEV), q.torch(DEV), m, torch.float32).cpu().numpy()
        o.append(0, ch, k.f64, v.f64)
        assert_chunk_bytes_equal(c.export(0, ch), nvfp4.quantize_kv_chunk(k.f64), nvfp4.quantize_kv_chunk(v.f64))
        check_fp32_out(O, o.attend(0, ch, q.f64, 3, 12))
