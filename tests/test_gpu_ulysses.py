"""Head-sharded (Ulysses) path on one GPU, with the all-to-all simulated by byte slicing (-m gpu).

Every rank's compute runs the library kernels (pack, unpack, quantize/append with the
piggybacked global amax, attention, O unpack); only the collective is replaced by the exact byte
movement NCCL's all_to_all_single performs.  Checks (readings Z2/Z18): each rank's cache bytes equal
the 1-GPU cache's bytes for its heads bit-exactly, and the reassembled O matches the oracle within
the fp32 tolerance and the 1-GPU result closely.
"""
import numpy as np
import pytest
import torch

from oracle import nvfp4
from oracle.cache import OracleKVCache
from paper_2605_18739_b200 import kvq, synth

from gpu_util import check_fp32_out

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _a2a(sends, send_sizes, recv_sizes):
    """all_to_all_single semantics: rank p receives, in source order, source r's p-th segment."""
    P = len(sends)
    offs = [np.concatenate([[0], np.cumsum(s)]) for s in send_sizes]
    return [torch.cat([sends[r][int(offs[r][p]):int(offs[r][p]) + send_sizes[r][p]] for r in range(P)])
            for p in range(P)]


@pytest.mark.parametrize("P,H", [(2, 12), (4, 12), (8, 12), (8, 24), (3, 7)])
def test_ulysses_simulated_matches_single_gpu(P, H):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tpf, fc, d = 40, 3, 128
    T = tpf * fc                       # 120 tokens per chunk, divisible by P for P in {2,3,4,8}
    Ts = T // P
    sink, window = 3, 9
    parts = [kvq.head_partition(H, P, r) for r in range(P)]
    caches = [kvq.KVCache(1, h1 - h0, d, tpf, fc, sink_frames=sink, window_frames=window, max_chunk_slots=8,
                          device=DEV) for h0, h1 in parts]
    ref = kvq.KVCache(1, H, d, tpf, fc, sink_frames=sink, window_frames=window, max_chunk_slots=8, device=DEV)
    orc = OracleKVCache(1, H, d, tpf, fc)
    for ch in range(5):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
        Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
        mask = kvq.Mask(ch, sink, window)
        # ---- 1 GPU reference
        ref.append(0, ch, K, V)
        O_ref = ref.attention(0, Q, mask, torch.float32)
        orc.append(0, ch, k.f64, v.f64)
        # ---- P ranks: pack -> all-to-all -> unpack -> append (global amax) -> attention -> a2a -> unpack
        packed = [kvq.ulysses_pack(Q[r * Ts:(r + 1) * Ts].contiguous(), K[r * Ts:(r + 1) * Ts].contiguous(),
                                   V[r * Ts:(r + 1) * Ts].contiguous(), P) for r in range(P)]
        recv = _a2a([s for s, _ in packed], [sz for _, sz in packed], None)
        O_locals = []
        for p, (h0, h1) in enumerate(parts):
            Hr = h1 - h0
            Ql, Kl, Vl, amax = kvq.ulysses_unpack_qkv(recv[p], Ts, Hr, d, P)
            assert torch.equal(Ql, Q[:, h0:h1]) and torch.equal(Kl, K[:, h0:h1]) and torch.equal(Vl, V[:, h0:h1])
            caches[p].append(0, ch, Kl, Vl, amax_kv=amax)
            O_locals.append(caches[p].attention(0, Ql, mask, torch.float32))
        # O return: rank p sends token block r of its O_local to rank r (equal splits)
        o_bytes = [[Ts * (h1 - h0) * d * 4 for _ in range(P)] for h0, h1 in parts]
        o_recv = _a2a([o.view(torch.uint8).reshape(-1) for o in O_locals], o_bytes, None)
        O_full = torch.cat([kvq.ulysses_unpack_o(o_recv[r], Ts, H, d, P, torch.float32) for r in range(P)])
        # ---- codes bit-exact per head (Z18), O close to 1 GPU and within tolerance of the oracle
        ex = ref.export(0, ch)
        for p, (h0, h1) in enumerate(parts):
            e = caches[p].export(0, ch)
            for name in ("codes_k", "scales_k", "codes_v", "scales_v"):
                full = ex[name].view(T, H, -1)[:, h0:h1].reshape(-1, ex[name].shape[1])
                assert torch.equal(e[name], full), (p, name)
            assert torch.equal(e["g_k"], ex["g_k"]) and torch.equal(e["g_v"], ex["g_v"])
        # not bit-identical: the stream-K split points differ, and a split piece rounds P to fp16
        # against its own running max
        assert torch.allclose(O_full, O_ref, rtol=1e-3, atol=2e-4)
        check_fp32_out(O_full.cpu().numpy(), orc.attend(0, ch, q.f64, sink, window))


def test_pack_trailer_carries_shard_amax():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    Ts, H, d, P = 16, 12, 64, 4
    Q, K, V = (synth.make_tensor((Ts, H, d), "bf16", seed=s).torch(DEV) for s in (1, 2, 3))
    send, sizes = kvq.ulysses_pack(Q, K, V, P)
    off = 0
    for p, sz in enumerate(sizes):
        tr = send[off + sz - 16: off + sz].view(torch.float32)
        assert tr[0].item() == K.float().abs().max().item() and tr[1].item() == V.float().abs().max().item()
        off += sz


@pytest.mark.parametrize("P,H,search,smooth", [(2, 12, False, False), (4, 12, False, False), (8, 12, False, False),
                                               (8, 24, False, False), (3, 7, False, False), (4, 12, True, False),
                                               (4, 12, False, True), (8, 12, True, True)])
def test_ulysses_nvfp4_exchange_simulated_matches_single_gpu(P, H, search, smooth):
    # §8(f) f3: K/V cross the all-to-all as NVFP4 bytes quantized on the sender
    # under the all-reduced global amax; each rank's cache must hold exactly the 1-GPU bytes of its heads
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tpf, fc, d = 40, 3, 128
    T = tpf * fc
    Ts = T // P
    sink, window = 3, 9
    parts = [kvq.head_partition(H, P, r) for r in range(P)]
    mk = dict(sink_frames=sink, window_frames=window, max_chunk_slots=8, device=DEV, scale_search=search,
              k_smoothing=smooth)
    caches = [kvq.KVCache(1, h1 - h0, d, tpf, fc, **mk) for h0, h1 in parts]
    ref = kvq.KVCache(1, H, d, tpf, fc, **mk)
    orc = OracleKVCache(1, H, d, tpf, fc, scale_search=search, k_smoothing=smooth)
    for ch in range(5):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch, variant="outlier" if ch % 2 else "iid")
        Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
        mask = kvq.Mask(ch, sink, window)
        ref.append(0, ch, K, V)
        O_ref = ref.attention(0, Q, mask, torch.float32)
        orc.append(0, ch, k.f64, v.f64)
        shards = [tuple(x[r * Ts:(r + 1) * Ts].contiguous() for x in (Q, K, V)) for r in range(P)]
        amax = torch.stack([kvq.ulysses_shard_amax(Kr, Vr, smooth) for _, Kr, Vr in shards]).max(0).values  # all-reduce
        packed = [kvq.ulysses_pack_nvfp4(Qr, Kr, Vr, P, amax, search, smooth) for Qr, Kr, Vr in shards]
        recv = _a2a([sd for sd, _ in packed], [sz for _, sz in packed], None)
        O_locals = []
        for p, (h0, h1) in enumerate(parts):
            Ql = caches[p].append_ulysses_nvfp4(0, ch, recv[p], P, amax)
            assert torch.equal(Ql, Q[:, h0:h1])
            O_locals.append(caches[p].attention(0, Ql, mask, torch.float32))
        o_bytes = [[Ts * (h1 - h0) * d * 4 for _ in range(P)] for h0, h1 in parts]
        o_recv = _a2a([o.view(torch.uint8).reshape(-1) for o in O_locals], o_bytes, None)
        O_full = torch.cat([kvq.ulysses_unpack_o(o_recv[r], Ts, H, d, P, torch.float32) for r in range(P)])
        ex = ref.export(0, ch)
        for p, (h0, h1) in enumerate(parts):
            e = caches[p].export(0, ch)
            for name in ("codes_k", "scales_k", "codes_v", "scales_v"):
                full = ex[name].view(T, H, -1)[:, h0:h1].reshape(-1, ex[name].shape[1])
                assert torch.equal(e[name], full), (p, name)
            assert torch.equal(e["g_k"], ex["g_k"]) and torch.equal(e["g_v"], ex["g_v"])
            if smooth:
                km = ref.export_kmean(0, ch).view(T, H)[:, h0:h1].reshape(-1)
                assert torch.equal(caches[p].export_kmean(0, ch), km)
        assert torch.allclose(O_full, O_ref, rtol=1e-3, atol=2e-4)
        check_fp32_out(O_full.cpu().numpy(), orc.attend(0, ch, q.f64, sink, window))



@pytest.mark.parametrize("P,H,search,smooth", [(2, 12, False, False), (4, 12, False, False), (8, 12, False, False),
                                               (3, 7, False, False), (4, 12, True, True)])
def test_peer_exchange_simulated_matches_single_gpu(P, H, search, smooth):
    # §8(f) f4: the exchange as device-initiated stores/loads into the ranks' windows (peer memory on a
    # multi-GPU box; P windows on one GPU here).  Kernels of all ranks run in phase order on one stream,
    # so every device-side wait is already satisfied when reached.
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tpf, fc, d = 40, 3, 128
    T = tpf * fc
    Ts = T // P
    sink, window = 3, 9
    parts = [kvq.head_partition(H, P, r) for r in range(P)]
    mk = dict(sink_frames=sink, window_frames=window, max_chunk_slots=8, device=DEV, scale_search=search,
              k_smoothing=smooth)
    caches = [kvq.KVCache(1, h1 - h0, d, tpf, fc, **mk) for h0, h1 in parts]
    ref = kvq.KVCache(1, H, d, tpf, fc, **mk)
    orc = OracleKVCache(1, H, d, tpf, fc, scale_search=search, k_smoothing=smooth)
    wb = kvq.peer_window_bytes(T, H, d, P, k_smoothing=smooth)
    wins = [torch.zeros(wb, dtype=torch.uint8, device=DEV) for _ in range(P)]
    ptrs = [w.data_ptr() for w in wins]
    pes = [kvq.PeerExchange(T, H, d, P, r, ptrs, scale_search=search, k_smoothing=smooth) for r in range(P)]
    for ch in range(5):
        ep = ch + 1
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch, variant="outlier" if ch % 2 else "iid")
        Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
        mask = kvq.Mask(ch, sink, window)
        ref.append(0, ch, K, V)
        O_ref = ref.attention(0, Q, mask, torch.float32)
        orc.append(0, ch, k.f64, v.f64)
        shards = [tuple(x[r * Ts:(r + 1) * Ts].contiguous() for x in (Q, K, V)) for r in range(P)]
        for r in range(P):
            pes[r].publish_amax(shards[r][1], shards[r][2], ep)
        for r in range(P):
            pes[r].pack(*shards[r], ep)
        for p, (h0, h1) in enumerate(parts):
            Ql = torch.empty((T, h1 - h0, d), dtype=torch.bfloat16, device=DEV)
            pes[p].append(caches[p], 0, ch, ep, Ql)
            assert torch.equal(Ql, Q[:, h0:h1])
            off = pes[p].o_local(ep) - wins[p].data_ptr()
            O_loc = wins[p][off:off + T * (h1 - h0) * d * 2].view(torch.bfloat16).view(T, h1 - h0, d)
            caches[p].attention(0, Ql, mask, out=O_loc)
        for p in range(P):
            pes[p].signal_o(ep)
        O_full = torch.cat([pes[r].pull_o(ep, torch.empty((Ts, H, d), dtype=torch.bfloat16, device=DEV))
                            for r in range(P)])
        O_ref_b = ref.attention(0, Q, mask, torch.bfloat16)
        ex = ref.export(0, ch)
        for p, (h0, h1) in enumerate(parts):
            e = caches[p].export(0, ch)
            for name in ("codes_k", "scales_k", "codes_v", "scales_v"):
                full = ex[name].view(T, H, -1)[:, h0:h1].reshape(-1, ex[name].shape[1])
                assert torch.equal(e[name], full), (p, name)
            assert torch.equal(e["g_k"], ex["g_k"]) and torch.equal(e["g_v"], ex["g_v"])
        assert torch.allclose(O_full.float(), O_ref_b.float(), rtol=1e-2, atol=2e-3)
        ref_o = orc.attend(0, ch, q.f64, sink, window)
        err = (O_full.float().cpu().numpy() - ref_o)
        assert np.abs(err).max() <= 2e-3 + np.abs(ref_o).max() * 2 ** -8


@pytest.mark.parametrize("P,H,search,smooth,order", [(2, 12, False, False, -1), (4, 12, False, False, 1),
                                                     (8, 12, False, False, -1), (3, 7, False, False, -1),
                                                     (4, 12, True, True, -1)])
def test_peer_direct_concurrent_ranks_match_single_gpu(P, H, search, smooth, order):
    # §8(f) f4 as specified: the pack kernel stores each owner's NVFP4 rows straight into the owner's
    # cache slot and the attention epilogue / combine store O rows straight into the token owner's
    # shard (no scatter, no pull).  The P simulated ranks each run on their OWN stream and are issued
    # rank P-1 first (order = -1), so every device-side wait (mailbox, arrivals, O-ready flags)
    # really blocks on kernels of other streams that are issued later; each rank's O shard, cache
    # bytes, g and K means must equal the single-GPU path's, O within the oracle bar.
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tpf, fc, d = 40, 3, 128
    T = tpf * fc
    Ts = T // P
    sink, window = 3, 9
    parts = [kvq.head_partition(H, P, r) for r in range(P)]
    mk = dict(sink_frames=sink, window_frames=window, max_chunk_slots=8, device=DEV, scale_search=search,
              k_smoothing=smooth)
    caches = [kvq.KVCache(1, h1 - h0, d, tpf, fc, **mk) for h0, h1 in parts]
    ref = kvq.KVCache(1, H, d, tpf, fc, **mk)
    orc = OracleKVCache(1, H, d, tpf, fc, scale_search=search, k_smoothing=smooth)
    wb = kvq.peer_window_bytes(T, H, d, P, k_smoothing=smooth)
    wins = [torch.zeros(wb, dtype=torch.uint8, device=DEV) for _ in range(P)]
    ptrs = [w.data_ptr() for w in wins]
    pes = [kvq.PeerExchange(T, H, d, P, r, ptrs, scale_search=search, k_smoothing=smooth) for r in range(P)]
    for r in range(P):
        pes[r].bind_caches(caches[r], [c.arena.data_ptr() for c in caches])
    streams = [torch.cuda.Stream() for _ in range(P)]
    ranks = list(range(P))[::order]
    # torch's own kernels load lazily too: run the O copy once before any device-side wait is pending
    scratch = torch.zeros((T, H, d), dtype=torch.bfloat16, device=DEV)
    scratch[:Ts].copy_(scratch[Ts:2 * Ts])
    torch.cuda.synchronize()
    for ch in range(5):
        ep = ch + 1
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch, variant="outlier" if ch % 2 else "iid")
        Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
        mask = kvq.Mask(ch, sink, window)
        ref.append(0, ch, K, V)
        orc.append(0, ch, k.f64, v.f64)
        shards = [tuple(x[r * Ts:(r + 1) * Ts].contiguous() for x in (Q, K, V)) for r in range(P)]
        O_full = torch.empty((T, H, d), dtype=torch.bfloat16, device=DEV)
        torch.cuda.synchronize()
        for r in ranks:  # one rank's whole step per stream, issued back to back, no host sync
            with torch.cuda.stream(streams[r]):
                pes[r].publish_amax(shards[r][1], shards[r][2], ep)
                pes[r].append_direct(0, ch, *shards[r], ep)
                pes[r].attention_direct(0, mask, ep)
                ptr = pes[r].wait_o(ep)
                off = ptr - wins[r].data_ptr()
                O_full[r * Ts:(r + 1) * Ts].copy_(wins[r][off:off + Ts * H * d * 2].view(torch.bfloat16).view(Ts, H, d))
        torch.cuda.synchronize()
        ex = ref.export(0, ch)
        for p, (h0, h1) in enumerate(parts):
            e = caches[p].export(0, ch)
            for name in ("codes_k", "scales_k", "codes_v", "scales_v"):
                full = ex[name].view(T, H, -1)[:, h0:h1].reshape(-1, ex[name].shape[1])
                assert torch.equal(e[name], full), (p, name)
            assert torch.equal(e["g_k"], ex["g_k"]) and torch.equal(e["g_v"], ex["g_v"])
            if smooth:
                km = ref.export_kmean(0, ch).view(T, H)[:, h0:h1].reshape(-1)
                assert torch.equal(caches[p].export_kmean(0, ch), km)
        O_ref_b = ref.attention(0, Q, mask, torch.bfloat16)
        assert torch.allclose(O_full.float(), O_ref_b.float(), rtol=1e-2, atol=2e-3)
        ref_o = orc.attend(0, ch, q.f64, sink, window)
        err = (O_full.float().cpu().numpy() - ref_o)
        assert np.abs(err).max() <= 2e-3 + np.abs(ref_o).max() * 2 ** -8


@pytest.mark.parametrize("exchange", ["bf16", "nvfp4", "peer", "nvfp4q"])
def test_ulysses_class_world1_nccl(exchange):
    # The Ulysses orchestration bench.py runs at N > 1 (NCCL all-to-all / all-reduce, torch symmetric
    # memory windows for the peer exchange), exercised end to end with a one-rank NCCL group: the step's
    # O and the cache bytes must equal the plain single-GPU path's
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    import socket

    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        tpf, fc, d, H = 40, 3, 128, 12
        T = tpf * fc
        mk = dict(sink_frames=3, window_frames=9, max_chunk_slots=8, device=DEV)
        c_ref = kvq.KVCache(1, H, d, tpf, fc, **mk)
        arena = None
        if exchange == "peer":  # f4 direct writes the owners' caches: the arena lives in symmetric memory
            import torch.distributed._symmetric_memory as symm_mem
            arena = symm_mem.empty(kvq.cache_bytes(1, H, d, tpf, fc, 3, 9, 8), dtype=torch.uint8, device=DEV)
        c_uly = kvq.KVCache(1, H, d, tpf, fc, arena=arena, **mk)
        uly = kvq.Ulysses(c_uly, H, d, T, 0, 1, nvfp4_kv=exchange == "nvfp4", peer=exchange == "peer",
                          nvfp4_q=exchange == "nvfp4q")
        for ch in range(4):
            q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
            Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
            mask = kvq.Mask(ch, 3, 9)
            c_ref.append(0, ch, K, V)
            O_ref = c_ref.attention(0, Q, mask)
            O = uly.step(0, ch, Q, K, V, mask)
            torch.cuda.synchronize()
            if exchange == "nvfp4q":  # quantized queries: a different result, close to the bf16-Q one
                assert torch.isfinite(O).all() and (O.float() - O_ref.float()).norm() < 0.2 * O_ref.float().norm()
            else:
                assert torch.equal(O, O_ref), (exchange, ch)
            a, b = c_ref.export(0, ch), c_uly.export(0, ch)
            assert all(torch.equal(a[n], b[n]) for n in a), (exchange, ch)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,H", [(2, 12), (4, 12), (3, 7)])
def test_ulysses_nvfp4_q_mode_simulated(P, H):
    # reading Z24: Q cast to NVFP4 before the all-to-all as well.  The receiver's fp16 Q
    # holds dec(c) dec(s) exactly and g_Q the global tensor scale; attention matches the oracle that
    # attends with the dequantized Q; K/V bytes still equal the 1-GPU cache's
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tpf, fc, d = 40, 3, 128
    T = tpf * fc
    Ts = T // P
    sink, window = 3, 9
    parts = [kvq.head_partition(H, P, r) for r in range(P)]
    mk = dict(sink_frames=sink, window_frames=window, max_chunk_slots=8, device=DEV)
    caches = [kvq.KVCache(1, h1 - h0, d, tpf, fc, **mk) for h0, h1 in parts]
    ref = kvq.KVCache(1, H, d, tpf, fc, **mk)
    orc = OracleKVCache(1, H, d, tpf, fc)
    for ch in range(4):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
        Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
        mask = kvq.Mask(ch, sink, window)
        ref.append(0, ch, K, V)
        orc.append(0, ch, k.f64, v.f64)
        shards = [tuple(x[r * Ts:(r + 1) * Ts].contiguous() for x in (Q, K, V)) for r in range(P)]
        amax = torch.stack([kvq.ulysses_shard_amax(Kr, Vr) for _, Kr, Vr in shards]).max(0).values
        amax_q = torch.stack([kvq.ulysses_q_amax(Qr) for Qr, _, _ in shards]).max(0).values
        packed = [kvq.ulysses_pack_nvfp4(Qr, Kr, Vr, P, amax, amax_q=amax_q) for Qr, Kr, Vr in shards]
        recv = _a2a([sd for sd, _ in packed], [sz for _, sz in packed], None)
        qq = nvfp4.quantize_kv_chunk(q.f64)
        q_lat = (nvfp4.e2m1_decode(nvfp4.unpack_codes(qq["codes"])).reshape(T * H, d // 16, 16) *
                 nvfp4.e4m3_decode(qq["scales"])[..., None]).reshape(T, H, d)      # dec(c) dec(s), exact
        O_locals = []
        for p, (h0, h1) in enumerate(parts):
            Q16, gq = caches[p].append_ulysses_nvfp4(0, ch, recv[p], P, amax, amax_q=amax_q)
            assert np.array_equal(Q16.double().cpu().numpy(), q_lat[:, h0:h1])
            assert gq.item() == np.float32(qq["g"])
            O_locals.append(caches[p].attention_qscaled(0, Q16, gq, mask, out_dtype=torch.float32))
        o_bytes = [[Ts * (h1 - h0) * d * 4 for _ in range(P)] for h0, h1 in parts]
        o_recv = _a2a([o.view(torch.uint8).reshape(-1) for o in O_locals], o_bytes, None)
        O_full = torch.cat([kvq.ulysses_unpack_o(o_recv[r], Ts, H, d, P, torch.float32) for r in range(P)])
        ex = ref.export(0, ch)
        for p, (h0, h1) in enumerate(parts):
            e = caches[p].export(0, ch)
            for name in ("codes_k", "scales_k", "codes_v", "scales_v"):
                full = ex[name].view(T, H, -1)[:, h0:h1].reshape(-1, ex[name].shape[1])
                assert torch.equal(e[name], full), (p, name)
        check_fp32_out(O_full.cpu().numpy(), orc.attend(0, ch, q.f64, sink, window, q_nvfp4=True))


def test_ulysses_nvfp4_exchange_wan_shape_p8():
    # BASELINE.json configs[4] shape: the Wan layer (12 x 128, T_c = 4680) head-sharded over P = 8
    # simulated ranks (2,2,2,2,1,1,1,1 heads), NVFP4 exchange: every rank's cache bytes equal the
    # 1-GPU cache's; sampled O rows within tolerance of the oracle
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    P, H, d, tpf, fc = 8, 12, 128, 1560, 3
    T = tpf * fc
    Ts = T // P
    parts = [kvq.head_partition(H, P, r) for r in range(P)]
    mk = dict(sink_frames=3, window_frames=21, max_chunk_slots=8, device=DEV)
    caches = [kvq.KVCache(1, h1 - h0, d, tpf, fc, **mk) for h0, h1 in parts]
    ref = kvq.KVCache(1, H, d, tpf, fc, **mk)
    orc = OracleKVCache(1, H, d, tpf, fc)
    rows = np.array([0, 584, 585, 2047, 4095, 4679])
    for ch in range(3):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
        Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
        mask = kvq.Mask(ch, 3, 21)
        ref.append(0, ch, K, V)
        orc.append(0, ch, k.f64, v.f64)
        shards = [tuple(x[r * Ts:(r + 1) * Ts].contiguous() for x in (Q, K, V)) for r in range(P)]
        amax = torch.stack([kvq.ulysses_shard_amax(Kr, Vr) for _, Kr, Vr in shards]).max(0).values
        packed = [kvq.ulysses_pack_nvfp4(Qr, Kr, Vr, P, amax) for Qr, Kr, Vr in shards]
        recv = _a2a([sd for sd, _ in packed], [sz for _, sz in packed], None)
        O_locals = []
        for p, (h0, h1) in enumerate(parts):
            Ql = caches[p].append_ulysses_nvfp4(0, ch, recv[p], P, amax)
            O_locals.append(caches[p].attention(0, Ql, mask, torch.float32))
        ex = ref.export(0, ch)
        for p, (h0, h1) in enumerate(parts):
            e = caches[p].export(0, ch)
            for name in ("codes_k", "scales_k", "codes_v", "scales_v"):
                full = ex[name].view(T, H, -1)[:, h0:h1].reshape(-1, ex[name].shape[1])
                assert torch.equal(e[name], full), (p, name)
        if ch == 2:
            O = torch.cat([O_locals[p] for p in range(P)], dim=1).cpu().numpy()   # [T, H, d] by head blocks
            check_fp32_out(O[rows], orc.attend(0, ch, q.f64, 3, 21, rows=rows))


@pytest.mark.parametrize("exchange,io", [(0, "bf16"), (1, "bf16"), (2, "bf16"), (0, "fp32"), (1, "fp32")])
def test_native_nccl_ulysses_world1(exchange, io):
    # ulysses_chunk_attention: the whole head-sharded step behind one C call with libkvq's own NCCL
    # communicator (one rank): O and the cache bytes equal the plain single-GPU path's
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tpf, fc, d, H = 40, 3, 128, 12
    T = tpf * fc
    dt = torch.bfloat16 if io == "bf16" else torch.float32
    mk = dict(sink_frames=3, window_frames=9, max_chunk_slots=8, device=DEV)
    c_ref = kvq.KVCache(1, H, d, tpf, fc, **mk)
    c_nat = kvq.KVCache(1, H, d, tpf, fc, **mk)
    nat = kvq.NcclUlysses(c_nat, H, 0, 1, exchange=exchange, in_dtype=dt, out_dtype=dt)
    try:
        for ch in range(4):
            q, k, v = synth.make_qkv(T, H, d, io, 0, ch)
            Q, K, V = q.torch(DEV), k.torch(DEV), v.torch(DEV)
            mask = kvq.Mask(ch, 3, 9)
            c_ref.append(0, ch, K, V)
            O_ref = c_ref.attention(0, Q, mask, dt)
            O = nat.step(0, ch, Q, K, V, mask)
            torch.cuda.synchronize()
            assert O.dtype == dt
            if exchange == 2:  # NVFP4 Q: a different numerics mode (reading Z24), close to the plain one
                assert torch.isfinite(O).all() and (O.float() - O_ref.float()).norm() < 0.2 * O_ref.float().norm()
            else:
                assert torch.equal(O, O_ref), (exchange, io, ch)
            a, b = c_ref.export(0, ch), c_nat.export(0, ch)
            assert all(torch.equal(a[n], b[n]) for n in a), (exchange, io, ch)
    finally:
        nat.close()


def test_native_nccl_ulysses_argument_errors():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tpf, fc, d, H = 40, 3, 128, 12
    c = kvq.KVCache(1, H, d, tpf, fc, sink_frames=3, window_frames=9, max_chunk_slots=8, device=DEV, k_smoothing=True)
    nat = kvq.NcclUlysses(c, H, 0, 1, exchange=kvq.EXCHANGE_INPUT)
    try:
        q, k, v = synth.make_qkv(tpf * fc, H, d, "bf16", 0, 0)
        with pytest.raises(kvq.KVQError, match="EINVAL"):  # K-smoothing needs the NVFP4 exchange
            nat.step(0, 0, q.torch(DEV), k.torch(DEV), v.torch(DEV), kvq.Mask(0, 3, 9))
    finally:
        nat.close()
    c2 = kvq.KVCache(1, 5, d, tpf, fc, sink_frames=3, window_frames=9, max_chunk_slots=8, device=DEV)
    nat2 = kvq.NcclUlysses(c2, H, 0, 1)
    try:
        q, k, v = synth.make_qkv(tpf * fc, H, d, "bf16", 0, 0)
        with pytest.raises(kvq.KVQError, match="ESHAPE"):  # the cache must hold this rank's 12 heads
            nat2.step(0, 0, q.torch(DEV), k.torch(DEV), v.torch(DEV), kvq.Mask(0, 3, 9))
    finally:
        nat2.close()
