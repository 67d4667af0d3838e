"""Every kernel once on small shapes, for compute-sanitizer:
    compute-sanitizer --tool memcheck python tools/sanitize_all.py
Single-pass and two-pass quantize/append (plain, 4/6 search, K-smoothing), dequantize, export,
window dequant, fused attention (bf16 Q, fp32 Q split, smoothing, bf16 output), bf16-KV attention,
Ulysses bf16 / NVFP4 (+ NVFP4 Q) / peer exchanges with simulated ranks, the persistent TMA bf16-KV
grid, out-of-fp16-range queries and the f4 direct path (one rank).  Prints OK at the end."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_18739_b200 import kvq, synth

dev = "cuda"


def a2a(sends, sizes):
    P = len(sends)
    offs = [np.concatenate([[0], np.cumsum(s)]) for s in sizes]
    return [torch.cat([sends[r][int(offs[r][p]):int(offs[r][p]) + sizes[r][p]] for r in range(P)]) for p in range(P)]


for d in (64, 128):
    for search, smooth in ((False, False), (True, False), (False, True)):
        for dt in ("bf16", "fp32"):
            T, H = 150, 3
            c = kvq.KVCache(1, H, d, 50, 3, sink_frames=1, window_frames=6, max_chunk_slots=4, device=dev,
                            scale_search=search, k_smoothing=smooth)
            for ch in range(3):
                q, k, v = synth.make_qkv(T, H, d, dt, 0, ch)
                c.force_two_pass(ch == 1)
                c.append(0, ch, k.torch(dev), v.torch(dev))
                c.attention(0, q.torch(dev), kvq.Mask(ch, 1, 6), torch.float32)
                c.attention(0, q.torch(dev), kvq.Mask(ch, 1, 6), torch.bfloat16)
            c.dequantize(0, 2, torch.float32)
            c.dequantize(0, 2, torch.bfloat16)
            c.export(0, 2)
            c.dequantize_window(0, kvq.Mask(2, 1, 6))
q, k, v = synth.make_qkv(150, 3, 128, "bf16", 0, 0)
kvq.chunk_attention_bf16kv(q.torch(dev), k.torch(dev), v.torch(dev))
for dd in (64, 128):  # A12 on the persistent grid: TMA-landed tiles, ragged key tail, stream-K partials
    qb, kb, vb = synth.make_qkv(300, 3, dd, "bf16", 0, 1)
    kvq.chunk_attention_bf16kv(qb.torch(dev), kb.torch(dev)[:233].contiguous(), vb.torch(dev)[:233].contiguous(),
                               workspace=kvq.new_bf16kv_workspace(dd, dev))
# queries outside fp16's range (per-row power-of-two scaling) and a score-range report (reading Z25)
cz = kvq.KVCache(1, 3, 128, 50, 3, sink_frames=1, window_frames=6, max_chunk_slots=4, device=dev)
qz, kz, vz = synth.make_qkv(150, 3, 128, "bf16", 0, 0)
cz.append(0, 0, kz.torch(dev), vz.torch(dev))
Qz = qz.torch(dev).clone()
Qz[3] *= 2.0 ** 40
Qz[7] *= 2.0 ** -40
cz.attention(0, Qz, kvq.Mask(0, 1, 6), torch.float32)
cz.attention(0, Qz, kvq.Mask(0, 1, 6), torch.bfloat16, workspace=cz.new_attention_workspace())
cz.status()
# exchanges, P = 2 simulated ranks
P, H, d, T = 2, 5, 128, 120
Ts = T // P
parts = [kvq.head_partition(H, P, r) for r in range(P)]
caches = [kvq.KVCache(1, h1 - h0, d, 40, 3, sink_frames=3, window_frames=9, max_chunk_slots=4, device=dev)
          for h0, h1 in parts]
q, k, v = synth.make_qkv(T, H, d, "bf16", 0, 0)
Q, K, V = q.torch(dev), k.torch(dev), v.torch(dev)
sh = [tuple(x[r * Ts:(r + 1) * Ts].contiguous() for x in (Q, K, V)) for r in range(P)]
packed = [kvq.ulysses_pack(*s, P) for s in sh]
recv = a2a([x for x, _ in packed], [y for _, y in packed])
for p, (h0, h1) in enumerate(parts):
    Ql, Kl, Vl, am = kvq.ulysses_unpack_qkv(recv[p], Ts, h1 - h0, d, P)
    caches[p].append(0, 0, Kl, Vl, amax_kv=am)
amax = torch.stack([kvq.ulysses_shard_amax(s[1], s[2]) for s in sh]).max(0).values
amax_q = torch.stack([kvq.ulysses_q_amax(s[0]) for s in sh]).max(0).values
for aq in (None, amax_q):
    packed = [kvq.ulysses_pack_nvfp4(*s, P, amax, amax_q=aq) for s in sh]
    recv = a2a([x for x, _ in packed], [y for _, y in packed])
    for p in range(P):
        r = caches[p].append_ulysses_nvfp4(0, 1 if aq is None else 2, recv[p], P, amax, amax_q=aq)
        if aq is not None:
            caches[p].attention_qscaled(0, r[0], r[1], kvq.Mask(2, 3, 9))
o = [torch.zeros(T * (h1 - h0) * d * 2, dtype=torch.uint8, device=dev) for h0, h1 in parts]
orecv = a2a(o, [[Ts * (h1 - h0) * d * 2] * P for h0, h1 in parts])
kvq.ulysses_unpack_o(orecv[0], Ts, H, d, P)
wb = kvq.peer_window_bytes(T, H, d, P)
wins = [torch.zeros(wb, dtype=torch.uint8, device=dev) for _ in range(P)]
pes = [kvq.PeerExchange(T, H, d, P, r, [w.data_ptr() for w in wins]) for r in range(P)]
for r in range(P):
    pes[r].publish_amax(sh[r][1], sh[r][2], 1)
for r in range(P):
    pes[r].pack(*sh[r], 1)
for p, (h0, h1) in enumerate(parts):
    Ql = torch.empty((T, h1 - h0, d), dtype=torch.bfloat16, device=dev)
    pes[p].append(caches[p], 0, 3, 1, Ql)
for p in range(P):
    pes[p].signal_o(1)
for r in range(P):
    pes[r].pull_o(1, torch.empty((Ts, H, d), dtype=torch.bfloat16, device=dev))
# f4 direct (owners' cache slots and O shards written in place), one rank: the sanitizer serializes
# kernels, so cross-rank device waits would never be satisfied with P > 1 under it
T1, H1 = 120, 5
c1 = kvq.KVCache(1, H1, 128, 40, 3, sink_frames=3, window_frames=9, max_chunk_slots=4, device=dev)
w1 = torch.zeros(kvq.peer_window_bytes(T1, H1, 128, 1), dtype=torch.uint8, device=dev)
pe1 = kvq.PeerExchange(T1, H1, 128, 1, 0, [w1.data_ptr()])
pe1.bind_caches(c1, [c1.arena.data_ptr()])
for ch in range(2):
    q1, k1, v1 = (x.torch(dev) for x in synth.make_qkv(T1, H1, 128, "bf16", 0, ch))
    pe1.publish_amax(k1, v1, ch + 1)
    pe1.append_direct(0, ch, q1, k1, v1, ch + 1)
    pe1.attention_direct(0, kvq.Mask(ch, 3, 9), ch + 1)
    pe1.wait_o(ch + 1)
torch.cuda.synchronize()
print("OK")
