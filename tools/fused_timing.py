"""Wan layer step (chunk 6, 32,760 keys) as append + attention (two launches) vs the fused
chunk_attention_append (one launch): CUDA events, L2 flushed before each step, median of 20."""
import os, sys
os.environ["KVQ_FUSED_APPEND"] = "1"  # the fused launch is opt-in (kvq.h)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq, synth

dev = "cuda"
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev)
qs = []
for ch in range(7):
    q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
    qs.append((q.torch(dev), k.torch(dev), v.torch(dev)))
    if ch < 6:
        c.append(0, ch, qs[-1][1], qs[-1][2])
Q, K, V = qs[6]
m = kvq.Mask(6, 3, 21)
O = torch.empty_like(Q)
c.append(0, 6, K, V)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def run(fn, n=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[n // 2]


sep = run(lambda: (c.append(0, 6, K, V), c.attention(0, Q, m, out=O)))
att = run(lambda: c.attention(0, Q, m, out=O))
fus = run(lambda: c.append_attention(0, 6, K, V, Q, m, out=O))
sep2 = run(lambda: (c.append(0, 6, K, V), c.attention(0, Q, m, out=O)))
fus2 = run(lambda: c.append_attention(0, 6, K, V, Q, m, out=O))
print(f"separate append+attention {sep:.1f} / {sep2:.1f} us | attention alone {att:.1f} us | fused {fus:.1f} / {fus2:.1f} us"
      f" | exposed append: separate {sep - att:.1f} us, fused {fus - att:.1f} us")
