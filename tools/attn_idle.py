"""Attention call time vs the GPU's recent load (development aid): back to back, after idle gaps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq, synth
dev = "cuda"
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev)
for ch in range(7):
    q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
    c.append(0, ch, k.torch(dev), v.torch(dev))
Q = q.torch(dev)
O = torch.empty_like(Q)
m = kvq.Mask(6, 3, 21)
def one():
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); c.attention(0, Q, m, out=O); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3
for _ in range(3): one()
bb = [one() for _ in range(20)]
print("back to back:", " ".join(f"{x:.0f}" for x in bb))
for gap in (0.001, 0.01, 0.1, 0.5):
    ts = []
    for _ in range(5):
        time.sleep(gap)
        ts.append(one())
    print(f"after {gap*1e3:.0f} ms idle:", " ".join(f"{x:.0f}" for x in ts))
# long back-to-back burst (power steady state)
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
for _ in range(200): c.attention(0, Q, m, out=O)
b.record(); torch.cuda.synchronize()
print(f"200 back-to-back: {a.elapsed_time(b) / 200 * 1e3:.0f} us each")
