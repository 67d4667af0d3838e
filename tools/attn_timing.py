"""Attention call timing under different cache conditions (development aid): events around one
call after (a) a 256 MiB zero-fill (dirty L2), (b) the fill + a read of it (clean-ish L2),
(c) no flush (packed window L2-resident), (d) a CUDA graph of 10 calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq, synth
dev = "cuda"
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev)
qs = []
for ch in range(7):
    q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
    c.append(0, ch, k.torch(dev), v.torch(dev))
    qs.append(q.torch(dev))
m = kvq.Mask(6, 3, 21)
Q = qs[6]
O = torch.empty_like(Q)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
FL = 4 * T * 32760 * d * H
def run(prep, n=20):
    ts = []
    for _ in range(n):
        prep()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); c.attention(0, Q, m, out=O); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2] * 1e3
for _ in range(3):
    c.attention(0, Q, m, out=O)
t_a = run(lambda: flush.zero_())
t_b = run(lambda: (flush.zero_(), flush.sum()))
t_c = run(lambda: None)
t_s = run(lambda: (flush.zero_(), torch.cuda.synchronize()))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    c.attention(0, Q, m, out=O)
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    for _ in range(10):
        c.attention(0, Q, m, out=O)
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
g.replay(); torch.cuda.synchronize()
a.record(); g.replay(); b.record(); torch.cuda.synchronize()
t_g = a.elapsed_time(b) * 100
for name, t in (("after zero-fill", t_a), ("after fill+read", t_b), ("no flush", t_c), ("after fill+sync", t_s), ("graph x10", t_g)):
    print(f"{name:16s} {t:7.1f} us  {FL / t / 1e6:6.0f} TFLOP/s")
