"""Quick device timing of the W single-layer step (development aid; bench.py is the contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq, synth

dev = "cuda"
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev)
chunks = [synth.make_qkv(T, H, d, "bf16", 0, ch) for ch in range(7)]
qs = [tuple(x.torch(dev) for x in ch) for ch in chunks]
for ch in range(7):
    c.append(0, ch, qs[ch][1], qs[ch][2])
m = kvq.Mask(6, 3, 21)
Q = qs[6][0]
O = torch.empty_like(Q)
def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3
ta = timeit(lambda: c.attention(0, Q, m, out=O))
flops = 4 * T * 32760 * d * H
print(f"attention: {ta:.1f} us  {flops/ta/1e6:.1f} TFLOP/s  {T/ta*1e6/1e6:.3f} M q-tok/s")
tq = timeit(lambda: c.append(0, 6, qs[6][1], qs[6][2]), 50)
print(f"append: {tq:.2f} us  {T*H*d*2*(2+9/16)/tq/1e3:.1f} GB/s")
# device time of the append alone: 20 appends captured in one CUDA graph (removes host launch cost)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    c.append(0, 6, qs[6][1], qs[6][2])
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    for _ in range(20):
        c.append(0, 6, qs[6][1], qs[6][2])
tg = timeit(lambda: g.replay(), 10) / 20
print(f"append (graph): {tg:.2f} us  {T*H*d*2*(2+9/16)/tg/1e3:.1f} GB/s")
c.force_two_pass(True)
g2 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    c.append(0, 6, qs[6][1], qs[6][2])
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g2):
    for _ in range(20):
        c.append(0, 6, qs[6][1], qs[6][2])
tg2 = timeit(lambda: g2.replay(), 10) / 20
print(f"append two-pass (graph): {tg2:.2f} us  {T*H*d*2*(2+9/16)/tg2/1e3:.1f} GB/s")
c.force_two_pass(False)
