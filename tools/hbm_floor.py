"""What does pure data movement of the append's size cost on this B200?  (Context for the
quantize/append roofline.)  Same timing method as bench.py's append: a CUDA graph of
24 operations cycling 6 distinct inputs (172 MB > L2), L2 flushed before each replay.
  read  : torch.amax over a bf16 K+V chunk pair (28.75 MB read)         -- the amax pass alone
  copy  : 18.4 MB -> 18.4 MB bf16 copy (36.8 MB moved = the append's algorithmic bytes)
  append: kv_quantize_append itself (28.75 MB read + 8.09 MB written)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq

dev = "cuda"
T, H, d = 4680, 12, 128
n = T * H * d
K = [torch.randn(n, device=dev).to(torch.bfloat16) for _ in range(6)]
V = [torch.randn(n, device=dev).to(torch.bfloat16) for _ in range(6)]
src = [torch.randn(n * 18420 // 14377, device=dev).to(torch.bfloat16) for _ in range(6)]
dst = [torch.empty_like(x) for x in src]
out = torch.empty(2, device=dev)
c = kvq.KVCache(1, H, d, 1560, 3, max_chunk_slots=2, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def graph_us(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(6):
            fn(i)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r in range(24):
            fn(r % 6)
    ts = []
    for _ in range(7):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 24)
    return sorted(ts)[3]


def rd(i):  # max |x| of K and V: two pure reductions (28.75 MB read, nothing written but 2 scalars)
    torch.linalg.vector_norm(K[i], float("inf"))
    torch.linalg.vector_norm(V[i], float("inf"))


r_us = graph_us(rd)
c_us = graph_us(lambda i: dst[i].copy_(src[i]))
a_us = graph_us(lambda i: c.append(0, 0, K[i].view(T, H, d), V[i].view(T, H, d)))
for name, us, b in (("amax read (torch)", r_us, 2 * n * 2), ("copy (torch)", c_us, 2 * src[0].numel() * 2),
                    ("kv_quantize_append", a_us, n * 2 * 2 + 2 * n * 9 // 16)):
    print(f"{name:20s} {us:7.2f} us  {b / us / 1e3:7.1f} GB/s  ({b / 1e6:.2f} MB)")
