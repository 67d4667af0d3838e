"""Phase timeline (ns, globaltimer, median/max over CTAs) of the single-pass quantize kernel in steady
state (development aid).  Events per CTA (thread 0): 0 start, 1 K landed + published, 5 K barrier
seen (thread 0 is a K poller during A(V)), 6 V landed + published, 8 K table, 10/12 K loop
iterations 1/2 done, 3 K quantized, 2 V barrier, 9 V table, 11/13 V iterations, 7 V quantized.
Needs a build with the trace points compiled in: KVQ_NVCC_FLAGS=-DKVQ_TRACE_BUILD=1 (quant.cu)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_18739_b200 import kvq, synth
dev = "cuda"
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
pool = [(torch.randn((T, H, d), generator=gen, device=dev).bfloat16(),
         torch.randn((T, H, d), generator=gen, device=dev).bfloat16()) for _ in range(6)]
c.append(0, 0, *pool[0])
tr = torch.zeros(256 * 16, dtype=torch.int64, device=dev)
kvq.lib().kvq_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
# steady state, as bench.py times it: a graph of 12 appends cycling 6 distinct chunks (inputs from
# HBM, code and barrier lines warm); the trace buffer keeps the last append's events
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    c.append(0, 0, *pool[0])
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(12):
        c.append(0, 0, *pool[i % 6])
for _ in range(3):
    flush.zero_()
    g.replay()
torch.cuda.synchronize()
kvq.lib().kvq_debug_set_trace(None)
t = tr.view(256, 16).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
t = t - t0
names = {0: "start", 1: "K landed", 5: "K barrier seen", 6: "V landed+published", 8: "K table", 10: "K it1",
         12: "K it2", 3: "K quant", 2: "V barrier", 9: "V table", 11: "V it1", 13: "V it2", 7: "V quant"}
print(f"{len(t)} CTAs: " + "  ".join(f"{n}: {int(np.median(t[:, e]))}/{t[:, e].max()}" for e, n in names.items()
                                     if t[:, e].min() >= 0))
