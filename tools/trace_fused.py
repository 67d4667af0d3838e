"""Timeline of the fused append + attention launch on the Wan layer (development aid): CTA 0's role
events (as tools/trace_attn.py), the fused-append phases of CTA 0 (clock64), and for every CTA when it
first needed the appended slot and how long it waited for it (globaltimer, ns).
Needs a build with the trace points compiled in: KVQ_NVCC_FLAGS=-DKVQ_TRACE_BUILD=1 (attention.cu)."""
import sys, os, ctypes
os.environ["KVQ_FUSED_APPEND"] = "1"  # the fused launch is opt-in (kvq.h)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_18739_b200 import kvq, synth

dev = "cuda"
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev)
for ch in range(6):
    q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
    c.append(0, ch, k.torch(dev), v.torch(dev))
q, k, v = synth.make_qkv(T, H, d, "bf16", 0, 6)
Q, K, V = q.torch(dev), k.torch(dev), v.torch(dev)
m = kvq.Mask(6, 3, 21)
O = c.append_attention(0, 6, K, V, Q, m)
tr = torch.zeros(1024 + 3 * 148, dtype=torch.int64, device=dev)
kvq.lib().kvq_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    c.append_attention(0, 6, K, V, Q, m, out=O)
torch.cuda.synchronize()
kvq.lib().kvq_debug_set_trace(None)
t = tr.cpu().numpy().astype("int64")
ap = t[63 * 16:63 * 16 + 5]
print("CTA0 fused-append phases (clock64 from role start): amax read", ap[1] - ap[0], " partials exchanged",
      ap[2] - ap[0], " quantized", ap[3] - ap[0], " all CTAs done", ap[4] - ap[0])
start = t[1024 + 296:1024 + 296 + 148]
w0, wl = t[1024:1024 + 296:2], t[1025:1024 + 296:2]
k0 = start.min()
has = w0 > 0
rel = (w0[has] - k0) / 1e3
print(f"CTAs that reached the appended slot: {has.sum()}; first reach at {rel.min():.1f} us after the first CTA "
      f"started, median {np.median(rel):.1f} us; wait: max {wl[has].max() / 1e3:.1f} us, median {np.median(wl[has]) / 1e3:.2f} us")
order = np.argsort(rel)[:10]
print("earliest:", [(int(np.flatnonzero(has)[i]), round(float(rel[i]), 1), round(float(wl[has][i]) / 1e3, 1)) for i in order])
