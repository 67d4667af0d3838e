"""Print the CTA-0 role timeline of chunk_attention on the Wan layer (development aid).
Needs a build with the trace points compiled in: KVQ_NVCC_FLAGS=-DKVQ_TRACE_BUILD=1 (attention.cu)."""
import sys, os, ctypes
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
m = kvq.Mask(6, 3, 21)
O = c.attention(0, Q, m)
tr = torch.zeros(64 * 16, dtype=torch.int64, device=dev)
kvq.lib().kvq_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    c.attention(0, Q, m, out=O)
torch.cuda.synchronize()
kvq.lib().kvq_debug_set_trace(None)
t = tr.view(64, 16).cpu().numpy().astype("int64")
t0 = t[0, 0]
names = ["w0", "s0", "p0", "w1", "s1", "p1", "dK", "dV", "PV0", "QK0n", "PV1", "QK1n"]
print("tile " + " ".join(f"{n:>7}" for n in names))
for g in range(0, 40):
    print(f"{g:4d} " + " ".join(f"{(t[g, e] - t0) if t[g, e] else 0:7d}" for e in range(12)))
import numpy as np
per = np.diff(t[5:60, 1])
print("WG0 S-ready period: median", np.median(per), "softmax0 dur median", np.median(t[5:60, 2] - t[5:60, 1]),
      "wait0 median", np.median(t[5:60, 1] - t[5:60, 0]))
print("WG1 softmax dur median", np.median(t[5:60, 5] - t[5:60, 4]), "wait1 median", np.median(t[5:60, 4] - t[5:60, 3]))
print("dequant K->V median", np.median(t[5:60, 7] - t[5:60, 6]), "dequant period", np.median(np.diff(t[5:60, 6])))
print("PV0 issue after P0 done", np.median(t[5:60, 8] - t[5:60, 2]), "PV1 issue after P1 done", np.median(t[5:60, 10] - t[5:60, 5]))
print("S0(g+1) ready after PV0(g) issue", np.median(t[6:61, 1] - t[5:60, 8]))
s = t[5:60]
print("WG0 softmax phases (median cycles): S-ready->LDTM done", np.median(s[:, 12] - s[:, 1]),
      " max", np.median(s[:, 13] - s[:, 12]), " exp loop", np.median(s[:, 14] - s[:, 13]),
      " P store+rescale", np.median(s[:, 15] - s[:, 14]), " ->arrive", np.median(s[:, 2] - s[:, 15]))
