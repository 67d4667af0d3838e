"""Phase timeline (ns, globaltimer) of the single-pass quantize kernel over all CTAs (development aid).
Events per CTA: 0 start, 1 K landed, 5 V landed, 6 K amax known (after polling every CTA's slot),
4 K fast path done, 3 K quantized, 2 V amax known, 7 V quantized."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_18739_b200 import kvq, synth
dev = "cuda"
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev)
q, k, v = synth.make_qkv(T, H, d, "bf16", 0, 0)
K, V = k.torch(dev), v.torch(dev)
c.append(0, 0, K, V)
tr = torch.zeros(256 * 8, dtype=torch.int64, device=dev)
kvq.lib().kvq_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    flush.zero_()
    c.append(0, 0, K, V)
torch.cuda.synchronize()
kvq.lib().kvq_debug_set_trace(None)
t = tr.view(256, 8).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
t = t - t0
names = {0: "start", 1: "K landed", 5: "V landed", 6: "K amax", 4: "K fast", 3: "K quant", 2: "V amax", 7: "V quant"}
print(f"{len(t)} CTAs: " + "  ".join(f"{n}: min {t[:, e].min()} med {int(np.median(t[:, e]))} max {t[:, e].max()}"
                                     for e, n in names.items()))
