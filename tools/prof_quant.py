"""Four single-pass appends of the Wan chunk (for ncu: -k regex:quant_fused -s 2 -c 1)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq, synth
dev = "cuda"
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev)
q, k, v = synth.make_qkv(T, H, d, "bf16", 0, 0)
K, V = k.torch(dev), v.torch(dev)
if "--two-pass" in sys.argv:
    c.force_two_pass(True)
for _ in range(4):
    c.append(0, 0, K, V)
torch.cuda.synchronize()
