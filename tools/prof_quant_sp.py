"""Eager appends on the Wan chunk for ncu (profile one quant_sp_kernel launch: -k regex:quant_sp -s 4 -c 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq
T, H, d = 4680, 12, 128
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device="cuda")
pool = [(torch.randn((T, H, d), device="cuda").bfloat16(), torch.randn((T, H, d), device="cuda").bfloat16()) for _ in range(6)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(8):
    flush.zero_()
    c.append(0, 0, *pool[i % 6])
torch.cuda.synchronize()
