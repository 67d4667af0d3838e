"""Max-abs / rel-L2 of chunk_attention (fp32-out) vs the float64 oracle on peaked and iid data at
the Wan shape (sampled rows) and the tiny config -- the tolerance margin of numerics choices."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.cache import OracleKVCache
from paper_2605_18739_b200 import kvq, synth
rows = np.array([0, 1, 127, 128, 1000, 2047, 3333, 4095, 4600, 4679])
for variant in ("iid", "peaked"):
    T, H, d = 4680, 12, 128
    c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device="cuda")
    o = OracleKVCache(1, H, d, 1560, 3)
    for ch in range(3):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch, variant=variant)
        c.append(0, ch, k.torch("cuda"), v.torch("cuda"))
        o.append(0, ch, k.f64, v.f64)
    if variant == "peaked":
        q = synth.Tensor(q.f64 * 3.0, "bf16")   # score std ~9: very peaked rows
    O = c.attention(0, q.torch("cuda"), kvq.Mask(2, 3, 21), torch.float32).cpu().numpy()[rows]
    ref = o.attend(0, 2, q.f64, 3, 21, rows=rows)
    print(f"{variant:7s} max-abs {np.abs(O - ref).max():.3e}  rel-L2 {np.linalg.norm(O - ref) / np.linalg.norm(ref):.3e}  |O|max {np.abs(ref).max():.2f}")
