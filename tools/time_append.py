"""Device time of kv_quantize_append on the Wan chunk as bench.py measures it (CUDA graph of 24
appends cycling 6 distinct K/V chunks, 172 MB > L2, so inputs come from HBM), plus the two-pass
fallback and an L2-hot figure for reference (development aid; bench.py is the contract)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq

dev = "cuda"
T, H, d = 4680, 12, 128
BYTES = T * H * d * 2 * (2 + 9 / 16)
c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device=dev,
                scale_search="--search" in sys.argv, k_smoothing="--smooth" in sys.argv)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
pool = [(torch.randn((T, H, d), generator=gen, device=dev).bfloat16(),
         torch.randn((T, H, d), generator=gen, device=dev).bfloat16()) for _ in range(6)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


amaxes = [torch.stack([k.float().abs().max(), v.float().abs().max()]).contiguous() for k, v in pool]


def graph_time(n_app, cycle, ext=False):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    kw = (lambda i: {"amax_kv": amaxes[i]}) if ext else (lambda i: {})
    with torch.cuda.stream(s):
        c.append(0, 0, *pool[0], **kw(0))
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n_app):
            j = i % len(pool) if cycle else 0
            c.append(0, 0, *pool[j], **kw(j))
    ts = []
    for _ in range(7):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / n_app)
    return sorted(ts)[len(ts) // 2]


t_cold = graph_time(24, True)
t_hot = graph_time(24, False)
c.force_two_pass(True)
t_two = graph_time(24, True)
t_two_ext = graph_time(24, True, ext=True)
c.force_two_pass(False)
t_ext = graph_time(24, True, ext=True)
print(f"append cold {t_cold:.2f} us ({BYTES / t_cold / 1e3:.0f} GB/s, {BYTES / t_cold / 1e3 / 6550.7:.1%} of 6550.7)"
      f" | L2-hot {t_hot:.2f} us | two-pass cold {t_two:.2f} us")
print(f"amax supplied: kv_quantize_append_amax {t_ext:.2f} us ({BYTES / t_ext / 1e3:.0f} GB/s) | "
      f"streaming quantize pass alone (forced) {t_two_ext:.2f} us ({BYTES / t_two_ext / 1e3:.0f} GB/s, "
      f"{BYTES / t_two_ext / 1e3 / 6550.7:.1%})")
