"""A12 bf16-KV attention timing against the window size (development aid): the persistent wave +
stream-K grid (chunk_attention_bf16kv_ws) and the data-parallel grid, Wan heads, bf16 K/V
[n_keys, H, d] in HBM, CUDA events, median of 10 calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_18739_b200 import kvq

T, H, d = 4680, 12, 128
Q = torch.randn(T, H, d, device="cuda").to(torch.bfloat16)
O = torch.empty_like(Q)
ws = kvq.new_bf16kv_workspace(d)


def ev(fn, n=10):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[n // 2]


for n in [int(x) for x in (sys.argv[1:] or ["4096", "16384", "37440"])]:
    K = torch.randn(n, H, d, device="cuda").to(torch.bfloat16)
    V = torch.randn(n, H, d, device="cuda").to(torch.bfloat16)
    fl = 4.0 * T * n * d * H
    tp = ev(lambda: kvq.chunk_attention_bf16kv(Q, K, V, out=O, workspace=ws))
    td = ev(lambda: kvq.chunk_attention_bf16kv(Q, K, V, out=O))
    print(f"n_keys {n:6d} window {2 * n * H * d * 2 / 1e6:6.1f} MB: persistent {tp:.3f} ms "
          f"{fl / tp / 1e9:6.0f} TFLOP/s | data-parallel {td:.3f} ms {fl / td / 1e9:6.0f} TFLOP/s")
