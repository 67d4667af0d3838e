"""Rollout measurements for BASELINE.json configs[2] (W30: 30 layers, frame sink + sliding window,
per-chunk append) and configs[3] (L240: 240 s rollout, NVFP4 vs bf16 KV footprint and throughput).

Reported (CUDA events, device time):
  * W30 chunk step t = 0..8: 30 x (kv_quantize_append + chunk_attention) back to back, layer-query-
    tokens/s, append share of the step (PAPER.md:146's "below 2%" context).
  * L240: 320 chunks x 30 layers, extrapolated from the measured ramp (t < 7) and steady (t >= 7)
    chunk steps; NVFP4 resident footprint vs bf16.
  * one steady layer step three ways: fused NVFP4 attention (this library), the paper's unfused
    design (kv_dequantize_window -> bf16 window, then attention over bf16 K/V), and attention over
    an already-bf16 KV window (the bf16-cache baseline; same kernel family, bf16 operands).
Prints one JSON line.  Run on the GPU box: python tools/rollout.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_18739_b200 import kvq, synth

T, H, D, TPF, FC, SINK, WIN, SLOTS, L = 4680, 12, 128, 1560, 3, 3, 21, 8, 30
dev = "cuda"


def ev_time(fn, reps=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    pool = [tuple(x.torch(dev) for x in synth.make_qkv(T, H, D, "bf16", 0, 200 + i)) for i in range(4)]
    cache = kvq.KVCache(L, H, D, TPF, FC, sink_frames=SINK, window_frames=WIN, max_chunk_slots=SLOTS, device=dev)
    O = torch.empty((T, H, D), dtype=torch.bfloat16, device=dev)
    steps = []
    for t in range(9):
        m = kvq.Mask(t, SINK, WIN)
        # the 30 layers run back to back (no host sync inside the chunk step, as a rollout runs them);
        # per-layer events on the stream then measure device time, the GPU never waits for the host
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(L)]
        torch.cuda.synchronize()
        for layer in range(L):
            q, k, v = pool[(layer * 7 + t) % 4]
            ev[layer][0].record()
            cache.append(layer, t, k, v)
            ev[layer][1].record()
            cache.attention(layer, q, m, out=O)
            ev[layer][2].record()
        torch.cuda.synchronize()
        app = sum(ev[layer][0].elapsed_time(ev[layer][1]) for layer in range(L))
        tot = ev[0][0].elapsed_time(ev[L - 1][2])
        steps.append({"chunk": t, "n_keys": cache.n_keys(0, m), "ms": tot, "append_ms": app,
                      "layer_query_tokens_per_s": L * T / (tot * 1e-3)})
    steady = steps[-1]["ms"]
    ramp = sum(s["ms"] for s in steps[:7])
    l240_chunks = 320
    l240_s = (ramp + steady * (l240_chunks - 7)) * 1e-3
    resident = cache.resident_bytes()
    bf16_resident = L * SLOTS * 2 * T * H * D * 2

    # one steady layer step three ways (layer 0, chunk 8 is resident)
    m = kvq.Mask(8, SINK, WIN)
    q = pool[(0 * 7 + 8) % 4][0]
    fused = ev_time(lambda: cache.attention(0, q, m, out=O), 10)
    Kw, Vw = cache.dequantize_window(0, m)
    deq = ev_time(lambda: cache.dequantize_window(0, m, Kw, Vw), 10)
    bf = ev_time(lambda: kvq.chunk_attention_bf16kv(q, Kw, Vw, out=O), 10)
    wsb = kvq.new_bf16kv_workspace(D)
    bfw = ev_time(lambda: kvq.chunk_attention_bf16kv(q, Kw, Vw, out=O, workspace=wsb), 10)
    flops = 4.0 * T * Kw.shape[0] * D * H
    out = {"config": "W30 + L240 (BASELINE.json configs[2], [3])", "w30_chunk_steps": steps,
           "w30_steady_chunk_ms": steady, "w30_steady_layer_query_tokens_per_s": L * T / (steady * 1e-3),
           "w30_append_share": steps[-1]["append_ms"] / steady,
           "l240_chunks": l240_chunks, "l240_extrapolated_s": l240_s, "l240_extrapolation": "ramp t<7 measured + steady x 313",
           "resident_nvfp4_bytes": resident, "resident_bf16_bytes": bf16_resident,
           "footprint_ratio": bf16_resident / resident,
           "layer_step_ms": {"fused_nvfp4": fused, "unfused_dequant_window": deq, "unfused_attention_bf16kv": bf,
                             "unfused_total": deq + bfw, "bf16_kv_cache_attention": bfw,
                             "bf16_kv_data_parallel_grid": bf},
           "layer_tflops": {"fused_nvfp4": flops / fused / 1e9, "bf16_kv": flops / bfw / 1e9,
                            "bf16_kv_data_parallel_grid": flops / bf / 1e9},
           "n_keys_steady": int(Kw.shape[0])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
