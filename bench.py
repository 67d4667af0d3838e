"""Benchmark of the LongLive-2.0 NVFP4 KV-cache hot path on B200 (driver contract: one JSON line).

Metric (BASELINE.json): attention query-tokens/s and KV HBM GB/s (% roofline).  Workload at N=1
is BASELINE.json configs[1], the Wan2.1-1.3B-shaped single layer: 12 heads x 128, chunk =
3 latent frames x 1560 tokens (T_c = 4680), window 21 frames incl. the current chunk + 3-frame
sink -> |K_eff| = 32,760 keys (chunk 6 of a rollout: 7 resident chunks).  One STEP = the whole
hot path for one (layer, chunk): kv_quantize_append(K, V) of the new chunk + chunk_attention of
its queries over the quantized window with fused dequant.  value = T_c / step time.

N>1 (torchrun, one process per GPU): the same layer step head-sharded Ulysses-style
(PAPER.md:556-564): pack -> NCCL all-to-all -> append + attention on the local heads -> NCCL
all-to-all of O -> unpack.  value = T_c / max-over-ranks step time (strong scaling: the layer
shape is fixed).

--impl reference: the float64 CPU oracle (oracle/) on the host cores, each step a bounded
sample of the same workload, printed with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

T_FRAMES, TPF, H, D = 3, 1560, 12, 128
T_C = T_FRAMES * TPF
SINK, WINDOW = 3, 21
CHUNK = 6                      # chunk index whose step is timed: 7 resident chunks, 32,760 keys
METRIC = "attention query-tokens/s and KV HBM GB/s (% roofline) at 1/2/4/8 B200"
WORKLOAD = "Wan2.1-1.3B-shaped single layer (BASELINE.json configs[1])"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            P = json.load(f)
        return P["hbm_gbs"], P["bf16_tflops"], P.get("bf16_tflops_sustained", P["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def n_keys():
    # |K_eff(6)| with a 3-frame sink and 21-frame window: frames [0, 21) -> 32,760 tokens
    f_end = (CHUNK + 1) * T_FRAMES
    frames = set(range(0, min(SINK, f_end))) | set(range(max(0, f_end - WINDOW), f_end))
    return len(frames) * TPF


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every 5 ms through NVML (the same counters
    nvidia-smi's clocks.sm / clocks_event_reasons.* report) while the timed region runs."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index, self.rows, self.stop = index, [], threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self.stop.is_set():
                    try:
                        self.rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                          pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    except Exception:
                        pass
                    time.sleep(0.005)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for _, bits in self.rows for n, b in self.REASONS.items() if bits & b})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(self.max_mhz), "sm_min_mhz": float(min(sm)),
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 5 ms"}


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        n = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
        return int(n)
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- CPU oracle leg
class OracleStep:
    """The float64 oracle (oracle/, as it stands) on one step of the bench workload: quantize the new
    chunk's K and V (the cache's history chunks were quantized by earlier steps), dequantize the
    21-frame window (7 chunks of K and V, Eq. 2) and attend all 4,680 queries of all 12 heads over its
    32,760 keys.  `full()` times exactly that; `sample()` times the per-head share of it -- 1/12 of the
    quantize rows, 1/12 of every window chunk's dequantize, the attention of head 0 -- scaled by 12
    (heads are independent and cost the same).  Both arms of bench.py report the sample."""

    def __init__(self):
        from oracle import nvfp4
        from paper_2605_18739_b200 import synth
        self.nvfp4 = nvfp4
        nk = n_keys()
        self.n_win = nk // T_C                      # 7 window chunks (sink deduplicated into the window)
        self.q, self.k, self.v = synth.make_qkv(T_C, H, D, "bf16", 0, CHUNK)
        hist = [synth.make_qkv(T_C, H, D, "bf16", 0, c) for c in range(CHUNK)]
        self.hist = [(nvfp4.quantize_kv_chunk(k.f64), nvfp4.quantize_kv_chunk(v.f64)) for _, k, v in hist]

    def full(self):
        from oracle.attention import attention
        nv = self.nvfp4
        t0 = time.perf_counter()
        qk, qv = nv.quantize_kv_chunk(self.k.f64), nv.quantize_kv_chunk(self.v.f64)
        win = self.hist + [(qk, qv)]
        K = np.concatenate([nv.dequantize_kv_chunk(a, T_C, H, D) for a, _ in win])
        V = np.concatenate([nv.dequantize_kv_chunk(b, T_C, H, D) for _, b in win])
        attention(self.q.f64, K, V)
        return time.perf_counter() - t0

    def sample(self):
        from oracle.attention import attention
        nv = self.nvfp4
        rows = T_C // H

        def head0(q):  # the head-0 rows (t, 0) of a quantized chunk: its per-head share of the dequantize
            return nv.dequantize_kv_chunk(dict(q, codes=q["codes"][0::H], scales=q["scales"][0::H]), T_C, 1, D)

        t0 = time.perf_counter()
        qk, qv = nv.quantize_kv_chunk(self.k.f64[:rows]), nv.quantize_kv_chunk(self.v.f64[:rows])
        win = self.hist + [self.hist[0]]   # the 7th (new) chunk's head-0 dequantize costs the same as any other
        K = np.concatenate([head0(a) for a, _ in win])
        V = np.concatenate([head0(b) for _, b in win])
        attention(self.q.f64[:, :1], K, V)
        return (time.perf_counter() - t0) * H

    SAMPLE_DESC = ("per-head share of one step, x12 heads: quantize 390 of the 4,680 token rows of the new K and V, "
                   "dequantize the head-0 rows of the 7 window chunks of K and V, attention of head 0 for all "
                   "4,680 queries over 32,760 keys")
    FULL_DESC = ("one full step, measured: quantize the new chunk's K and V (4,680 x 12 x 128 each), dequantize "
                 "the 7-chunk window, attention of all 4,680 queries x 12 heads over 32,760 keys")


# ----------------------------------------------------------------------------- GPU leg
def sustained_attention(cache, q, mask, O, st, dev_index, seconds=2.0):
    """chunk_attention back to back for >= `seconds` (no flush: a long step's steady state), NVML clocks
    sampled throughout; returns the mean ms per call and the clock summary."""
    import torch
    cache.attention(0, q, mask, out=O)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        cache.attention(0, q, mask, out=O)
    e1.record(st)
    torch.cuda.synchronize()
    n = max(20, int(seconds / (e0.elapsed_time(e1) * 1e-3 / 20)))
    with ClockSampler(dev_index) as clk:
        e0.record(st)
        for _ in range(n):
            cache.attention(0, q, mask, out=O)
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    return {"ms": ms, "calls": n, "seconds": ms * n * 1e-3, "clocks": clk.summary()}


def rollout_w30(dev, steps=3):
    """BASELINE.json configs[2] (W30) and configs[3] (L240) on one GPU: 30 layers, 3-frame sink +
    21-frame window; one chunk step = append + attention for every layer.  Inputs: a pool of 4 seeded
    chunk triples (as the W30 parity test).  Returns the steady chunk-step time (37,440 keys per layer),
    the append share, the ramp steps, the L240 extrapolation and the cache footprint."""
    import torch
    from paper_2605_18739_b200 import kvq, synth
    L, SLOTS, POOL = 30, 8, 4
    pool = [tuple(x.torch(dev) for x in synth.make_qkv(T_C, H, D, "bf16", 0, 100 + i)) for i in range(POOL)]
    cache = kvq.KVCache(L, H, D, TPF, T_FRAMES, sink_frames=SINK, window_frames=WINDOW, max_chunk_slots=SLOTS,
                        device=dev)
    O = torch.empty((T_C, H, D), dtype=torch.bfloat16, device=dev)
    st = torch.cuda.current_stream()

    def chunk_step(t, attend=True, append=True):
        for layer in range(L):
            q, k, v = pool[(layer * 7 + t) % POOL]
            if append:
                cache.append(layer, t, k, v)
            if attend:
                cache.attention(layer, q, kvq.Mask(t, SINK, WINDOW), out=O)

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    ramp = [timed(lambda: chunk_step(t)) for t in range(7)]            # t = 0..6: 4,680 (t+1) keys
    steady = [timed(lambda: chunk_step(t)) for t in range(7, 7 + steps)]  # t >= 7: 37,440 keys
    t_last = 7 + steps - 1
    app = [timed(lambda: chunk_step(t_last, attend=False)) for _ in range(steps)]   # re-append = overwrite
    step_ms = float(np.median(steady))
    app_ms = float(np.median(app))
    n_chunks = 320                       # 240 s x 16 fps / 4 (VAE) / 3 frames per chunk
    l240_s = (sum(ramp) + step_ms * (n_chunks - 7)) * 1e-3
    nv = cache.resident_bytes()
    bf16 = L * SLOTS * 2 * T_C * H * D * 2
    # D4 throughput: one steady layer step's attention three ways (layer 0, chunk t_last resident):
    # fused NVFP4 (the product), a bf16 KV cache (the same kernel family with TMA-landed bf16 tiles on
    # the persistent grid, A12) and the paper's unfused design (dequantize the window to bf16, then A12)
    m = kvq.Mask(t_last, SINK, WINDOW)
    q = pool[(0 * 7 + t_last) % POOL][0]
    Kw, Vw = cache.dequantize_window(0, m)
    wsb = kvq.new_bf16kv_workspace(D)
    fused = float(np.median([timed(lambda: cache.attention(0, q, m, out=O)) for _ in range(5)]))
    bfkv = float(np.median([timed(lambda: kvq.chunk_attention_bf16kv(q, Kw, Vw, out=O, workspace=wsb)) for _ in range(5)]))
    deq = float(np.median([timed(lambda: cache.dequantize_window(0, m, Kw, Vw)) for _ in range(5)]))
    fl = 4.0 * T_C * Kw.shape[0] * D * H
    cmp_ = {"n_keys": int(Kw.shape[0]), "fused_nvfp4_ms": fused, "bf16_kv_ms": bfkv, "unfused_dequant_ms": deq,
            "unfused_total_ms": deq + bfkv, "fused_nvfp4_tflops": fl / fused / 1e9, "bf16_kv_tflops": fl / bfkv / 1e9,
            "kv_bytes_per_layer_step": {"nvfp4": int(2 * Kw.shape[0] * H * D * 9 // 16), "bf16": int(2 * Kw.shape[0] * H * D * 2)}}
    return {"w30": {"config": "BASELINE.json configs[2]: 30 layers, sink 3 frames + window 21 frames, chunk t >= 7 "
                              "(37,440 keys per layer)",
                    "steady_chunk_step_ms": step_ms, "layer_query_tokens_per_s": L * T_C / (step_ms * 1e-3),
                    "append_share": app_ms / step_ms, "appends_ms_per_chunk_step": app_ms,
                    "ramp_chunk_step_ms": ramp, "attention_tflops": L * 4.0 * T_C * 37440 * D * H / (step_ms * 1e-3) / 1e12},
            "l240": {"config": "BASELINE.json configs[3]: 320 chunks x 30 layers, one denoising pass",
                     "pass_s_extrapolated": l240_s, "extrapolation": "measured ramp steps t = 0..6 + 313 x the "
                     "measured steady chunk step", "resident_bytes_nvfp4": nv, "resident_bytes_bf16_kv": bf16,
                     "footprint_ratio": bf16 / nv, "layer_step_nvfp4_vs_bf16_kv": cmp_}}



def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2605_18739_b200 import kvq, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    force = args.force_ulysses and world == 1  # debug: the N>1 code path on one GPU (one-rank NCCL group)
    if world > 1 or force:
        dist.init_process_group("nccl", device_id=dev)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    P = world
    h0, h1 = kvq.head_partition(H, P, rank)
    Hr = h1 - h0
    nk = n_keys()

    arena = None
    if args.exchange == "peer" and (P > 1 or force):  # f4 direct: the owners' caches are written over peer memory
        import torch.distributed._symmetric_memory as symm_mem
        arena = symm_mem.empty(kvq.cache_bytes(1, Hr, D, TPF, T_FRAMES, SINK, WINDOW, 8), dtype=torch.uint8, device=dev)
    cache = kvq.KVCache(1, Hr, D, TPF, T_FRAMES, sink_frames=SINK, window_frames=WINDOW, max_chunk_slots=8,
                        device=dev, arena=arena)
    mask = kvq.Mask(CHUNK, SINK, WINDOW)
    Ts = T_C // P
    # synthetic chunk data (seeded); each rank holds its sequence shard of the full [T_c, H, d]
    chunks = []
    for ch in range(CHUNK + 1):
        q, k, v = synth.make_qkv(T_C, H, D, "bf16", 0, ch)
        chunks.append(tuple(x.torch("cpu")[rank * Ts:(rank + 1) * Ts].contiguous() for x in (q, k, v)))
    dq = [tuple(x.to(dev) for x in c) for c in chunks]
    native = args.exchange.startswith("native")
    if not (P > 1 or force):
        uly = None
    elif native:  # the one-call C step with libkvq's own NCCL communicator
        uly = kvq.NcclUlysses(cache, H, rank, P, exchange=kvq.EXCHANGE_NVFP4 if args.exchange == "native-nvfp4"
                              else kvq.EXCHANGE_INPUT)
    else:
        uly = kvq.Ulysses(cache, H, D, T_C, rank, P, nvfp4_kv=args.exchange == "nvfp4", peer=args.exchange == "peer",
                          nvfp4_q=args.exchange == "nvfp4q")

    def step(c, out=None):
        q, k, v = dq[c]
        if uly is None:
            cache.append(0, c, k, v)
            return cache.attention(0, q, mask if c == CHUNK else kvq.Mask(c, SINK, WINDOW), out=out)
        return uly.step(0, c, q, k, v, mask if c == CHUNK else kvq.Mask(c, SINK, WINDOW), out=out)

    for c in range(CHUNK):          # fill the window: chunks 0..5
        step(c)
    # the timed step re-writes chunk 6 each time (a denoising step of the in-progress chunk)
    O = torch.empty((Ts, H, D), dtype=torch.bfloat16, device=dev)
    step(CHUNK, O)
    torch.cuda.synchronize()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # 256 MiB > 126 MB L2
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ev_att = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ev_app = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    q6, k6, v6 = dq[CHUNK]
    Olocal = torch.empty((T_C, Hr, D), dtype=torch.bfloat16, device=dev)

    for _ in range(args.warmup):
        flush.zero_()
        step(CHUNK, O)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev_mid = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()                                  # L2 flushed before every step
            ev[i][0].record(st)
            if uly is None:  # step(CHUNK, O) with an event between the append and the attention launch
                cache.append(0, CHUNK, k6, v6)
                ev_mid[i].record(st)
                cache.attention(0, q6, mask, out=O)
            else:
                step(CHUNK, O)
            ev[i][1].record(st)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # per-kernel timing on this rank's local head set (1-GPU shapes when P = 1)
        if uly is None:
            for i in range(args.steps):
                flush.zero_()
                ev_app[i][0].record(st)
                cache.append(0, CHUNK, k6, v6)
                ev_app[i][1].record(st)
                flush.zero_()
                ev_att[i][0].record(st)
                cache.attention(0, q6, mask, out=O)
                ev_att[i][1].record(st)
            torch.cuda.synchronize()
    step_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms = float(t.item())
    value = T_C / (step_ms * 1e-3)

    # ---- end-to-end through the public API with host buffers (pinned), copies inside the region
    # (each rank copies its own shard in and its O shard out; at N=1 the shard is the whole chunk).
    # Steps are pipelined the way a serving loop runs them: step i's inputs are copied host->device
    # on a copy stream while step i-1 computes, and step i-1's O is read back on a third stream
    # (two device buffer sets, events between the streams); every step still copies all of its
    # inputs in and its output out inside the timed region.
    hq, hk, hv = (x.pin_memory() for x in chunks[CHUNK])
    hO = [torch.empty((Ts, H, D), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    dbuf = [tuple(torch.empty_like(x, device=dev) for x in (hq, hk, hv)) + (torch.empty((Ts, H, D), dtype=torch.bfloat16,
                                                                                      device=dev),)
            for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def e2e_run(n):
        for i in range(n):
            b = i & 1
            gq, gk, gv, Ob = dbuf[b]
            if i >= 2:
                s_in.wait_event(ev_comp[b])          # step i-2 has consumed this input set
            with torch.cuda.stream(s_in):
                gq.copy_(hq, non_blocking=True)
                gk.copy_(hk, non_blocking=True)
                gv.copy_(hv, non_blocking=True)
                ev_in[b].record(s_in)
            st.wait_event(ev_in[b])
            if i >= 2:
                st.wait_event(ev_out[b])             # step i-2's O has been read back
            if uly is None:
                cache.append(0, CHUNK, gk, gv)
                cache.attention(0, gq, mask, out=Ob)
            else:
                uly.step(0, CHUNK, gq, gk, gv, mask, out=Ob)
            ev_comp[b].record(st)
            s_out.wait_event(ev_comp[b])
            with torch.cuda.stream(s_out):
                hO[b].copy_(Ob, non_blocking=True)
                ev_out[b].record(s_out)

    e2e_run(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    e2e_run(args.steps)
    e1.record(s_out)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv)) * world
    e2e = {"value": T_C / (e2e_ms * 1e-3), "unit": "query-tokens/s", "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(hO[0].numel() * 2 * world),
           "note": "bytes summed over ranks; pinned host buffers, every step's copies inside the timed region; "
                   "steps pipelined (H2D of step i on a copy stream during step i-1's compute, D2H on a third "
                   "stream), timed from the first H2D to the last D2H"}

    hbm, tf_burst, tf_sus, src = peaks()
    flops = 4.0 * T_C * nk * D * H
    out = {"metric": METRIC, "value": value, "unit": "query-tokens/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "fp16",
           "dtype_detail": "NVFP4 KV cache (e2m1 codes, e4m3 block scales, fp32 tensor scales); tensor-core "
           "MMA in fp16 with fp32 accumulate; bf16 Q/K/V in, bf16 O out",
           "data": "synthetic (seeded SplitMix64 -> Box-Muller N(0,1) -> bf16; no weights needed)",
           "config": {"workload": WORKLOAD, "heads": H, "head_dim": D, "T_c": T_C, "tokens_per_frame": TPF,
                      "frames_per_chunk": T_FRAMES, "sink_frames": SINK, "window_frames": WINDOW,
                      "n_keys": nk, "chunk_index": CHUNK, "parallelism": f"ulysses-heads{world}" if world > 1 else "1 GPU",
                      "exchange": args.exchange if world > 1 else None,
                      "l2": "flushed (256 MiB write) before every timed step"},
           # per step: N=1 quantize/append (1) + attention (1) + split-KV combine (1);
           # N>1 bf16 adds amax + pack, unpack Q/K/V and unpack O (NCCL kernels not counted); nvfp4: amax (2-3),
           # reduce, pack, scatter, attention + combine, unpack O; peer: amax (2-3), reduce, publish, pack, scatter,
           # attention + combine, signal, pull
           "gpu_launches": args.steps * (3 if world == 1 else {"bf16": 7, "nvfp4": 8, "nvfp4q": 11, "peer": 10, "native": 7,
                                                                       "native-nvfp4": 8}[args.exchange])}
    if uly is None:
        # the attention launch (+ its split-KV combine) as it runs inside the timed steps: CUDA events
        # between the append and the end of every timed step
        att_ms = float(np.mean([ev_mid[i].elapsed_time(ev[i][1]) for i in range(args.steps)]))
        att_ms_iso = float(np.mean([a.elapsed_time(b) for a, b in ev_att]))
        app_ms_ev = float(np.mean([a.elapsed_time(b) for a, b in ev_app]))
        # the append alone is ~10 us: time it as N_APP appends captured in one CUDA graph (removes the
        # host launch cost an event pair around one python call would include).  The appends cycle
        # through a pool of 6 distinct K/V chunks (6 x 28.75 MB = 172 MB > the 126 MB L2), so each
        # append reads its inputs from HBM, not from the previous append's L2-resident copy; L2 is
        # also flushed before every replay.
        gen = torch.Generator(device=dev)
        gen.manual_seed(0x4C4C32)
        pool = [(torch.randn(k6.shape, generator=gen, device=dev).to(torch.bfloat16),
                 torch.randn(v6.shape, generator=gen, device=dev).to(torch.bfloat16)) for _ in range(6)]
        n_app = 24
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(st)
        with torch.cuda.stream(side):
            cache.append(0, CHUNK, *pool[0])
        st.wait_stream(side)
        with torch.cuda.graph(g):
            for i in range(n_app):
                cache.append(0, CHUNK, *pool[i % len(pool)])
        gs = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            torch.cuda.synchronize()
            gs.append(e0.elapsed_time(e1) / n_app)
        app_ms = float(np.median(gs))
        del pool
        cache.append(0, CHUNK, k6, v6)
        ach = flops / (att_ms * 1e-3) / 1e12
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tj = json.load(f)
                traffic = tj.get("attn_ws_kernel", {}).get("bytes")
                traffic_app = tj.get("quant_sp_kernel", {}).get("bytes")
        except Exception:
            traffic_app = None
        # the same call back to back for >= 2 s (clocks sampled), against the SUSTAINED peak
        sus = sustained_attention(cache, q6, mask, O, st, local, seconds=args.sustain_s)
        sus["achieved"] = flops / (sus["ms"] * 1e-3) / 1e12
        sus["peak"] = tf_sus
        sus["frac"] = sus["achieved"] / tf_sus
        sus["peak_source"] = f"{src} bf16_tflops_sustained"
        out["roofline"] = {"bound": "tensor", "kernel": "attn_ws_kernel + combine_kernel (fused dequant, QK^T, "
                           "online softmax, PV on tcgen05)", "achieved": ach, "peak": tf_burst, "unit": "TFLOP/s",
                           "frac": ach / tf_burst, "traffic": traffic,
                           "peak_source": f"{src} bf16_tflops (burst: the launch is timed inside each of the "
                                          f"{args.steps} short timed steps; fp16 kind::f16 runs at the bf16 rate)",
                           "ms": att_ms, "timing": "CUDA events on the launching stream between the append and the "
                                                   "end of every timed step (L2 flushed before each step)",
                           "ms_isolated": att_ms_iso,
                           "ms_isolated_timing": "the call alone, 256 MiB zero-fill (dirty L2) immediately before it",
                           "flops_per_launch": flops,
                           "algorithmic_flops": "4 * T_c * |K_eff| * d * H", "sustained": sus}
        app_bytes = T_C * H * D * 2 * (2 + 9 / 16)
        out["roofline_append"] = {"bound": "hbm", "kernel": "quant_sp_kernel (single-pass quantize/append)",
                                  "achieved": app_bytes / (app_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                                  "frac": app_bytes / (app_ms * 1e-3) / 1e9 / hbm, "us": app_ms * 1e3,
                                  "us_event_single_call": app_ms_ev * 1e3, "traffic": traffic_app,
                                  "algorithmic_bytes": app_bytes,
                                  "timing": f"CUDA graph of {n_app} appends cycling 6 distinct K/V chunks "
                                            "(172 MB > L2, inputs read from HBM), L2 flushed before each replay"}
        out["kv_stream_gbs"] = 2 * nk * H * D * 9 / 16 / (att_ms * 1e-3) / 1e9
        out["attention_tflops"] = ach
        if not args.no_rollout:
            del flush
            torch.cuda.empty_cache()
            out.update(rollout_w30(dev))
    else:
        # per-phase breakdown of one distributed layer step (CUDA events per phase, median of 5 steps,
        # max over ranks) -- SURVEY.md §8(d) D5
        bd = uly.breakdown(lambda: step(CHUNK, O)) if not native else {"step": step_ms}
        names = list(bd)
        tb = torch.tensor([bd[n] for n in names], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        out["breakdown_ms"] = {n: float(v) for n, v in zip(names, tb.tolist())}
        out["breakdown_ms"]["note"] = "per phase, median of 5 steps, max over ranks; exchange " + args.exchange
        # multi-GPU: the whole distributed layer step against the tensor roofline of all N GPUs
        ach = flops / (step_ms * 1e-3) / 1e12
        out["roofline"] = {"bound": "tensor", "kernel": "whole head-sharded layer step (pack, NCCL all-to-all, "
                           "append, attention, all-to-all, unpack), max over ranks", "achieved": ach,
                           "peak": tf_sus * world, "unit": "TFLOP/s", "frac": ach / (tf_sus * world), "traffic": None,
                           "peak_source": f"{src} bf16_tflops_sustained x {world} GPUs",
                           "head_split": [kvq.head_partition(H, P, r) for r in range(P)]}
    out["e2e"] = e2e
    out["clocks"] = clk.summary()
    if rank == 0 and world == 1 and not args.no_cpu:
        ostep = OracleStep()
        t_full = ostep.full()
        t_smp = ostep.sample()
        out["cpu_baseline"] = {"value": T_C / t_full, "unit": "query-tokens/s", "cores": cpu_cores(), "kind": "oracle",
                               "sample": OracleStep.FULL_DESC, "step_s": t_full,
                               "per_head_sample": {"value": T_C / t_smp, "step_s": t_smp,
                                                   "desc": OracleStep.SAMPLE_DESC + " (the --impl reference step)"}}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1 or force:
        dist.barrier()
        if native:
            uly.close()
        dist.destroy_process_group()


def run_reference(args):
    """The oracle arm: each step is OracleStep.sample() (the per-head share of one full step, x12)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    ostep = OracleStep()
    setup = time.perf_counter() - t0
    for _ in range(args.warmup):
        ostep.sample()
    t0 = time.perf_counter()
    ts = [ostep.sample() / H for _ in range(args.steps)]   # actual seconds of each sample
    wall = time.perf_counter() - t0
    t_s = float(np.mean(ts))
    v = (T_C / H) / t_s       # one sample = one head's share: T_C/H query-token equivalents
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "query-tokens/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_s * 1e3, "higher_is_better": True,
           "step_definition": "one step = the per-head share (1/12) of one layer step; value counts it as "
                              "T_c/12 query tokens (each query token carries all 12 heads)",
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64 (CPU oracle)",
           "data": "synthetic (same seeded inputs)", "config": {"workload": WORKLOAD, "heads": H, "head_dim": D,
                                                                 "T_c": T_C, "n_keys": n_keys()},
           "cpu_baseline": {"value": v, "unit": "query-tokens/s", "cores": cpu_cores(), "kind": "oracle",
                            "sample": OracleStep.SAMPLE_DESC + "; each bench step is one such sample",
                            "wall_s": wall, "setup_s": setup},
           "e2e": {"value": v, "unit": "query-tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kvq", choices=["kvq", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle timing")
    ap.add_argument("--no-rollout", action="store_true", help="skip the W30 / L240 keys")
    ap.add_argument("--sustain-s", type=float, default=2.0, help="seconds of the back-to-back attention loop")
    ap.add_argument("--force-ulysses", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--exchange", default="bf16", choices=["bf16", "nvfp4", "nvfp4q", "peer", "native", "native-nvfp4"],
                    help="N>1: bf16 all-to-all (NCCL), nvfp4 = §8(f) f3 (K/V quantized on the sender, NCCL), "
                         "nvfp4q = nvfp4 with Q cast to NVFP4 too (PAPER.md:646; a different numerics mode), "
                         "peer = §8(f) f4 (the kernels store/load over NVLink peer memory, no NCCL on the data path), "
                         "native / native-nvfp4 = the bf16 / nvfp4 exchange behind the one C call "
                         "ulysses_chunk_attention with libkvq's own NCCL communicator")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
