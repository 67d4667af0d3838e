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
def oracle_sample(q_rows=16, quant_frac=8):
    """Time the oracle (as it stands) on a bounded sample of one step; returns (est step s, desc)."""
    from oracle import nvfp4
    from oracle.attention import attention
    from oracle.keyset import key_token_ranges
    from paper_2605_18739_b200 import synth

    q, k, v = synth.make_qkv(T_C, H, D, "bf16", 0, CHUNK)
    rows = T_C // quant_frac
    t0 = time.perf_counter()
    nvfp4.quantize_kv_chunk(k.f64[:rows])
    nvfp4.quantize_kv_chunk(v.f64[:rows])
    t_quant = (time.perf_counter() - t0) * quant_frac
    # dequantize the window (7 chunks of K and V) -- one chunk timed, x7
    qk = nvfp4.quantize_kv_chunk(k.f64)
    t0 = time.perf_counter()
    Kc = nvfp4.dequantize_kv_chunk(qk, T_C, H, D)
    t_deq = (time.perf_counter() - t0) * 2 * (n_keys() // T_C)
    nk = n_keys()
    Kw = np.concatenate([Kc] * (nk // T_C))
    rows_idx = np.linspace(0, T_C - 1, q_rows).astype(int)
    t0 = time.perf_counter()
    attention(q.f64, Kw, Kw, rows=rows_idx)
    t_att = (time.perf_counter() - t0) * T_C / q_rows
    est = t_quant + t_deq + t_att
    desc = (f"quantize {rows} of {T_C} tokens (x{quant_frac}) + dequantize 1 of {2 * nk // T_C} window chunk "
            f"tensors (x{2 * nk // T_C}) + attention for {q_rows} of {T_C} query rows over {nk} keys "
            f"(x{T_C // q_rows}); extrapolated to one full step")
    return est, desc


# ----------------------------------------------------------------------------- GPU leg
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

    cache = kvq.KVCache(1, Hr, D, TPF, T_FRAMES, sink_frames=SINK, window_frames=WINDOW, max_chunk_slots=8,
                        device=dev)
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
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()                                  # L2 flushed before every step
            ev[i][0].record(st)
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
        att_ms = float(np.mean([a.elapsed_time(b) for a, b in ev_att]))
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
        out["roofline"] = {"bound": "tensor", "kernel": "attn_ws_kernel + combine_kernel (fused dequant, QK^T, "
                           "online softmax, PV on tcgen05)", "achieved": ach, "peak": tf_sus, "unit": "TFLOP/s",
                           "frac": ach / tf_sus, "traffic": traffic,
                           "peak_source": f"{src} bf16_tflops_sustained (fp16 kind::f16 runs at the bf16 rate)",
                           "frac_of_burst": ach / tf_burst, "ms": att_ms, "flops_per_launch": flops,
                           "algorithmic_flops": "4 * T_c * |K_eff| * d * H"}
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
        est, desc = oracle_sample()
        out["cpu_baseline"] = {"value": T_C / est, "unit": "query-tokens/s", "cores": cpu_cores(), "kind": "oracle",
                               "sample": desc, "est_step_s": est}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1 or force:
        dist.barrier()
        if native:
            uly.close()
        dist.destroy_process_group()


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup):
        oracle_sample(q_rows=4, quant_frac=32)
    ts = []
    desc = ""
    t0 = time.perf_counter()
    for _ in range(args.steps):
        est, desc = oracle_sample(q_rows=4, quant_frac=32)
        ts.append(est)
    wall = time.perf_counter() - t0
    est = float(np.mean(ts))
    v = T_C / est
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "query-tokens/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64 (CPU oracle)",
           "data": "synthetic (same seeded inputs)", "config": {"workload": WORKLOAD, "heads": H, "head_dim": D,
                                                                 "T_c": T_C, "n_keys": n_keys()},
           "cpu_baseline": {"value": v, "unit": "query-tokens/s", "cores": cpu_cores(), "kind": "oracle",
                            "sample": desc + "; each bench step is one such sample", "wall_s": wall},
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
