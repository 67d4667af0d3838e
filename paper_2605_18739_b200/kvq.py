"""Thin Python binding of libkvq.so (include/kvq.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch supplies device memory
(the cache arena and all tensors), the current CUDA stream, and -- for the multi-GPU path --
the process group.  There is no CPU fallback: if libkvq.so is missing or fails to load, every
call raises.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libkvq.so")
_lib = None

KVQ_BF16, KVQ_FP32, KVQ_FP16 = 0, 1, 2
_STATUS = {0: "KVQ_OK", -1: "KVQ_EINVAL", -2: "KVQ_ESHAPE", -3: "KVQ_EDTYPE", -4: "KVQ_ENOCHUNK",
           -5: "KVQ_ECAPACITY", -6: "KVQ_ENONFINITE", -7: "KVQ_ERANGE", -8: "KVQ_ECUDA", -9: "KVQ_ENCCL"}


class KVQError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        super().__init__(f"{where}: {_STATUS.get(code, code)} ({code})")


class Config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "num_layers", "num_heads", "head_dim", "tokens_per_frame", "frames_per_chunk", "sink_frames",
        "window_frames", "max_chunk_slots", "scale_mode", "k_smoothing")]


class _Mask(ctypes.Structure):
    _fields_ = [("chunk_index", ctypes.c_int64), ("sink_frames", ctypes.c_int32),
                ("window_frames", ctypes.c_int32), ("shot_start_frame", ctypes.c_int64),
                ("shot_len_frames", ctypes.c_int64)]


@dataclass
class Mask:
    """K_eff(t) = A_g U A_s U KV_[t-W,t) U {chunk t}, all in frames."""
    chunk_index: int
    sink_frames: int
    window_frames: int
    shot_start_frame: int = 0
    shot_len_frames: int = 0

    def _c(self):
        return _Mask(self.chunk_index, self.sink_frames, self.window_frames, self.shot_start_frame,
                     self.shot_len_frames)


_P = ctypes.c_void_p
_SIGS = {
    "kvq_cache_bytes": (ctypes.c_size_t, [ctypes.POINTER(Config)]),
    "kvq_cache_create": (ctypes.c_int, [ctypes.POINTER(Config), _P, ctypes.c_size_t, _P, ctypes.POINTER(_P)]),
    "kvq_cache_destroy": (ctypes.c_int, [_P]),
    "kvq_cache_reset": (ctypes.c_int, [_P, _P]),
    "kvq_set_shot": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int64]),
    "kv_quantize_append": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P, ctypes.c_int, _P]),
    "kv_quantize_append_amax": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P, ctypes.c_int, _P, _P]),
    "chunk_attention": (ctypes.c_int, [_P, ctypes.c_int32, _P, ctypes.c_int, ctypes.POINTER(_Mask), ctypes.c_float,
                                       _P, ctypes.c_int, _P]),
    "chunk_attention_ws": (ctypes.c_int, [_P, ctypes.c_int32, _P, ctypes.c_int, ctypes.POINTER(_Mask), ctypes.c_float,
                                          _P, ctypes.c_int, _P, ctypes.c_size_t, _P]),
    "kvq_attention_workspace_bytes": (ctypes.c_size_t, [_P]),
    "kv_dequantize": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P, ctypes.c_int, _P]),
    "kv_export_chunk": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "kv_export_kmean": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P]),
    "kvq_resident_bytes": (ctypes.c_size_t, [_P]),
    "kvq_resident_chunks": (ctypes.c_int32, [_P, ctypes.c_int32]),
    "kv_dequantize_window": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.POINTER(_Mask), _P, _P,
                                            ctypes.POINTER(ctypes.c_int64), _P]),
    "chunk_attention_bf16kv": (ctypes.c_int, [_P, _P, _P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_float, _P, ctypes.c_int, _P]),
    "kvq_bf16kv_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32]),
    "chunk_attention_append": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P, ctypes.c_int, _P, ctypes.c_int,
                                              ctypes.POINTER(_Mask), ctypes.c_float, _P, ctypes.c_int, _P,
                                              ctypes.c_size_t, _P]),
    "chunk_attention_bf16kv_ws": (ctypes.c_int, [_P, _P, _P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                                 ctypes.c_int32, ctypes.c_float, _P, ctypes.c_int, _P,
                                                 ctypes.c_size_t, _P]),
    "kvq_get_status": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_int64)]),
    "kvq_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "kvq_head_partition": (None, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                  ctypes.POINTER(ctypes.c_int32)]),
    "kvq_ulysses_qkv_bytes": (ctypes.c_size_t, [ctypes.c_int32] * 5 + [ctypes.c_int]),
    "kvq_ulysses_pack_qkv": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32, _P, _P, _P]),
    "kvq_ulysses_unpack_qkv": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, _P, _P, _P, _P, _P]),
    "kvq_ulysses_unpack_o": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32, _P, _P]),
    "kvq_ulysses_shard_scratch_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32]),
    "kvq_ulysses_nvfp4_bytes": (ctypes.c_size_t, [ctypes.c_int32] * 5 + [ctypes.c_int, ctypes.c_int32, ctypes.c_int32]),
    "kvq_ulysses_q_amax": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _P]),
    "chunk_attention_qscaled": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, ctypes.POINTER(_Mask), ctypes.c_float, _P,
                                               ctypes.c_int, _P]),
    "kvq_ulysses_shard_amax": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, _P, _P, _P]),
    "kvq_ulysses_pack_nvfp4": (ctypes.c_int, [_P, _P, _P, ctypes.c_int] + [ctypes.c_int32] * 4 +
                               [_P, _P, ctypes.c_int32, ctypes.c_int32, _P, _P]),
    "kv_append_ulysses_nvfp4": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, ctypes.c_int32, _P, _P, _P,
                                               ctypes.c_int, _P, _P]),
    "kvq_peer_window_bytes": (ctypes.c_size_t, [ctypes.c_int32] * 4 + [ctypes.c_int, ctypes.c_int32]),
    "kvq_peer_create": (ctypes.c_int, [ctypes.c_int32] * 5 + [ctypes.c_int, ctypes.c_int32, ctypes.c_int32,
                                                               ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "kvq_peer_destroy": (ctypes.c_int, [_P]),
    "kvq_peer_o_local": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.POINTER(_P)]),
    "kvq_peer_publish_amax": (ctypes.c_int, [_P, _P, _P, ctypes.c_int64, _P, _P]),
    "kvq_peer_pack": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int64, _P]),
    "kv_append_peer": (ctypes.c_int, [_P, _P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, _P, _P]),
    "kvq_peer_signal_o": (ctypes.c_int, [_P, ctypes.c_int64, _P]),
    "kvq_peer_pull_o": (ctypes.c_int, [_P, ctypes.c_int64, _P, _P]),
    "kvq_peer_bind_caches": (ctypes.c_int, [_P, _P, _P]),
    "kv_append_peer_direct": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _P, _P, _P, ctypes.c_int64, _P]),
    "chunk_attention_peer": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.POINTER(_Mask), ctypes.c_float,
                                            ctypes.c_int64, _P, ctypes.c_size_t, _P]),
    "kvq_peer_wait_o": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.POINTER(_P), _P]),
    "kvq_cache_get_config": (ctypes.c_int, [_P, ctypes.POINTER(Config)]),
    "kvq_get_unique_id": (ctypes.c_int, [_P]),
    "kvq_comm_create": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_P)]),
    "kvq_comm_destroy": (ctypes.c_int, [_P]),
    "kvq_ulysses_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32] * 6 + [ctypes.c_int, ctypes.c_int]),
    "kvq_comm_configure": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, _P, ctypes.c_size_t]),
    "ulysses_chunk_attention": (ctypes.c_int, [_P, _P, ctypes.c_int32, ctypes.c_int64, _P, _P, _P, ctypes.c_int,
                                               ctypes.POINTER(_Mask), ctypes.c_float, _P, ctypes.c_int, _P]),
    "kvq_debug_probe": (ctypes.c_int, [ctypes.c_int32, _P, _P, ctypes.c_int64, _P]),
    "kvq_debug_set_trace": (ctypes.c_int, [_P]),
    "kvq_debug_force_two_pass": (ctypes.c_int, [_P, ctypes.c_int32]),
}


def lib():
    """Load libkvq.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"libkvq.so not built ({_LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(code, where):
    if code != 0:
        raise KVQError(code, where)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dt(t: torch.Tensor):
    if t.dtype == torch.bfloat16:
        return KVQ_BF16
    if t.dtype == torch.float32:
        return KVQ_FP32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _ptr(t: torch.Tensor):
    if not t.is_cuda:
        raise ValueError("tensor must be on a CUDA device")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _out_code(dtype):
    return {torch.bfloat16: KVQ_BF16, torch.float32: KVQ_FP32}[dtype]


class KVCache:
    """Chunkwise NVFP4 KV cache of one rank over a torch-owned arena."""

    def __init__(self, num_layers, num_heads, head_dim, tokens_per_frame, frames_per_chunk,
                 sink_frames=0, window_frames=None, max_chunk_slots=8, device=None,
                 scale_search=False, k_smoothing=False, arena=None):
        """scale_search: Four-Over-Six block scales for K and V;
        k_smoothing: keys stored mean-centred per (t, h), means restored;
        arena: a caller-allocated uint8 device tensor of >= cache_bytes(...) (e.g. torch symmetric
        memory for the f4 direct exchange), else one is allocated."""
        L = lib()
        window_frames = window_frames if window_frames is not None else max_chunk_slots * frames_per_chunk
        self.cfg = Config(num_layers, num_heads, head_dim, tokens_per_frame, frames_per_chunk, sink_frames,
                          window_frames, max_chunk_slots, 1 if scale_search else 0, 1 if k_smoothing else 0)
        self.scale_search, self.k_smoothing = bool(scale_search), bool(k_smoothing)
        nbytes = L.kvq_cache_bytes(ctypes.byref(self.cfg))
        if nbytes == 0:
            raise KVQError(-1, "kvq_cache_bytes (bad config)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        if arena is not None:
            if arena.dtype != torch.uint8 or arena.numel() < nbytes or arena.device != self.device:
                raise KVQError(-1, "arena: uint8 tensor of >= cache bytes on the cache's device")
            self.arena = arena
        else:
            self.arena = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.T_c = tokens_per_frame * frames_per_chunk
        self.H, self.d = num_heads, head_dim
        h = ctypes.c_void_p()
        _check(L.kvq_cache_create(ctypes.byref(self.cfg), _ptr(self.arena), nbytes, _stream(), ctypes.byref(h)),
               "kvq_cache_create")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.kvq_cache_destroy(self._h)
            self._h = None

    @property
    def arena_bytes(self):
        return self.arena.numel()

    def reset(self):
        _check(lib().kvq_cache_reset(self._h, _stream()), "kvq_cache_reset")

    def force_two_pass(self, on=True):
        """Debug: route appends through the amax + quantize two-launch path."""
        _check(lib().kvq_debug_force_two_pass(self._h, 1 if on else 0), "kvq_debug_force_two_pass")

    def set_shot(self, start_frame, len_frames):
        _check(lib().kvq_set_shot(self._h, start_frame, len_frames), "kvq_set_shot")

    def _shape_ok(self, t):
        if tuple(t.shape) != (self.T_c, self.H, self.d):
            raise ValueError(f"expected [{self.T_c}, {self.H}, {self.d}], got {tuple(t.shape)}")

    def append(self, layer, chunk_index, K, V, amax_kv=None):
        """kv_quantize_append (or kv_quantize_append_amax when amax_kv, a 2-float device tensor, is given)."""
        self._shape_ok(K)
        self._shape_ok(V)
        if K.dtype != V.dtype:
            raise TypeError("K and V dtypes differ")
        if amax_kv is None:
            _check(lib().kv_quantize_append(self._h, layer, chunk_index, _ptr(K), _ptr(V), _dt(K), _stream()),
                   "kv_quantize_append")
        else:
            _check(lib().kv_quantize_append_amax(self._h, layer, chunk_index, _ptr(K), _ptr(V), _dt(K),
                                                 _ptr(amax_kv), _stream()), "kv_quantize_append_amax")

    def attention(self, layer, Q, mask: Mask, out_dtype=torch.bfloat16, softmax_scale=0.0, out=None, workspace=None):
        """chunk_attention: O = softmax(Q K^T * scale) V over K_eff(mask) with fused dequant.
        workspace: a tensor from new_attention_workspace() -> chunk_attention_ws (calls running
        concurrently on different streams each need their own)."""
        self._shape_ok(Q)
        if out is None:
            out = torch.empty(Q.shape, dtype=out_dtype, device=Q.device)
        m = mask._c()
        if workspace is None:
            _check(lib().chunk_attention(self._h, layer, _ptr(Q), _dt(Q), ctypes.byref(m), softmax_scale, _ptr(out),
                                         _out_code(out.dtype), _stream()), "chunk_attention")
        else:
            _check(lib().chunk_attention_ws(self._h, layer, _ptr(Q), _dt(Q), ctypes.byref(m), softmax_scale,
                                            _ptr(out), _out_code(out.dtype), _ptr(workspace), workspace.numel(),
                                            _stream()), "chunk_attention_ws")
        return out

    def append_attention(self, layer, chunk_index, K, V, Q, mask: Mask, out_dtype=torch.bfloat16, softmax_scale=0.0,
                         out=None, workspace=None):
        """chunk_attention_append: append chunk `chunk_index`'s K, V and attend its queries in one launch
        (the quantization fused into the attention kernel; falls back to the two calls where not fused)."""
        self._shape_ok(K)
        self._shape_ok(V)
        self._shape_ok(Q)
        if K.dtype != V.dtype:
            raise KVQError(-3, "K and V dtypes differ")
        if out is None:
            out = torch.empty(Q.shape, dtype=out_dtype, device=Q.device)
        m = mask._c()
        _check(lib().chunk_attention_append(self._h, layer, chunk_index, _ptr(K), _ptr(V), _dt(K), _ptr(Q), _dt(Q),
                                            ctypes.byref(m), softmax_scale, _ptr(out), _out_code(out.dtype),
                                            _ptr(workspace) if workspace is not None else None,
                                            workspace.numel() if workspace is not None else 0, _stream()),
               "chunk_attention_append")
        return out

    def new_attention_workspace(self):
        """A caller-owned split-KV workspace of kvq_attention_workspace_bytes (one per concurrent stream)."""
        n = int(lib().kvq_attention_workspace_bytes(self._h))
        return torch.empty(n, dtype=torch.uint8, device=self.device)

    def append_ulysses_nvfp4(self, layer, chunk_index, recv, P, amax_kv, q_dtype=torch.bfloat16, Q_out=None,
                             amax_q=None, q_scale=None):
        """kv_append_ulysses_nvfp4: the P received NVFP4 segments become chunk `chunk_index`; returns Q
        (with amax_q: fp16 dec(c) dec(s), and q_scale [1] receives g_Q)."""
        if Q_out is None:
            Q_out = torch.empty((self.T_c, self.H, self.d), dtype=torch.float16 if amax_q is not None else q_dtype,
                                device=self.device)
        if amax_q is not None and q_scale is None:
            q_scale = torch.empty(1, dtype=torch.float32, device=self.device)
        qd = q_dtype if amax_q is not None else Q_out.dtype
        _check(lib().kv_append_ulysses_nvfp4(self._h, layer, chunk_index, _ptr(recv), P, _ptr(amax_kv),
                                             _ptr(amax_q) if amax_q is not None else None, _ptr(Q_out), _out_code(qd),
                                             _ptr(q_scale) if q_scale is not None else None, _stream()),
               "kv_append_ulysses_nvfp4")
        return (Q_out, q_scale) if amax_q is not None else Q_out

    def attention_qscaled(self, layer, Q16, q_scale, mask: Mask, out_dtype=torch.bfloat16, softmax_scale=0.0, out=None):
        """chunk_attention_qscaled: attention for NVFP4-exchanged queries (fp16 dec(c) dec(s), scale g_Q)."""
        self._shape_ok(Q16)
        if out is None:
            out = torch.empty(Q16.shape, dtype=out_dtype, device=Q16.device)
        m = mask._c()
        _check(lib().chunk_attention_qscaled(self._h, layer, _ptr(Q16), _ptr(q_scale), ctypes.byref(m), softmax_scale,
                                             _ptr(out), _out_code(out.dtype), _stream()), "chunk_attention_qscaled")
        return out

    def dequantize(self, layer, chunk_index, out_dtype=torch.float32):
        K = torch.empty((self.T_c, self.H, self.d), dtype=out_dtype, device=self.device)
        V = torch.empty_like(K)
        _check(lib().kv_dequantize(self._h, layer, chunk_index, _ptr(K), _ptr(V), _out_code(out_dtype), _stream()),
               "kv_dequantize")
        return K, V

    def export(self, layer, chunk_index):
        rows = self.T_c * self.H
        dev = self.device
        out = {k: torch.empty((rows, self.d // 2), dtype=torch.uint8, device=dev) for k in ("codes_k", "codes_v")}
        out.update({k: torch.empty((rows, self.d // 16), dtype=torch.uint8, device=dev) for k in ("scales_k", "scales_v")})
        out.update({k: torch.empty(1, dtype=torch.float32, device=dev) for k in ("g_k", "g_v")})
        _check(lib().kv_export_chunk(self._h, layer, chunk_index, _ptr(out["codes_k"]), _ptr(out["scales_k"]),
                                     _ptr(out["g_k"]), _ptr(out["codes_v"]), _ptr(out["scales_v"]), _ptr(out["g_v"]),
                                     _stream()), "kv_export_chunk")
        return out

    def export_kmean(self, layer, chunk_index):
        """K-smoothing row means of a resident chunk, fp32 [T_c*H] (t, h) t-major."""
        out = torch.empty(self.T_c * self.H, dtype=torch.float32, device=self.device)
        _check(lib().kv_export_kmean(self._h, layer, chunk_index, _ptr(out), _stream()), "kv_export_kmean")
        return out

    def n_keys(self, layer, mask: Mask):
        n = ctypes.c_int64()
        m = mask._c()
        _check(lib().kv_dequantize_window(self._h, layer, ctypes.byref(m), None, None, ctypes.byref(n), _stream()),
               "kv_dequantize_window")
        return n.value

    def dequantize_window(self, layer, mask: Mask, K_out=None, V_out=None):
        """The paper's unfused reconstruction of K_eff into contiguous bf16 (bench comparison)."""
        n = self.n_keys(layer, mask)
        if K_out is None:
            K_out = torch.empty((n, self.H, self.d), dtype=torch.bfloat16, device=self.device)
            V_out = torch.empty_like(K_out)
        nk = ctypes.c_int64()
        m = mask._c()
        _check(lib().kv_dequantize_window(self._h, layer, ctypes.byref(m), _ptr(K_out), _ptr(V_out),
                                          ctypes.byref(nk), _stream()), "kv_dequantize_window")
        return K_out, V_out

    def resident_bytes(self):
        return int(lib().kvq_resident_bytes(self._h))

    def resident_chunks(self, layer):
        return int(lib().kvq_resident_chunks(self._h, layer))

    def status(self):
        idx = ctypes.c_int64()
        code = lib().kvq_get_status(self._h, _stream(), ctypes.byref(idx))
        return code, idx.value


def new_bf16kv_workspace(d, device="cuda"):
    """A caller-owned workspace of kvq_bf16kv_workspace_bytes(d) for chunk_attention_bf16kv(workspace=...)."""
    n = int(lib().kvq_bf16kv_workspace_bytes(d))
    return torch.empty(n, dtype=torch.uint8, device=device)


def chunk_attention_bf16kv(Q, K, V, out_dtype=torch.bfloat16, softmax_scale=0.0, out=None, workspace=None):
    """Attention over caller-provided bf16 K/V [n_keys, H, d] (the A12 bf16-KV comparison mode).
    workspace (new_bf16kv_workspace): the persistent wave + stream-K grid (chunk_attention_bf16kv_ws)."""
    Tq, H, d = Q.shape
    if out is None:
        out = torch.empty(Q.shape, dtype=out_dtype, device=Q.device)
    if workspace is None:
        _check(lib().chunk_attention_bf16kv(_ptr(Q), _ptr(K), _ptr(V), Tq, K.shape[0], H, d, softmax_scale,
                                            _ptr(out), _out_code(out.dtype), _stream()), "chunk_attention_bf16kv")
    else:
        _check(lib().chunk_attention_bf16kv_ws(_ptr(Q), _ptr(K), _ptr(V), Tq, K.shape[0], H, d, softmax_scale,
                                               _ptr(out), _out_code(out.dtype), _ptr(workspace), workspace.numel(),
                                               _stream()), "chunk_attention_bf16kv_ws")
    return out


def probe(which, x, n):
    """kvq_debug_probe: run one hardware NVFP4 conversion over a device buffer (codec checks)."""
    out_shape = {0: (2 * n,), 1: (n,), 2: (2 * n,), 3: (n,)}[which]
    out_dtype = {0: torch.uint8, 1: torch.uint8, 2: torch.float32, 3: torch.float32}[which]
    out = torch.empty(out_shape, dtype=out_dtype, device=x.device)
    _check(lib().kvq_debug_probe(which, _ptr(x), _ptr(out), n, _stream()), "kvq_debug_probe")
    return out


def head_partition(H, P, rank):
    h0, h1 = ctypes.c_int32(), ctypes.c_int32()
    lib().kvq_head_partition(H, P, rank, ctypes.byref(h0), ctypes.byref(h1))
    return h0.value, h1.value


def ulysses_qkv_bytes(Ts, H, d, P, dst, dtype=torch.bfloat16):
    return int(lib().kvq_ulysses_qkv_bytes(Ts, H, d, P, dst, _out_code(dtype)))


def ulysses_pack(Q, K, V, P, send=None, scratch=None):
    """kvq_ulysses_pack_qkv: this rank's shards [Ts, H, d] -> the all-to-allv send buffer (u8)."""
    Ts, H, d = Q.shape
    sizes = [ulysses_qkv_bytes(Ts, H, d, P, p, Q.dtype) for p in range(P)]
    if send is None:
        send = torch.empty(sum(sizes), dtype=torch.uint8, device=Q.device)
    if scratch is None:
        scratch = torch.empty(8192, dtype=torch.uint8, device=Q.device)
    _check(lib().kvq_ulysses_pack_qkv(_ptr(Q), _ptr(K), _ptr(V), _dt(Q), Ts, H, d, P, _ptr(send), _ptr(scratch),
                                      _stream()), "kvq_ulysses_pack_qkv")
    return send, sizes


def ulysses_unpack_qkv(recv, Ts, Hr, d, P, dtype=torch.bfloat16):
    """kvq_ulysses_unpack_qkv: P received segments -> Q, K, V [P*Ts, Hr, d] + global amax (K, V)."""
    Q = torch.empty((P * Ts, Hr, d), dtype=dtype, device=recv.device)
    K, V = torch.empty_like(Q), torch.empty_like(Q)
    amax = torch.empty(2, dtype=torch.float32, device=recv.device)
    _check(lib().kvq_ulysses_unpack_qkv(_ptr(recv), _out_code(dtype), Ts, Hr, d, P, _ptr(Q), _ptr(K), _ptr(V),
                                        _ptr(amax), _stream()), "kvq_ulysses_unpack_qkv")
    return Q, K, V, amax


def ulysses_unpack_o(recv, Ts, H, d, P, dtype=torch.bfloat16, out=None):
    """kvq_ulysses_unpack_o: P received O token blocks [Ts, H_p, d] -> this rank's O shard [Ts, H, d]."""
    if out is None:
        out = torch.empty((Ts, H, d), dtype=dtype, device=recv.device)
    _check(lib().kvq_ulysses_unpack_o(_ptr(recv), _out_code(dtype), Ts, H, d, P, _ptr(out), _stream()),
           "kvq_ulysses_unpack_o")
    return out


def ulysses_nvfp4_bytes(Ts, H, d, P, dst, q_dtype=torch.bfloat16, k_smoothing=False, q_nvfp4=False):
    return int(lib().kvq_ulysses_nvfp4_bytes(Ts, H, d, P, dst, _out_code(q_dtype), int(k_smoothing), int(q_nvfp4)))


def ulysses_q_amax(Q, out=None, scratch=None):
    """kvq_ulysses_q_amax: max |Q| of this rank's shard (dev fp32[1])."""
    Ts, H, d = Q.shape
    if out is None:
        out = torch.empty(1, dtype=torch.float32, device=Q.device)
    if scratch is None:
        scratch = torch.empty(int(lib().kvq_ulysses_shard_scratch_bytes(Ts, H)), dtype=torch.uint8, device=Q.device)
    _check(lib().kvq_ulysses_q_amax(_ptr(Q), _dt(Q), Ts, H, d, _ptr(out), _ptr(scratch), _stream()),
           "kvq_ulysses_q_amax")
    return out


def ulysses_shard_amax(K, V, k_smoothing=False, out=None, scratch=None):
    """kvq_ulysses_shard_amax: [max |K| (|K - row mean| with smoothing), max |V|] of this rank's shard."""
    Ts, H, d = K.shape
    if out is None:
        out = torch.empty(2, dtype=torch.float32, device=K.device)
    if scratch is None:
        scratch = torch.empty(int(lib().kvq_ulysses_shard_scratch_bytes(Ts, H)), dtype=torch.uint8, device=K.device)
    _check(lib().kvq_ulysses_shard_amax(_ptr(K), _ptr(V), _dt(K), Ts, H, d, int(k_smoothing), _ptr(out),
                                        _ptr(scratch), _stream()), "kvq_ulysses_shard_amax")
    return out


def ulysses_pack_nvfp4(Q, K, V, P, amax_kv, scale_search=False, k_smoothing=False, send=None, amax_q=None):
    """kvq_ulysses_pack_nvfp4: shard -> send buffer with K/V (and Q when amax_q is given) as NVFP4 under
    the GLOBAL amaxes."""
    Ts, H, d = Q.shape
    sizes = [ulysses_nvfp4_bytes(Ts, H, d, P, p, Q.dtype, k_smoothing, amax_q is not None) for p in range(P)]
    if send is None:
        send = torch.empty(sum(sizes), dtype=torch.uint8, device=Q.device)
    _check(lib().kvq_ulysses_pack_nvfp4(_ptr(Q), _ptr(K), _ptr(V), _dt(Q), Ts, H, d, P, _ptr(amax_kv),
                                        _ptr(amax_q) if amax_q is not None else None, int(bool(scale_search)),
                                        int(bool(k_smoothing)), _ptr(send), _stream()), "kvq_ulysses_pack_nvfp4")
    return send, sizes


def cache_bytes(num_layers, num_heads, head_dim, tokens_per_frame, frames_per_chunk, sink_frames=0,
                window_frames=None, max_chunk_slots=8, scale_search=False, k_smoothing=False):
    """kvq_cache_bytes: device arena bytes of a KVCache with this geometry (e.g. to allocate it in
    torch symmetric memory for the f4 direct exchange)."""
    window_frames = window_frames if window_frames is not None else max_chunk_slots * frames_per_chunk
    cfg = Config(num_layers, num_heads, head_dim, tokens_per_frame, frames_per_chunk, sink_frames, window_frames,
                 max_chunk_slots, 1 if scale_search else 0, 1 if k_smoothing else 0)
    return int(lib().kvq_cache_bytes(ctypes.byref(cfg)))


def peer_window_bytes(T_c, H, d, P, q_dtype=torch.bfloat16, k_smoothing=False):
    return int(lib().kvq_peer_window_bytes(T_c, H, d, P, _out_code(q_dtype), int(k_smoothing)))


class PeerExchange:
    """§8(f) f4: the NVFP4 exchange as device-initiated stores/loads over peer memory (include/kvq.h).
    `window_ptrs`: the P ranks' window base addresses as seen from this rank (ints)."""

    def __init__(self, T_c, H, d, P, rank, window_ptrs, q_dtype=torch.bfloat16, scale_search=False,
                 k_smoothing=False, device="cuda"):
        self.T_c, self.H, self.d, self.P, self.rank = T_c, H, d, P, rank
        self.Ts = T_c // P
        self.h0, self.h1 = head_partition(H, P, rank)
        arr = (_P * P)(*[ctypes.c_void_p(int(w)) for w in window_ptrs])
        self._arr = arr
        h = _P()
        _check(lib().kvq_peer_create(T_c, H, d, P, rank, _out_code(q_dtype), int(bool(scale_search)),
                                     int(bool(k_smoothing)), arr, ctypes.byref(h)), "kvq_peer_create")
        self._h = h
        self.q_dtype = q_dtype
        self.scratch = torch.empty(int(lib().kvq_ulysses_shard_scratch_bytes(self.Ts, H)) + 16, dtype=torch.uint8,
                                   device=device)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().kvq_peer_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def o_local(self, epoch):
        ptr = _P()
        _check(lib().kvq_peer_o_local(self._h, epoch, ctypes.byref(ptr)), "kvq_peer_o_local")
        return ptr.value

    def publish_amax(self, K, V, epoch):
        _check(lib().kvq_peer_publish_amax(self._h, _ptr(K), _ptr(V), epoch, _ptr(self.scratch), _stream()),
               "kvq_peer_publish_amax")

    def pack(self, Q, K, V, epoch):
        _check(lib().kvq_peer_pack(self._h, _ptr(Q), _ptr(K), _ptr(V), epoch, _stream()), "kvq_peer_pack")

    def append(self, cache, layer, chunk_index, epoch, Q_out):
        _check(lib().kv_append_peer(self._h, cache._h, layer, chunk_index, epoch, _ptr(Q_out), _stream()),
               "kv_append_peer")
        return Q_out

    def signal_o(self, epoch):
        _check(lib().kvq_peer_signal_o(self._h, epoch, _stream()), "kvq_peer_signal_o")

    def pull_o(self, epoch, out):
        _check(lib().kvq_peer_pull_o(self._h, epoch, _ptr(out), _stream()), "kvq_peer_pull_o")
        return out

    # ---- f4 direct (include/kvq.h): owners' cache slots and O shards written in place
    def bind_caches(self, cache, arena_ptrs):
        """cache: this rank's KVCache; arena_ptrs: the P ranks' cache arena addresses seen from here."""
        arr = (_P * self.P)(*[ctypes.c_void_p(int(a)) for a in arena_ptrs])
        _check(lib().kvq_peer_bind_caches(self._h, cache._h, arr), "kvq_peer_bind_caches")
        self.cache = cache

    def append_direct(self, layer, chunk_index, Q, K, V, epoch):
        _check(lib().kv_append_peer_direct(self._h, layer, chunk_index, _ptr(Q), _ptr(K), _ptr(V), epoch, _stream()),
               "kv_append_peer_direct")

    def attention_direct(self, layer, mask, epoch, softmax_scale=0.0, workspace=None):
        m = mask._c()
        _check(lib().chunk_attention_peer(self._h, layer, ctypes.byref(m), softmax_scale, epoch,
                                          _ptr(workspace) if workspace is not None else None,
                                          workspace.numel() if workspace is not None else 0, _stream()),
               "chunk_attention_peer")

    def wait_o(self, epoch):
        """Address of this rank's O shard [T_c/P, H, d] bf16 for `epoch` (inside its window)."""
        ptr = _P()
        _check(lib().kvq_peer_wait_o(self._h, epoch, ctypes.byref(ptr), _stream()), "kvq_peer_wait_o")
        return ptr.value


class Ulysses:
    """Head-sharded chunk step of one rank (App. C; App. D).

    pack (kernel) -> all_to_all_single (NCCL, torch.distributed) -> unpack + global amax (kernel)
    -> kv_quantize_append_amax + chunk_attention on the local heads (kernels) -> all_to_all_single
    of O (NCCL) -> head interleave (kernel).
    """

    def __init__(self, cache: KVCache, H, d, T_c, rank, world, group=None, dtype=torch.bfloat16, nvfp4_kv=False,
                 peer=False, nvfp4_q=False):
        """nvfp4_kv (§8(f) f3): ship K/V as NVFP4 bytes quantized on the sender with
        the all-reduced global amax (one extra tiny NCCL all-reduce; ~3.6x less K/V volume).
        peer (§8(f) f4): the same payload moved by the kernels themselves over NVLink peer memory
        (torch symmetric memory windows; no NCCL on the data path).
        nvfp4_q (with nvfp4_kv): Q is cast to NVFP4 before the all-to-all too -- the
        attention then sees the quantized Q (a different numerics mode, reading Z24)."""
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.cache, self.H, self.d, self.T_c = cache, H, d, T_c
        self.rank, self.P = rank, world
        if T_c % world:
            raise ValueError("T_c must be divisible by the SP degree")
        self.Ts = T_c // world
        self.h0, self.h1 = head_partition(H, world, rank)
        self.Hr = self.h1 - self.h0
        if cache.H != self.Hr:
            raise ValueError("cache must hold exactly this rank's heads")
        dev = cache.device
        es = 2 if dtype == torch.bfloat16 else 4
        self.dtype = dtype
        self.send_sizes = [ulysses_qkv_bytes(self.Ts, H, d, world, p, dtype) for p in range(world)]
        self.recv_seg = ulysses_qkv_bytes(self.Ts, H, d, world, rank, dtype)
        self.send = torch.empty(sum(self.send_sizes), dtype=torch.uint8, device=dev)
        self.recv = torch.empty(self.recv_seg * world, dtype=torch.uint8, device=dev)
        self.scratch = torch.empty(8192, dtype=torch.uint8, device=dev)
        self.Q = torch.empty((T_c, self.Hr, d), dtype=dtype, device=dev)
        self.K = torch.empty_like(self.Q)
        self.V = torch.empty_like(self.Q)
        self.amax = torch.empty(2, dtype=torch.float32, device=dev)
        self.O_local = torch.empty((T_c, self.Hr, d), dtype=torch.bfloat16, device=dev)
        self.o_recv_sizes = [self.Ts * (head_partition(H, world, p)[1] - head_partition(H, world, p)[0]) * d * 2
                             for p in range(world)]
        self.o_recv = torch.empty(sum(self.o_recv_sizes), dtype=torch.uint8, device=dev)
        self.es = es
        self.marks = None
        self.peer = None
        if peer:
            import torch.distributed._symmetric_memory as symm_mem
            grp = group if group is not None else dist.group.WORLD
            wb = peer_window_bytes(T_c, H, d, world, dtype, cache.k_smoothing)
            self.win = symm_mem.empty(wb, dtype=torch.uint8, device=dev)
            self.win.zero_()
            hdl = symm_mem.rendezvous(self.win, grp)
            self.peer = PeerExchange(T_c, H, d, world, rank, list(hdl.buffer_ptrs), dtype, cache.scale_search,
                                     cache.k_smoothing, device=dev)
            # f4 direct: every rank's cache arena must be peer-accessible (torch symmetric memory)
            try:
                ahdl = symm_mem.rendezvous(cache.arena, grp)
            except Exception as e:
                raise ValueError("the peer exchange stores into the owners' caches: create the KVCache with "
                                 "arena=symm_mem.empty(cache_bytes(...))") from e
            self.peer.bind_caches(cache, list(ahdl.buffer_ptrs))
            self.epoch = 0
            torch.cuda.synchronize(dev)
            dist.barrier(group=grp)
        # K-smoothing needs the amax of K_bar, which the bf16 exchange's piggybacked shard amax is not
        self.nvfp4_q = bool(nvfp4_q)
        self.nvfp4_kv = bool(nvfp4_kv) or cache.k_smoothing or self.nvfp4_q
        if self.nvfp4_kv:
            sm, qn = cache.k_smoothing, self.nvfp4_q
            self.nv_send_sizes = [ulysses_nvfp4_bytes(self.Ts, H, d, world, p, dtype, sm, qn) for p in range(world)]
            self.nv_recv_seg = ulysses_nvfp4_bytes(self.Ts, H, d, world, rank, dtype, sm, qn)
            self.amax3 = torch.empty(3, dtype=torch.float32, device=dev)  # [K, V, Q] all-reduced together
            if qn:
                self.Q16 = torch.empty((T_c, self.Hr, d), dtype=torch.float16, device=dev)
                self.q_scale = torch.empty(1, dtype=torch.float32, device=dev)
            self.nv_send = torch.empty(sum(self.nv_send_sizes), dtype=torch.uint8, device=dev)
            self.nv_recv = torch.empty(self.nv_recv_seg * world, dtype=torch.uint8, device=dev)
            self.amax_scratch = torch.empty(int(lib().kvq_ulysses_shard_scratch_bytes(self.Ts, H)), dtype=torch.uint8,
                                            device=dev)

    def _mark(self, name):
        """Phase boundary for the per-phase breakdown (CUDA event on the current stream) when
        self.marks is a list; a no-op otherwise."""
        if self.marks is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.marks.append((name, e))

    def step(self, layer, chunk_index, Q, K, V, mask: Mask, out=None):
        """One layer of one chunk: Q, K, V are this rank's sequence shards [T_c/P, H, d]."""
        L, st = lib(), _stream()
        dt = _dt(Q)
        self._mark("start")
        if self.peer is not None:  # f4 direct: amax mailbox -> owners' cache slots -> attention -> owners' O
            self.epoch += 1
            ep, pe = self.epoch, self.peer
            pe.publish_amax(K, V, ep)
            self._mark("amax_publish")
            pe.append_direct(layer, chunk_index, Q, K, V, ep)
            self._mark("quantize_store_to_owners")
            pe.attention_direct(layer, mask, ep)
            self._mark("attention_o_to_owners")
            off = pe.wait_o(ep) - self.win.data_ptr()
            n = self.Ts * self.H * self.d * 2
            O_sh = self.win[off:off + n].view(torch.bfloat16).view(self.Ts, self.H, self.d)
            self._mark("o_wait")
            if out is None:
                return O_sh  # valid until this rank's step after next (epoch + 2)
            out.copy_(O_sh)
            return out
        if self.nvfp4_kv:
            c, qn = self.cache, self.nvfp4_q
            ulysses_shard_amax(K, V, c.k_smoothing, out=self.amax3[:2], scratch=self.amax_scratch)
            if qn:
                ulysses_q_amax(Q, out=self.amax3[2:], scratch=self.amax_scratch)
            self._mark("shard_amax")
            self.dist.all_reduce(self.amax3, op=self.dist.ReduceOp.MAX, group=self.group)
            self._mark("amax_allreduce")
            aq = self.amax3[2:] if qn else None
            ulysses_pack_nvfp4(Q, K, V, self.P, self.amax3, c.scale_search, c.k_smoothing, send=self.nv_send, amax_q=aq)
            self._mark("quantize_pack")
            self.dist.all_to_all_single(self.nv_recv, self.nv_send, output_split_sizes=[self.nv_recv_seg] * self.P,
                                        input_split_sizes=self.nv_send_sizes, group=self.group)
            self._mark("a2a_in")
            if qn:
                c.append_ulysses_nvfp4(layer, chunk_index, self.nv_recv, self.P, self.amax3, q_dtype=Q.dtype,
                                       Q_out=self.Q16, amax_q=aq, q_scale=self.q_scale)
            else:
                c.append_ulysses_nvfp4(layer, chunk_index, self.nv_recv, self.P, self.amax3, Q_out=self.Q)
            self._mark("scatter_append")
            return self._attend_and_return(layer, mask, out, Q)
        _check(L.kvq_ulysses_pack_qkv(_ptr(Q), _ptr(K), _ptr(V), dt, self.Ts, self.H, self.d, self.P,
                                      _ptr(self.send), _ptr(self.scratch), st), "kvq_ulysses_pack_qkv")
        self._mark("pack")
        self.dist.all_to_all_single(self.recv, self.send, output_split_sizes=[self.recv_seg] * self.P,
                                    input_split_sizes=self.send_sizes, group=self.group)
        self._mark("a2a_in")
        _check(L.kvq_ulysses_unpack_qkv(_ptr(self.recv), dt, self.Ts, self.Hr, self.d, self.P, _ptr(self.Q),
                                        _ptr(self.K), _ptr(self.V), _ptr(self.amax), st), "kvq_ulysses_unpack_qkv")
        self._mark("unpack")
        self.cache.append(layer, chunk_index, self.K, self.V, amax_kv=self.amax)
        self._mark("quantize_append")
        return self._attend_and_return(layer, mask, out, Q)

    def _attend_and_return(self, layer, mask, out, Q):
        L, st = lib(), _stream()
        if self.nvfp4_q:
            self.cache.attention_qscaled(layer, self.Q16, self.q_scale, mask, out=self.O_local)
        else:
            self.cache.attention(layer, self.Q, mask, out=self.O_local)
        self._mark("attention")
        o_send = self.O_local.view(torch.uint8).reshape(-1)
        self.dist.all_to_all_single(self.o_recv, o_send, output_split_sizes=self.o_recv_sizes,
                                    input_split_sizes=[o_send.numel() // self.P] * self.P, group=self.group)
        self._mark("a2a_out")
        if out is None:
            out = torch.empty((self.Ts, self.H, self.d), dtype=torch.bfloat16, device=Q.device)
        _check(L.kvq_ulysses_unpack_o(_ptr(self.o_recv), KVQ_BF16, self.Ts, self.H, self.d, self.P, _ptr(out), st),
               "kvq_ulysses_unpack_o")
        self._mark("unpack_o")
        return out

    def breakdown(self, fn, reps=5):
        """Median per-phase device time (ms) of `fn()` (one step), phases as marked in step()."""
        rows = []
        for _ in range(reps):
            self.marks = []
            fn()
            torch.cuda.synchronize()
            rows.append([(n, self.marks[i - 1][1].elapsed_time(e)) for i, (n, e) in enumerate(self.marks) if i])
            self.marks = None
        names = [n for n, _ in rows[0]]
        return {n: float(np.median([r[i][1] for r in rows])) for i, n in enumerate(names)}


def softmax_scale_default(d):
    return 1.0 / math.sqrt(d)


EXCHANGE_INPUT, EXCHANGE_NVFP4, EXCHANGE_NVFP4_Q = 0, 1, 2


class NcclUlysses:
    """ulysses_chunk_attention with the library's own NCCL communicator (include/kvq.h, "One-call
    head-sharded chunk step"; App. C, App. D).  The unique id is
    made on rank 0 and broadcast over `group` (torch.distributed, any backend); after that every
    collective of the step is issued by libkvq itself on the current stream."""

    def __init__(self, cache: KVCache, H, rank, world, group=None, exchange=EXCHANGE_INPUT,
                 in_dtype=torch.bfloat16, out_dtype=torch.bfloat16):
        import torch.distributed as dist
        L = lib()
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            _check(L.kvq_get_unique_id(buf), "kvq_get_unique_id")
            uid = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).clone()
        if world > 1:
            dev_uid = uid.to(cache.device) if dist.get_backend(group) == "nccl" else uid
            dist.broadcast(dev_uid, 0, group=group)
            uid = dev_uid.cpu()
        raw = bytes(uid.numpy().tobytes())
        h = ctypes.c_void_p()
        _check(L.kvq_comm_create(ctypes.create_string_buffer(raw, 128), world, rank, ctypes.byref(h)),
               "kvq_comm_create")
        self._h = h
        self.cache, self.H, self.P, self.rank = cache, H, world, rank
        self.in_dtype, self.out_dtype = in_dtype, out_dtype
        nb = int(L.kvq_ulysses_workspace_bytes(cache.T_c, H, cache.d, world, rank, exchange, _out_code(in_dtype),
                                               _out_code(out_dtype)))
        if nb == 0:
            raise KVQError(-2, "kvq_ulysses_workspace_bytes")
        self.ws = torch.empty(nb, dtype=torch.uint8, device=cache.device)
        _check(L.kvq_comm_configure(self._h, H, exchange, _ptr(self.ws), nb), "kvq_comm_configure")

    def step(self, layer, chunk_index, Q, K, V, mask: Mask, out=None, softmax_scale=0.0):
        """Q, K, V: this rank's sequence shard [T_c/P, H, d] -> O shard [T_c/P, H, d] (out_dtype)."""
        Ts = self.cache.T_c // self.P
        for t in (Q, K, V):
            if tuple(t.shape) != (Ts, self.H, self.cache.d) or t.dtype != self.in_dtype:
                raise ValueError(f"expected [{Ts}, {self.H}, {self.cache.d}] {self.in_dtype}")
        if out is None:
            out = torch.empty((Ts, self.H, self.cache.d), dtype=self.out_dtype, device=Q.device)
        m = mask._c()
        _check(lib().ulysses_chunk_attention(self._h, self.cache._h, layer, chunk_index, _ptr(Q), _ptr(K), _ptr(V),
                                             _dt(Q), ctypes.byref(m), softmax_scale, _ptr(out),
                                             _out_code(self.out_dtype), _stream()), "ulysses_chunk_attention")
        return out

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _check(_lib.kvq_comm_destroy(self._h), "kvq_comm_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
