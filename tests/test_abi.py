"""C-ABI library checks that need no GPU (-m "not gpu"): libkvq.so loads, exports every symbol
include/*.h declares, and the pure host functions behave (head partition, exchange sizes,
config validation)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_18739_b200", "libkvq.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2605_18739_b200 import build
        build.build()
    from paper_2605_18739_b200 import kvq
    return kvq.lib()


def _declared():
    names = set()
    for h in ("kvq.h", "kvq_debug.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s+\*?([a-z_][a-z0-9_]*)\s*\(", src, re.M):
            names.add(m.group(1))
    return names


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("kv_quantize_append", "chunk_attention", "kv_dequantize", "kv_export_chunk", "kvq_cache_create",
              "kvq_ulysses_pack_qkv", "kvq_head_partition", "ulysses_chunk_attention", "kvq_comm_create",
              "kvq_get_unique_id"):
        assert n in names
    assert len(names) >= 22


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing


def test_head_partition(lib):
    from paper_2605_18739_b200 import kvq
    # first H % P ranks get one more head (12 heads on 8 ranks: 2,2,2,2,1,1,1,1)
    assert [kvq.head_partition(12, 8, r) for r in range(8)] == [(0, 2), (2, 4), (4, 6), (6, 8), (8, 9), (9, 10),
                                                                (10, 11), (11, 12)]
    for H, P in [(12, 1), (12, 2), (12, 4), (24, 8), (7, 3)]:
        parts = [kvq.head_partition(H, P, r) for r in range(P)]
        assert parts[0][0] == 0 and parts[-1][1] == H
        assert all(parts[i][1] == parts[i + 1][0] for i in range(P - 1))
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1


def test_exchange_sizes(lib):
    from paper_2605_18739_b200 import kvq
    Ts, H, d = 4680 // 8, 12, 128
    sizes = [kvq.ulysses_qkv_bytes(Ts, H, d, 8, p) for p in range(8)]
    assert sizes[0] == 3 * Ts * 2 * d * 2 + 16 and sizes[7] == 3 * Ts * 1 * d * 2 + 16
    # total payload of one rank = its whole Q|K|V shard + one 16-byte trailer per destination
    assert sum(sizes) == 3 * Ts * H * d * 2 + 16 * 8


def test_cache_bytes_and_validation(lib):
    from paper_2605_18739_b200.kvq import Config
    c = Config(30, 12, 128, 1560, 3, 3, 21, 8, 0, 0)
    n = lib.kvq_cache_bytes(ctypes.byref(c))
    T_pad = 4736
    payload = 30 * 12 * 8 * T_pad * (64 + 8) * 2
    attn_ws = 2 * 148 * (256 * 128 + 512) * 4      # stream-K partial-piece workspace
    assert payload + attn_ws <= n <= payload + attn_ws + 64 * 1024
    # NVFP4 resident bytes vs bf16 for 8 slots x 30 layers (1.94 GB vs 6.90 GB)
    assert abs(30 * 12 * 8 * 4680 * 72 * 2 / 1e9 - 1.94) < 0.01
    for bad in (Config(30, 12, 96, 1560, 3, 3, 21, 8, 0, 0), Config(30, 12, 128, 1560, 3, 3, 21, 8, 2, 0),
                Config(30, 12, 128, 1560, 3, 3, 21, 8, 0, 2), Config(30, 12, 128, 1560, 3, 3, 21, 0, 0, 0),
                Config(0, 12, 128, 1560, 3, 3, 21, 8, 0, 0)):
        assert lib.kvq_cache_bytes(ctypes.byref(bad)) == 0
    # Four-Over-Six needs no extra bytes; K-smoothing adds one fp32 mean per cached K row
    assert lib.kvq_cache_bytes(ctypes.byref(Config(30, 12, 128, 1560, 3, 3, 21, 8, 1, 0))) == n
    ns = lib.kvq_cache_bytes(ctypes.byref(Config(30, 12, 128, 1560, 3, 3, 21, 8, 1, 1)))
    assert n + 30 * 12 * 8 * T_pad * 4 <= ns <= n + 30 * 12 * 8 * T_pad * 4 + 4096


def test_strerror(lib):
    assert lib.kvq_strerror(0) == b"ok"
    assert lib.kvq_strerror(-4).startswith(b"chunk")


def test_native_ulysses_workspace_and_argument_checks(lib):
    # host-only: workspace sizing and the synchronous argument errors (no NCCL call is reached)
    T_c, H, d = 4680, 12, 128
    b0 = lib.kvq_ulysses_workspace_bytes(T_c, H, d, 8, 0, 0, 0, 0)
    b1 = lib.kvq_ulysses_workspace_bytes(T_c, H, d, 8, 0, 1, 0, 0)
    b7 = lib.kvq_ulysses_workspace_bytes(T_c, H, d, 8, 7, 0, 0, 0)
    Ts, act0 = T_c // 8, T_c * 2 * d * 2
    # exchange 0 holds at least: send (the whole shard Q|K|V) + recv (3 x 2 heads x T_c) + local Q/K/V + O
    assert b0 >= 3 * Ts * H * d * 2 + 3 * act0 + 3 * act0 + act0
    assert b1 < b0 and b7 < b0  # NVFP4 K/V payload, and rank 7 owns one head instead of two
    assert all(x % 256 == 0 for x in (b0, b1, b7))
    assert lib.kvq_ulysses_workspace_bytes(T_c, H, d, 7, 0, 0, 0, 0) == 0  # T_c % P != 0
    assert lib.kvq_ulysses_workspace_bytes(T_c, H, d, 8, 8, 0, 0, 0) == 0  # rank out of range
    assert lib.kvq_ulysses_workspace_bytes(T_c, H, d, 8, 0, 3, 0, 0) == 0  # unknown exchange
    out = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert lib.kvq_comm_create(uid, 0, 0, ctypes.byref(out)) == -1
    assert lib.kvq_comm_create(uid, 2, 2, ctypes.byref(out)) == -1
    assert lib.kvq_comm_create(None, 1, 0, ctypes.byref(out)) == -1
    assert lib.kvq_comm_destroy(None) == -1
    assert lib.kvq_get_unique_id(None) == -1
    assert lib.ulysses_chunk_attention(None, None, 0, 0, None, None, None, 0, None, 0.0, None, 0, None) == -1
