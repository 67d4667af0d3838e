"""N>1 host logic on CPU (-m "not gpu"): two processes over torch.distributed gloo exchange exactly the
byte segments the Ulysses path sends (sizes from the C ABI's kvq_ulysses_qkv_bytes, heads from
kvq_head_partition), with the packing laid out on the CPU as include/kvq.h documents it.  Checks
that every rank receives the Q/K/V of its heads for all tokens (L/P x H x d ->
L x H/P x d), the piggybacked amax reduces to the global amax (reading Z18), and the O return
restores the sequence shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

T, H, D = 24, 5, 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _full():
    from paper_2605_18739_b200 import synth
    return [synth.make_tensor((T, H, D), "fp32", seed=s).raw for s in (1, 2, 3)]


def _pack_cpu(Q, K, V, P, rank, Ts):
    """The send layout of kvq_ulysses_pack_qkv, per destination p: [3][Ts][H_p][d] + trailer."""
    from paper_2605_18739_b200 import kvq
    segs = []
    amk = np.abs(K).max().astype(np.float32).view(np.uint32)
    amv = np.abs(V).max().astype(np.float32).view(np.uint32)
    for p in range(P):
        h0, h1 = kvq.head_partition(H, P, p)
        body = np.stack([Q[:, h0:h1], K[:, h0:h1], V[:, h0:h1]]).astype(np.float32).tobytes()
        trailer = np.array([amk, amv, 0, 0], dtype=np.uint32).tobytes()
        segs.append(np.frombuffer(body + trailer, dtype=np.uint8))
        assert segs[-1].size == kvq.ulysses_qkv_bytes(Ts, H, D, P, p, torch.float32)
    return np.concatenate(segs)


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2605_18739_b200 import kvq
        Qf, Kf, Vf = _full()
        Ts = T // world
        sl = slice(rank * Ts, (rank + 1) * Ts)
        send = torch.from_numpy(_pack_cpu(Qf[sl], Kf[sl], Vf[sl], world, rank, Ts).copy())
        sizes = [kvq.ulysses_qkv_bytes(Ts, H, D, world, p, torch.float32) for p in range(world)]
        h0, h1 = kvq.head_partition(H, world, rank)
        seg = kvq.ulysses_qkv_bytes(Ts, H, D, world, rank, torch.float32)
        recv = torch.empty(seg * world, dtype=torch.uint8)
        dist.all_to_all_single(recv, send, output_split_sizes=[seg] * world, input_split_sizes=sizes)
        r = recv.numpy()
        Hr = h1 - h0
        body = 3 * Ts * Hr * D * 4
        got = [np.frombuffer(r[s * seg:s * seg + body].tobytes(), dtype=np.float32).reshape(3, Ts, Hr, D)
               for s in range(world)]
        for i, full in enumerate((Qf, Kf, Vf)):
            assert np.array_equal(np.concatenate([g[i] for g in got]), full[:, h0:h1])
        amax = [max(np.frombuffer(r[s * seg + body:s * seg + body + 8].tobytes(), dtype=np.float32)[j]
                    for s in range(world)) for j in range(2)]
        assert amax[0] == np.abs(Kf).max() and amax[1] == np.abs(Vf).max()
        # O return: O_local [T, Hr, D] sent as equal token blocks; reassemble this rank's shard
        O_full = Qf * 2.0 + 1.0
        O_local = torch.from_numpy(np.ascontiguousarray(O_full[:, h0:h1]))
        o_sizes = [Ts * (kvq.head_partition(H, world, p)[1] - kvq.head_partition(H, world, p)[0]) * D for p in range(world)]
        o_recv = torch.empty(sum(o_sizes), dtype=torch.float32)
        dist.all_to_all_single(o_recv, O_local.reshape(-1), output_split_sizes=o_sizes,
                               input_split_sizes=[Ts * Hr * D] * world)
        parts, off = [], 0
        for p in range(world):
            hp0, hp1 = kvq.head_partition(H, world, p)
            parts.append(o_recv[off:off + o_sizes[p]].numpy().reshape(Ts, hp1 - hp0, D))
            off += o_sizes[p]
        assert np.array_equal(np.concatenate(parts, axis=1), O_full[sl])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 3])
def test_ulysses_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(msg == "ok" for _, msg in res), res


def _pad16(n):
    return (n + 15) // 16 * 16


def _worker_nvfp4(rank, world, port, q):
    """§8(f) f3: the NVFP4 exchange's host logic -- shard amax all-reduced (MAX) over the group, the
    per-destination segment layout of kvq_ulysses_nvfp4_bytes / include/kvq.h built on the CPU from the
    oracle's quantization under the global scale, and the receiver's view of every source segment."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import nvfp4
        from paper_2605_18739_b200 import kvq
        Qf, Kf, Vf = _full()
        Ts = T // world
        sl = slice(rank * Ts, (rank + 1) * Ts)
        # shard amax -> all-reduce(MAX): the global amax every rank quantizes with (reading Z18)
        amax = torch.tensor([np.abs(Kf[sl]).max(), np.abs(Vf[sl]).max()], dtype=torch.float32)
        dist.all_reduce(amax, op=dist.ReduceOp.MAX)
        assert amax[0].item() == np.abs(Kf).max() and amax[1].item() == np.abs(Vf).max()
        qk = nvfp4.quantize_kv_chunk(Kf.astype(np.float64))   # codes are row-local: slicing = shard packing
        qv = nvfp4.quantize_kv_chunk(Vf.astype(np.float64))
        cod = [q_["codes"].reshape(T, H, D // 2) for q_ in (qk, qv)]
        sca = [q_["scales"].reshape(T, H, D // 16) for q_ in (qk, qv)]
        segs, sizes = [], []
        for p in range(world):
            h0, h1 = kvq.head_partition(H, world, p)
            rows = Ts * (h1 - h0)
            parts = [np.ascontiguousarray(Qf[sl, h0:h1]).astype(np.float32).tobytes()]
            for i in range(2):
                parts.append(np.ascontiguousarray(cod[i][sl, h0:h1]).tobytes())
                parts.append(np.ascontiguousarray(sca[i][sl, h0:h1]).tobytes())
            seg = b"".join(x + bytes(_pad16(len(x)) - len(x)) for x in parts)
            assert len(seg) == kvq.ulysses_nvfp4_bytes(Ts, H, D, world, p, torch.float32), (len(seg), rows)
            segs.append(np.frombuffer(seg, dtype=np.uint8))
            sizes.append(len(seg))
        send = torch.from_numpy(np.concatenate(segs).copy())
        h0, h1 = kvq.head_partition(H, world, rank)
        Hr = h1 - h0
        seg = kvq.ulysses_nvfp4_bytes(Ts, H, D, world, rank, torch.float32)
        recv = torch.empty(seg * world, dtype=torch.uint8)
        dist.all_to_all_single(recv, send, output_split_sizes=[seg] * world, input_split_sizes=sizes)
        r = recv.numpy()
        rows = Ts * Hr
        off_q, n_q = 0, rows * D * 4
        off_kc = _pad16(n_q)
        off_ks = off_kc + _pad16(rows * D // 2)
        for s in range(world):
            base = s * seg
            qs = np.frombuffer(r[base + off_q:base + off_q + n_q].tobytes(), dtype=np.float32).reshape(Ts, Hr, D)
            assert np.array_equal(qs, Qf[s * Ts:(s + 1) * Ts, h0:h1])
            kc = r[base + off_kc:base + off_kc + rows * D // 2].reshape(Ts, Hr, D // 2)
            assert np.array_equal(kc, cod[0][s * Ts:(s + 1) * Ts, h0:h1])
            ks = r[base + off_ks:base + off_ks + rows * D // 16].reshape(Ts, Hr, D // 16)
            assert np.array_equal(ks, sca[0][s * Ts:(s + 1) * Ts, h0:h1])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 3])
def test_ulysses_nvfp4_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_nvfp4, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(msg == "ok" for _, msg in res), res


def test_ulysses_nvfp4_payload_is_32_over_9_smaller_for_kv():
    # PAPER.md:642-650 ("reduced by roughly 3.6x"): per (t, h) row, K and V travel as d/2 code bytes +
    # d/16 scale bytes instead of 2d bf16 bytes -- 32/9 -- with each part padded to 16 bytes
    from paper_2605_18739_b200 import kvq
    Ts, Hh, d, P = 585, 12, 128, 8
    for dst in range(P):
        h0, h1 = kvq.head_partition(Hh, P, dst)
        rows = Ts * (h1 - h0)
        nv = kvq.ulysses_nvfp4_bytes(Ts, Hh, d, P, dst)
        assert nv == _pad16(rows * d * 2) + 2 * (_pad16(rows * d // 2) + _pad16(rows * d // 16))
        assert kvq.ulysses_qkv_bytes(Ts, Hh, d, P, dst) == 3 * rows * d * 2 + 16
        assert (2 * rows * d * 2) / (2 * (rows * d // 2 + rows * d // 16)) == 32 / 9
        assert kvq.ulysses_nvfp4_bytes(Ts, Hh, d, P, dst, k_smoothing=True) == nv + _pad16(rows * 4)
