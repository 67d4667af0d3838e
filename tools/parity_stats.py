"""Full-size parity statistics of the Wan layer (all 4680 rows x 12 heads) against the float64 oracle:
fp32-out error, and the bf16-out criteria of reading Z17 (per-element bf16 ulp, row-scale bf16 ulp,
rel-L2 vs RN_bf16(oracle)).  Diagnostic only (prints one JSON line); the asserts live in tests/."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gpu_util import bf16_round, bf16_ulp  # noqa: E402
from oracle.attention import attention  # noqa: E402
from oracle.cache import OracleKVCache  # noqa: E402
from paper_2605_18739_b200 import kvq, synth  # noqa: E402


def main():
    T, H, d = 4680, 12, 128
    out = {"nproc": os.cpu_count(), "torch_threads": torch.get_num_threads()}
    c = kvq.KVCache(1, H, d, 1560, 3, sink_frames=3, window_frames=21, max_chunk_slots=8, device="cuda")
    o = OracleKVCache(1, H, d, 1560, 3)
    t0 = time.time()
    for ch in range(7):
        q, k, v = synth.make_qkv(T, H, d, "bf16", 0, ch)
        c.append(0, ch, k.torch("cuda"), v.torch("cuda"))
        o.append(0, ch, k.f64, v.f64)
    out["oracle_quant_7chunks_s"] = time.time() - t0
    m = kvq.Mask(6, 3, 21)
    O32 = c.attention(0, q.torch("cuda"), m, torch.float32).cpu().numpy().astype(np.float64)
    Ob = c.attention(0, q.torch("cuda"), m, torch.bfloat16).float().cpu().numpy().astype(np.float64)
    t0 = time.time()
    K, V = o.keys(0, 6, 3, 21)
    ref = attention(q.f64, K, V)
    out["oracle_attention_full_s"] = time.time() - t0
    out["fp32_maxabs"] = float(np.abs(O32 - ref).max())
    out["fp32_rel"] = float(np.linalg.norm(O32 - ref) / np.linalg.norm(ref))
    rb = bf16_round(ref)
    diff = np.abs(Ob - rb)
    lit = diff > bf16_ulp(rb) * (1 + 1e-9)
    rowmax = np.abs(ref).max(axis=2, keepdims=True)
    rowv = diff > bf16_ulp(rowmax) * (1 + 1e-9)
    out["bf16_literal_ulp_violations"] = int(lit.sum())
    out["bf16_literal_viol_max_absref"] = float(np.abs(ref[lit]).max()) if lit.any() else 0.0
    out["bf16_rowscale_ulp_violations"] = int(rowv.sum())
    out["bf16_rel_vs_rnbf16"] = float(np.linalg.norm(Ob - rb) / np.linalg.norm(rb))
    out["bf16_eq_rn_fp32"] = bool(np.array_equal(Ob, bf16_round(O32)))
    out["bf16_max_diff_in_ulps"] = float((diff / bf16_ulp(rb)).max())
    out["elements"] = int(ref.size)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
