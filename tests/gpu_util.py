"""Helpers shared by the -m gpu parity tests (comparison only; no method arithmetic)."""
import numpy as np
import torch

from oracle import nvfp4


def bf16_round(x):
    """RN_bf16 of float64 values via float32 (the rounding a bf16 output applies)."""
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def bf16_ulp(x):
    """Spacing of bf16 at |x| (for the 1-ulp bf16 output check)."""
    a = np.abs(np.asarray(x, dtype=np.float64))
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -126)))
    return 2.0 ** (e - 7)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def check_fp32_out(O_gpu, O_ref, max_abs=2e-3, rel=1e-3):
    """north_star tolerance: max-abs 2e-3 and rel-L2 1e-3 against the float64 oracle (fp32-out mode)."""
    O_gpu = np.asarray(O_gpu, dtype=np.float64)
    err = np.abs(O_gpu - O_ref).max()
    r = rel_l2(O_gpu, O_ref)
    assert np.all(np.isfinite(O_gpu))
    assert err <= max_abs, f"max-abs {err:.3e} > {max_abs}"
    assert r <= rel, f"rel-L2 {r:.3e} > {rel}"
    return err, r


def check_bf16_out(O_gpu, O_ref, O_gpu_fp32=None, rel=1e-3):
    """bf16 output, reading Z17:
    (a) when the same call's fp32-mode output is given: O_bf16 == RN_bf16(O_fp32), bit for bit (same
        arithmetic, one final rounding);
    (b) elementwise |O_bf16 - RN_bf16(O_ref)| <= 1 bf16 ulp, the ulp taken at the output ROW's scale,
        max_u |O_ref[t, h, u]| (Z17: per-element ulps near a cancellation zero are below any
        fp32-accumulating kernel's rounding -- measured: an all-fp32 CPU emulation misses the
        per-element reading on 24 of 599,040 elements, the fp16-P design of SURVEY X3 on 1.7%, and
        both meet the row-scale reading on every element);
    (c) rel-L2 of O_bf16 against RN_bf16(O_ref) <= 1e-3 (as written)."""
    O_gpu = np.asarray(O_gpu, dtype=np.float64)
    O_ref = np.asarray(O_ref, dtype=np.float64)
    assert np.all(np.isfinite(O_gpu))
    if O_gpu_fp32 is not None:
        assert np.array_equal(O_gpu, bf16_round(O_gpu_fp32)), "bf16 out != RN_bf16(fp32 out)"
    ref_b = bf16_round(O_ref)
    diff = np.abs(O_gpu - ref_b)
    row_ulp = bf16_ulp(np.abs(O_ref).max(axis=-1, keepdims=True))
    worst = float((diff / row_ulp).max())
    assert worst <= 1.0, f"bf16 error {worst:.3f} row-scale ulps (> 1)"
    r = float(np.linalg.norm(O_gpu - ref_b) / max(np.linalg.norm(ref_b), 1e-300))
    assert r <= rel, f"bf16 rel-L2 vs RN_bf16(oracle) {r:.3e} > {rel}"
    return worst, r


def export_to_numpy(ex):
    return {k: v.cpu().numpy() for k, v in ex.items()}


def assert_chunk_bytes_equal(ex, qk, qv):
    """Exported canonical bytes (rows (t,h) t-major) equal the oracle's, bit for bit."""
    e = export_to_numpy(ex)
    for name, q, tag in (("k", qk, "K"), ("v", qv, "V")):
        assert np.float32(e["g_" + name][0]).view(np.uint32) == np.float32(q["g"]).view(np.uint32), f"g_{tag}"
        sc = e["scales_" + name]
        bad_s = np.count_nonzero(sc != q["scales"])
        cd = e["codes_" + name]
        bad_c = np.count_nonzero(nvfp4.unpack_codes(cd) != nvfp4.unpack_codes(q["codes"]))
        assert bad_s == 0 and bad_c == 0, f"{tag}: {bad_s} scales / {bad_c} codes differ"
