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


def check_bf16_out(O_gpu, O_ref, O_gpu_fp32=None, max_abs=2e-3):
    """bf16 output (reading Z17).  Rounding the exact answer to bf16 alone exceeds the fp32-mode
    tolerance, so the bf16 product is checked as: (a) bit-identical to RN_bf16 of the kernel's
    fp32-mode output (same arithmetic, different final rounding), when given; (b) elementwise
    |O_bf16 - O_ref| <= 1 bf16 ulp(O_ref) + max_abs (one output rounding on top of the fp32 bar);
    (c) ||O_bf16 - O_ref|| <= ||RN_bf16(O_ref) - O_ref|| + 1e-3 ||O_ref||: no worse than rounding
    the exact answer to bf16, plus the fp32-mode rel-L2 budget."""
    O_gpu = np.asarray(O_gpu, dtype=np.float64)
    if O_gpu_fp32 is not None:
        assert np.array_equal(O_gpu, bf16_round(O_gpu_fp32)), "bf16 out != RN_bf16(fp32 out)"
    excess = np.abs(O_gpu - O_ref) - bf16_ulp(O_ref)
    assert excess.max() <= max_abs, f"bf16 error exceeds 1 ulp + {max_abs} by {excess.max():.3e}"
    ref_b = bf16_round(O_ref)
    nref = np.linalg.norm(O_ref)
    e_gpu = np.linalg.norm(O_gpu - O_ref)
    e_round = np.linalg.norm(ref_b - O_ref)
    assert e_gpu <= e_round + 1e-3 * nref, f"bf16 rel-L2 {e_gpu / nref:.3e} vs rounding floor {e_round / nref:.3e}"
    return float(excess.max()), (e_gpu - e_round) / nref


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
