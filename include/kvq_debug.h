/*
 * kvq_debug.h -- diagnostic entry points of libkvq.so (not the product path).
 *
 * kvq_debug_probe runs the hardware NVFP4 conversions used by the kernels element by element so
 * tests can compare them with the float64 oracle's codecs (PAPER.md:719 E2M1 value set,
 * PAPER.md:102 E4M3 max 448; readings Z3, Z6-Z8 of DESIGN.md):
 *   which = 0: E2M1 encode, dev_in fp32[2n] -> dev_out u8[2n] (one code per element;
 *              cvt.rn.satfinite.e2m1x2.f32, element 2k taken from the low nibble)
 *   which = 1: E4M3 encode of non-negative values, fp32[n] -> u8[n] (cvt.rn.satfinite.e4m3x2.f32)
 *   which = 2: E2M1 decode, u8[n] (two codes per byte) -> fp32[2n], low nibble first
 *   which = 3: E4M3 decode, u8[n] -> fp32[n]
 * Returns KVQ_EINVAL on a bad `which` or null pointer; stream-ordered on `stream`.
 */
#ifndef KVQ_DEBUG_H_
#define KVQ_DEBUG_H_
#include "kvq.h"
#ifdef __cplusplus
extern "C" {
#endif
kvq_status kvq_debug_probe(int32_t which, const void* dev_in, void* dev_out, int64_t n, void* stream);

/* Timeline instrumentation of chunk_attention: when dev_buf (>= 64*16 u64, caller-owned device
 * memory) is set, CTA 0 of every later chunk_attention records SM clock64() at its warp-role
 * hand-offs for its first 64 key tiles (row = tile, column = event: 0/1/2 softmax WG0 wait
 * start / S ready / P done, 3/4/5 the same for WG1, 6/7 dequant K / V row written, 8/9/10/11
 * MMA issue of PV0 / QK0(next) / PV1 / QK1(next) done).  NULL disables (the default). */
kvq_status kvq_debug_set_trace(void* dev_buf);

/* on != 0: kv_quantize_append always uses the two-launch path (amax pass + quantize pass) instead
 * of the single-pass cooperative kernel, so tests can check both produce identical bytes. */
kvq_status kvq_debug_force_two_pass(kvq_cache* cache, int32_t on);
#ifdef __cplusplus
}
#endif
#endif
