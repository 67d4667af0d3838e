// attention.cu -- chunk attention over the NVFP4 KV cache with dequantization fused into the
// kernel, on tcgen05 tensor cores (sm_100a).
//
// Computes chunk_attention (include/kvq.h): for the current chunk's queries and head h,
//   O = softmax(Q K^T * scale) V over the effective key set K_eff(t)
// (§4.2; the cache of PAPER.md:134-146 §3.2), where K^, V^ are the
// NVFP4 values of Eq. 2.  Dequantization is fused: the paper's separate
// "parallel dequantization kernel" is prior art that this kernel replaces.
//
// Numerics: K^' = dec(code) * dec(s) and V^' likewise are EXACT in fp16, so the
// tensor cores see the exact quantized lattice; the FP32 tensor scales g_K, g_V are applied in
// fp32 outside the MMA (g_K in the exponent scale, g_V folded into the O rescale factor).
// bf16 Q is exact in fp16; fp32 Q is split into fp16 hi + lo (QSPLIT).  P is fp16, accumulation is
// fp32 in TMEM, the running max is lazy (moves only when a tile exceeds it by 2^kLazyLog2), and l is
// summed in fp32 from the fp16-rounded P.
//
// Structure: one CTA = one head x two 128-query tiles (256 rows share every dequantized KV
// tile), warp-specialized, 13 warps:
//   warps 0-3   softmax WG0  (query tile 0; thread i owns row i = TMEM lane i)
//   warps 4-7   softmax WG1  (query tile 1)
//   warps 8-11  dequant WG   (packed codes + E4M3 scales from L2 -> fp16 K^', V^' rows in
//                             128B-swizzled smem, double buffered)
//   warp 12     MMA issuer   (one thread issues tcgen05.mma; TMEM allocator)
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); P_i (fp16) overwrites
// the first 64 columns of S_i.  Ping-pong: while WG0 exponentiates S0(j) the tensor core runs
// QK1(j); while WG1 works on S1(j) it runs PV0(j) and QK0(j+1).  All hand-offs are mbarriers
// (tcgen05.commit for MMA completion); MMAs execute in issue order, so the commit that signals
// S_i(j+1) also guarantees PV_i(j) finished (O_i stable for the rescale, P_i(j) consumed).
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "quant_core.cuh"

namespace kvq {
namespace {

constexpr int kThreads = 16 * 32;  // 4 warpgroups: softmax0, softmax1, dequant, MMA (+3 idle warps)
// Register budget per SM sub-partition (16K regs = 4 warps x 128 at launch), rebalanced with
// setmaxnreg: softmax 168 + 168, dequant 88, MMA warpgroup 88 (sum 512 per thread slot).  Swept
// (tools/ab_attn.sh, same box, after the debug trace was compiled out -- KVQ_TRACE_BUILD): softmax
// 160 / 168 / 176 -> 919 (spills) / 832 / 861 us after an L2 flush; at 168 the MMA/dequant split
// 80/96, 88/88, 96/80 is 830 / 832 / 830 us (noise).  Round 1 (trace compiled in) had found 176.
#ifndef KVQ_REG_SOFTMAX
#define KVQ_REG_SOFTMAX 168
#endif
#ifndef KVQ_REG_MMA
#define KVQ_REG_MMA (256 - KVQ_REG_SOFTMAX)
#endif
constexpr int kRegSoftmax = KVQ_REG_SOFTMAX, kRegMma = KVQ_REG_MMA, kRegDequant = 512 - 2 * KVQ_REG_SOFTMAX - KVQ_REG_MMA;
// the fused-append kernel (APPEND) carries a little more state through the softmax loop
#ifndef KVQ_REG_SOFTMAX_AP
#define KVQ_REG_SOFTMAX_AP 184
#endif
#ifndef KVQ_REG_MMA_AP
#define KVQ_REG_MMA_AP 72
#endif
constexpr int kRegSoftmaxAp = KVQ_REG_SOFTMAX_AP, kRegMmaAp = KVQ_REG_MMA_AP,
              kRegDequantAp = 512 - 2 * KVQ_REG_SOFTMAX_AP - KVQ_REG_MMA_AP;
// Of every 8 exponential pairs of a score row, this many are evaluated by exp2_poly_pair on the
// FMA pipe instead of MUFU.EX2 (MUFU alone would equal the tensor-core time at d = 128).  Round 2
// same-box sweeps: 1 -> 886-892 us, 2 -> 910-916 us, 3 -> 937 us (round 1 had found 2 best).
#ifndef KVQ_POLY_PAIRS
#define KVQ_POLY_PAIRS 1
#endif
constexpr int kPolyPairs = KVQ_POLY_PAIRS;
// Lazy-rescale threshold in log2 units (0 = exact running max, O rescaled whenever it grows).
#ifndef KVQ_LAZY_LOG2
#define KVQ_LAZY_LOG2 4.0f
#endif
constexpr float kLazyLog2 = KVQ_LAZY_LOG2;
// Rotating S/P regions (build knob, default on).  The 256 S/P columns of TMEM are four 64-column
// regions R0..R3; the k-th QK of a piece (k = 2 j + tile) writes keys 0-63 into region a(k) and keys
// 64-127 into region b(k) (two N = 64 MMAs), and the softmax stores P (fp16, 64 columns) into b(k).
// a is free again as soon as the softmax has loaded S into registers (`sfree`), b once the PV that
// reads P has been issued (the tensor core runs in issue order).  k = 0, 1: (R0, R1), (R2, R3); then
// a = R0 and b cycles R2, R1, R3 -- each b is exactly the P region of the PV issued just before, so
// QK_i(j+1) waits only for the OTHER tile's softmax to have loaded its S, not for PV_i(j): the next
// scores are computed while this tile's softmax still runs, and each softmax warpgroup goes from one
// tile to the next without waiting for its own PV + QK round trip.  Correct (parity suite) but
// measured SLOWER (942 vs 914 us): the N = 64 halves re-read the whole Q tile per MMA, so a QK moves
// 1.5x the shared-memory bytes of an N = 128 one (6 KB per 32-cycle MMA > 128 B/clk), and no
// rotation keeps both halves of every S in adjacent regions.  Off by default.
#ifndef KVQ_SP_ROTATE
#define KVQ_SP_ROTATE 0
#endif
constexpr bool kRotate = KVQ_SP_ROTATE != 0;
// Split rows (build knob): the two softmax warpgroups work TOGETHER on each query tile -- warpgroup h
// takes key columns [64 h, 64 h + 64) of every row of S -- and go through the two tiles in turn
// (tile 0, tile 1, tile 0, ...), instead of one warpgroup per tile.  Each tile's softmax then takes
// half the time, so the per-tile chain softmax -> PV -> QK -> softmax (P reuses S's TMEM columns)
// shrinks, while the tensor core still alternates between the tiles.  The halves exchange their
// partial row maxima through shared memory (one 256-thread named barrier per tile) so both take the
// same lazy max; the row sums are combined once per piece.  Correct (parity suite) and a tile's
// softmax does take less time (1,660-1,790 vs 2,180 cycles), but both warpgroups now run their
// exponential loops at the same time on every SM sub-partition, so MUFU and the FMA pipe are shared
// and the two tiles' softmax together still take ~3,500 cycles: 898-903 us against 886-892 us for
// the per-tile design with one polynomial pair in eight.  Off by default.
#ifndef KVQ_SPLIT_ROWS
#define KVQ_SPLIT_ROWS 0
#endif
constexpr bool kSplitRows = KVQ_SPLIT_ROWS != 0;
static_assert(!(kSplitRows && kRotate), "split rows and rotating S/P regions are exclusive");
KVQ_DEV void sp_regions(int k, uint32_t& a, uint32_t& b) {
  if (k < 2) {
    a = 2u * k;
    b = 2u * k + 1u;
  } else {
    const int m = (k - 2) % 3;
    a = 0u;
    b = m == 0 ? 2u : (m == 1 ? 1u : 3u);
  }
}
// Store P of keys 0-63 to TMEM from inside the exponential loop (build knob), overlapping the
// tcgen05.st with the second half of the loop (the MMA still waits for the whole tile's P).
#ifndef KVQ_EARLY_STTM
#define KVQ_EARLY_STTM 0
#endif
constexpr bool kEarlySttm = KVQ_EARLY_STTM != 0;
// Row max as a 3-input max tree (build knob) instead of four dependent chains.
#ifndef KVQ_MAX_TREE
#define KVQ_MAX_TREE 0
#endif
// Largest |row max score| (log2 units, after the exponent scale) the product supports: 2^12
// (reading Z25; the Wan workloads peak at ~30).
constexpr float kScoreRangeLog2 = 4096.0f;

template <int N>
KVQ_DEV void reg_alloc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
KVQ_DEV void reg_dealloc() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

// QSPLIT (fp32 Q): Q = Q_hi + Q_lo, both fp16, and S = Q_hi K^T + Q_lo K^T accumulate in TMEM, so
// fp32 queries lose ~2^-22 instead of fp16's 2^-11 (the single rounding costs up to 5e-3 max-abs on
// peaked rows with large key offsets).  The two Q_lo tiles take the second K/V buffers at d = 128
// (single-buffered K/V; the fp32-Q mode is the parity configuration, not the bench one) and two extra
// tiles at d = 64.
template <int D, bool QSPLIT = false>
struct WsSmem {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kNBuf = (QSPLIT && D == 128) ? 1 : 2;  // K^/V^ buffers
  static constexpr int kQ0 = 0;
  static constexpr int kQ1 = kTile;
  static constexpr int kK0 = 2 * kTile;
  static constexpr int kK1 = 3 * kTile;
  static constexpr int kV0 = 4 * kTile;
  static constexpr int kV1 = 5 * kTile;
  static constexpr int kQL0 = D == 128 ? 3 * kTile : 6 * kTile;  // QSPLIT only
  static constexpr int kQL1 = D == 128 ? 5 * kTile : 7 * kTile;
  static constexpr int kBar = (QSPLIT && D != 128) ? 8 * kTile : 6 * kTile;
  // barriers: kfull[2] vfull[2] kempty[2] vempty[2] sfull[2] pfull[2] ofull[2] + tmem slot
  static constexpr int kMean = kBar + 20 * 8 + 16;  // K-smoothing: [WG][2 buffers][128] fp32 means
  static constexpr int kAp = kMean + 2 * 2 * 128 * 4;  // fused append: launch epoch, shard amax partials
  // split rows: partial row maxima [2 steps][2 halves][128] fp32, query-row info [2 tiles][128] x
  // (sum(q) * scale, exponent scale, non-finite flag), row sums [2 tiles][2 halves][128]
  static constexpr int kXch = kAp + 64;
  static constexpr int kBytes = kXch + 2 * 2 * 128 * 4 + 2 * 128 * 12 + 2 * 2 * 128 * 4 + 1024;
  // K^/V^ buffer of global tile g, and the mbarrier parities of its full / empty waits
  static KVQ_DEV int buf(int g) { return kNBuf == 2 ? (g & 1) : 0; }
  static KVQ_DEV uint32_t full_par(int g) { return kNBuf == 2 ? ((g >> 1) & 1) : (g & 1); }
  static KVQ_DEV uint32_t empty_par(int g) { return kNBuf == 2 ? (((g >> 1) - 1) & 1) : ((g - 1) & 1); }
};

// address of 16-byte chunk c (8 consecutive elements along d) of row r in a 128-row tile
KVQ_DEV uint32_t chunk_addr(uint32_t base, int r, int c) {
  return base + (uint32_t)(c >> 3) * 16384u + sw128_off(r, c & 7);
}

KVQ_DEV uint32_t pack_half2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
KVQ_DEV uint32_t pack_bf162(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Packed cache row (D values): D/2 code bytes + D/16 scale bytes, loaded to registers.
template <int D>
struct PackedRow {
  uint4 c[D / 32];
  uint32_t s[D / 64 > 0 ? D / 64 : 1];
};

// CG: L2 loads (__ldcg) for rows written during this launch (the fused append's slot), else the
// read-only path.
template <int D, bool CG = false>
KVQ_DEV void load_packed_row(PackedRow<D>& r, const uint8_t* crow, const uint8_t* srow) {
#pragma unroll
  for (int k = 0; k < D / 32; ++k)
    r.c[k] = CG ? __ldcg(reinterpret_cast<const uint4*>(crow) + k) : __ldg(reinterpret_cast<const uint4*>(crow) + k);
  if (D == 128) {
    uint2 s2 = CG ? __ldcg(reinterpret_cast<const uint2*>(srow)) : __ldg(reinterpret_cast<const uint2*>(srow));
    r.s[0] = s2.x;
    r.s[1] = s2.y;
  } else {
    r.s[0] = CG ? __ldcg(reinterpret_cast<const uint32_t*>(srow)) : __ldg(reinterpret_cast<const uint32_t*>(srow));
  }
}

// K^' = dec(code) * dec(s) in fp16 (exact), written as one 128B-swizzled tile row.
template <int D>
KVQ_DEV void store_dequant_row(uint32_t base, int r, const PackedRow<D>& pr) {
#pragma unroll
  for (int j = 0; j < D / 16; ++j) {
    const uint32_t sb = (pr.s[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    const uint32_t s2 = f16x2_from_e4m3x2(sb | (sb << 8));
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int wi = 2 * j + half;  // 32-bit code word index
      const uint4 q = pr.c[wi >> 2];
      const uint32_t w = (wi & 3) == 0 ? q.x : (wi & 3) == 1 ? q.y : (wi & 3) == 2 ? q.z : q.w;
      uint32_t o[4];
      dequant_word_f16(w, s2, o);
      st_shared_v4(chunk_addr(base, r, wi), o[0], o[1], o[2], o[3]);
    }
  }
}

// Q row -> fp16 (bf16 in bf16-KV mode) into a tile row.
//
// Range (kvq.h, chunk_attention): bf16 / fp32 queries are scaled by 2^shift per row so that the
// row's max |q| lands in [2^14, 2^15) before the fp16 conversion -- a power-of-two scale is exact,
// so every finite query row fits fp16's normal range (values below max|q| * 2^-29 lose bits, a
// relative 2^-29 of the row's largest term), and 2^-shift (returned as qscale) joins the row's
// exponent scale.  For rows already inside fp16's range the scores are bit-identical to the
// unscaled kernel (scaling by 2^shift commutes with every rounding).  A non-finite query element
// is reported as KVQ_ENONFINITE with its flat index in Q.
// SUM: also returns sum_u Q_iu in unscaled units (fp32; the K-smoothing restitution term, see
// attn_ws_kernel).  QSPLIT (fp32 Q): hi = RN16(q 2^shift) into the tile, lo = RN16(q 2^shift - hi)
// (exact in fp32) into the lo tile, and the sum is over the input values.
struct QRow {
  float qsum, qscale;
  bool nonfinite;  // a query element was inf / NaN (reported; the row's scores are then not range-checked)
};
KVQ_DEV void report_status(DevStatus* st, int code, unsigned long long index) {
  if (st == nullptr) return;
  atomicCAS(&st->code, 0, code);
  atomicMin(&st->first_bad, index);
}

template <int D, bool MMA_BF16, bool SUM = false, bool QSPLIT = false>
KVQ_DEV QRow load_q_row(uint32_t base, uint32_t base_lo, int r, const void* Q, int q_dtype, int64_t row_index,
                        bool valid, DevStatus* status) {
  float qsum = 0.0f;
  // pass 1: max |q| bit pattern of the row (integer max on non-negative floats; NaN / inf sort last)
  const bool scaled = valid && !MMA_BF16 && (QSPLIT || q_dtype == DT_BF16);
  float sc = 1.0f, qscale = 1.0f;
  bool nonfinite = false;
  if (scaled) {
    uint32_t amax = 0;
    int bad = -1;
    if (!QSPLIT) {
      const uint4* src = reinterpret_cast<const uint4*>((const __nv_bfloat16*)Q + row_index * D);
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        const uint4 v = __ldg(src + c);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t lo = w[k] & 0x7FFFu, hi = (w[k] >> 16) & 0x7FFFu;
          if (bad < 0 && lo >= 0x7F80u) bad = 8 * c + 2 * k;
          if (bad < 0 && hi >= 0x7F80u) bad = 8 * c + 2 * k + 1;
          amax = max(amax, max(lo, hi) << 16);
        }
      }
    } else {
      const float4* src = reinterpret_cast<const float4*>((const float*)Q + row_index * D);
#pragma unroll
      for (int c = 0; c < D / 4; ++c) {
        const float4 v = __ldg(src + c);
        const uint32_t w[4] = {__float_as_uint(v.x) & 0x7FFFFFFFu, __float_as_uint(v.y) & 0x7FFFFFFFu,
                               __float_as_uint(v.z) & 0x7FFFFFFFu, __float_as_uint(v.w) & 0x7FFFFFFFu};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (bad < 0 && w[k] >= 0x7F800000u) bad = 4 * c + k;
          amax = max(amax, w[k]);
        }
      }
    }
    nonfinite = bad >= 0;
    if (nonfinite) report_status(status, -6 /* KVQ_ENONFINITE */, (unsigned long long)(row_index * D + bad));
    if (amax != 0 && amax < 0x7F800000u) {
      int ex;
      frexpf(__uint_as_float(amax), &ex);  // amax in [2^(ex-1), 2^ex)
      const int shift = min(15 - ex, 120);
      sc = ldexpf(1.0f, shift);
      qscale = ldexpf(1.0f, -shift);
    }
  }
#pragma unroll
  for (int c = 0; c < D / 8; ++c) {
    uint32_t o[4] = {0, 0, 0, 0}, ol[4] = {0, 0, 0, 0};
    if (valid) {
      float f[8];
      if (!QSPLIT && q_dtype == DT_FP16) {  // NVFP4-exchanged Q: fp16 dec(c) dec(s), copied as is
        const uint4 v = __ldg(reinterpret_cast<const uint4*>((const __half*)Q + row_index * D) + c);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
      } else if (!QSPLIT && q_dtype == DT_BF16) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)Q + row_index * D) + c);
        if (MMA_BF16) {
          o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
        } else {
          uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k)
            o[k] = pack_half2(__uint_as_float(w[k] << 16) * sc, __uint_as_float(w[k] & 0xFFFF0000u) * sc);
        }
      } else {
        const float4* src = reinterpret_cast<const float4*>((const float*)Q + row_index * D) + 2 * c;
        float4 a = __ldg(src), b = __ldg(src + 1);
        f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float f0 = f[2 * k] * sc, f1 = f[2 * k + 1] * sc;
          o[k] = MMA_BF16 ? pack_bf162(f[2 * k], f[2 * k + 1]) : pack_half2(f0, f1);
          if (QSPLIT) {
            const float2 h2 = __half22float2(*reinterpret_cast<const __half2*>(&o[k]));
            ol[k] = pack_half2(f0 - h2.x, f1 - h2.y);
            if (SUM) qsum += f[2 * k] + f[2 * k + 1];
          }
        }
      }
    }
    if (SUM && !QSPLIT) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&o[k]));
        qsum += f2.x + f2.y;
      }
    }
    st_shared_v4(chunk_addr(base, r, c), o[0], o[1], o[2], o[3]);
    if (QSPLIT) st_shared_v4(chunk_addr(base_lo, r, c), ol[0], ol[1], ol[2], ol[3]);
  }
  if (SUM && !QSPLIT) qsum *= qscale;  // the fp16 values were scaled by 2^shift
  return QRow{qsum, qscale, nonfinite};
}

// Tile iteration over the key segments: tile = 128 slot-aligned rows, valid rows [lo, hi).
struct TileIter {
  int seg, t0;
};
KVQ_DEV bool tile_first(const AttnParams& p, TileIter& it) {
  it.seg = 0;
  if (p.nseg == 0) return false;
  it.t0 = p.seg[0].begin & ~127;
  return true;
}
KVQ_DEV bool tile_next(const AttnParams& p, TileIter& it) {
  it.t0 += 128;
  if (it.t0 < p.seg[it.seg].end) return true;
  if (++it.seg >= p.nseg) return false;
  it.t0 = p.seg[it.seg].begin & ~127;
  return true;
}
KVQ_DEV int count_tiles(const AttnParams& p) {
  int n = 0;
  for (int s = 0; s < p.nseg; ++s) n += ((p.seg[s].end + 127) >> 7) - (p.seg[s].begin >> 7);
  return n;
}

// ---------------------------------------------------------------------------------------------
// Persistent stream-K schedule.  A work UNIT is (head, pair of 128-query tiles); every unit has
// the same n key tiles.  The U*n (unit, tile) steps are cut into gridDim.x equal contiguous
// ranges, one per CTA (one CTA per SM), so every SM gets the same tensor-core work regardless of
// how U compares with the SM count.  A range covers whole units (written directly) and at most
// a partial unit at each end; a partial piece writes unnormalized O (real units), the running
// max m (log2 domain) and the row sum l to a workspace slot: slot 2c for CTA c's first piece,
// 2c+1 for its last, and combine_kernel merges the pieces of every split unit in a fixed order.
struct Piece {
  int unit, tb, te;   // unit index, tile range [tb, te)
  bool full;          // covers the whole unit -> final output
  int slot;           // workspace slot when !full
};

// Hybrid schedule (AttnParams::full_units, a multiple of the grid G): the first full_units units
// are handed out whole in waves -- CTA c takes units c, c + G, ... -- so the CTAs of one wave walk
// the key tiles of the same heads in step (L2 reuse of a window that does not fit L2: the bf16-KV
// mode); the remaining (units - full_units) * n steps are cut into G equal contiguous stream-K
// ranges.  full_units = 0 is plain stream-K.
// Step indices are 32-bit (launch_t checks units * n < 2^31): the MMA warp's 80 registers hold the
// schedule next to its descriptors without spilling.
struct Sched {
  int base, W;  // first stream-K step, stream-K steps
  int G, n, waves;
};
KVQ_DEV Sched make_sched(const AttnParams& p, int n, int G) {
  return Sched{p.full_units * n, (p.units - p.full_units) * n, G, n, p.full_units / G};
}
KVQ_DEV int range_begin(const Sched& s, int c) {
  return s.base + (int)(((unsigned long long)(unsigned)s.W * (unsigned)c) / (unsigned)s.G);
}

// piece k of CTA c (k = 0, 1, ...); false when past the end of the range
KVQ_DEV bool get_piece(const Sched& sc, int c, int k, Piece& pc) {
  if (k < sc.waves) {
    pc.unit = c + k * sc.G;
    pc.tb = 0;
    pc.te = sc.n;
    pc.full = true;
    pc.slot = -1;
    return true;
  }
  k -= sc.waves;
  const int n = sc.n;
  const int beg = range_begin(sc, c), end = range_begin(sc, c + 1);
  int s = beg;
  for (int i = 0; i < k && s < end; ++i) s = min((s / n + 1) * n, end);
  if (s >= end) return false;
  const int u = s / n;
  pc.unit = u;
  pc.tb = s - u * n;
  pc.te = min((u + 1) * n, end) - u * n;
  pc.full = (pc.tb == 0 && pc.te == n);
  pc.slot = (s == beg) ? 2 * c : 2 * c + 1;
  return true;
}

// position the tile iterator at tile index tb of the key-tile sequence
KVQ_DEV void tile_seek(const AttnParams& p, int tb, TileIter& it) {
  int s = 0;
  for (; s < p.nseg; ++s) {
    const int nt = ((p.seg[s].end + 127) >> 7) - (p.seg[s].begin >> 7);
    if (tb < nt) break;
    tb -= nt;
  }
  it.seg = s;
  it.t0 = (p.seg[s].begin & ~127) + 128 * tb;
}

// debug timeline (CTA 0, first 64 tiles): SM clock at role events, only when p.trace != null, and
// compiled in only with -DKVQ_TRACE_BUILD=1 (tools/trace_attn.py): the runtime check alone cost the
// MMA warp (80 registers) two spill/fill pairs per tile in its issue loop.
#ifndef KVQ_TRACE_BUILD
#define KVQ_TRACE_BUILD 0
#endif
#ifdef KVQ_TRACE_SOFTMAX
#define KVQ_TRACE_SM(tile, ev) \
  do {                                                                                             \
    if (qi == 0) KVQ_TRACE(tile, ev);                                                              \
  } while (0)
#else
#define KVQ_TRACE_SM(tile, ev) \
  do {                         \
  } while (0)
#endif
#if KVQ_TRACE_BUILD
#define KVQ_TRACE(tile, ev)                                                                        \
  do {                                                                                           \
    if (p.trace != nullptr && blockIdx.x == 0 && (tile) < 64 && ((tid & 127) == 0 || tid == 384)) \
      p.trace[(tile) * 16 + (ev)] = clock64();                                                   \
  } while (0)
#else
#define KVQ_TRACE(tile, ev) \
  do {                      \
  } while (0)
#endif

// ---------------------------------------------------------------------------------------------
// Append fused into the attention launch (AttnParams::ap_*; kv_quantize_append's bytes exactly:
// definition R1 through quant_core.cuh, whose arithmetic is explicit round-to-nearest intrinsics).
KVQ_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
KVQ_DEV void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
KVQ_DEV float ld_relaxed_f32(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
KVQ_DEV unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// The nthreads threads of a group (lane `lt`) together wait until every CTA's done tag of this launch
// (epoch E) is set: each polls its own tags with relaxed loads (an acquire per poll costs ~0.3 us;
// 148 of them in sequence were 40 us), then one acquire fence; the caller then syncs the group.
KVQ_DEV void ap_wait_all_done(const unsigned long long* sync, int G, unsigned long long E, int lt, int nthreads) {
  for (int i = lt; i < G; i += nthreads)
    while (ld_relaxed_u64(sync + 1 + 2 * kMaxCtas + i) != E + 1) __nanosleep(64);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// flat index of the first non-finite element of a block (rare path)
template <int DT>
KVQ_DEV int first_nonfinite16(const uint8_t* src) {
  for (int e = 0; e < 16; ++e) {
    const uint32_t b = DT == DT_BF16 ? ((uint32_t)reinterpret_cast<const uint16_t*>(src)[e] & 0x7FFFu) << 16
                                     : reinterpret_cast<const uint32_t*>(src)[e] & 0x7FFFFFFFu;
    if (b >= 0x7F800000u) return e;
  }
  return 0;
}

// Warps 13-15 of CTA c (qt = 0..95): amax of the CTA's block range of K and V -> publish (epoch-tagged)
// -> every CTA's partial -> g = RN32(amax / 2688) -> quantize the range into the slot -> done tag.
// Cooperative launch: all G CTAs are co-resident, so the partial exchange cannot deadlock.
template <int D, int DT>
KVQ_DEV void fused_append_role(const AttnParams& p, uint8_t* smem_ap, int qt, unsigned long long E) {
#define KVQ_TRACE_AP(ev)                                                           \
  do {                                                                             \
    if (p.trace != nullptr && blockIdx.x == 0 && qt == 0) p.trace[63 * 16 + (ev)] = clock64(); \
  } while (0)
  KVQ_TRACE_AP(0);
  constexpr int kNB = D / 16, kUB = 16 * (DT == DT_BF16 ? 2 : 4);
  const int G = gridDim.x, c = blockIdx.x, H = p.H;
  const int64_t n = (int64_t)p.Tq * H * D, nblk = n / 16;
  const int64_t u0 = nblk * c / G, u1 = nblk * (c + 1) / G;
  unsigned long long* sync = p.ap_sync;
  uint32_t* red = reinterpret_cast<uint32_t*>(smem_ap + 16);  // [2 tensors][3 warps]
  float* gsh = reinterpret_cast<float*>(smem_ap + 48);         // g of K, V (NaN bits: non-finite)
  // ---- A: block maxima (as fp32 bit patterns) over [u0, u1) of K and V, non-finite reported
  uint32_t m[2] = {0u, 0u};
#ifdef KVQ_AP_EXPERIMENT_NOWORK  // timing experiment only (wrong bytes): the exchange without the work
  for (int t = 0; t < 0; ++t) {
#else
  for (int t = 0; t < 2; ++t) {
#endif
    const uint8_t* x = static_cast<const uint8_t*>(p.ap_x[t]);
    for (int64_t u = u0 + qt; u < u1; u += 96) {
      uint32_t bm = 0;
#pragma unroll
      for (int k = 0; k < kUB / 16; ++k) bm = max(bm, vec_absmax_bits<DT>(ld_nc_v4(x + u * kUB + 16 * k)));
      if (bm >= 0x7F800000u)
        report_status(p.status, -6 /* KVQ_ENONFINITE */,
                      (unsigned long long)(t * n + u * 16 + first_nonfinite16<DT>(x + u * kUB)));
      m[t] = max(m[t], bm);
    }
  }
  KVQ_TRACE_AP(1);
  const int w = qt >> 5;
  for (int t = 0; t < 2; ++t) {
    const uint32_t v = warp_max_u32(m[t]);
    if ((qt & 31) == 0) red[t * 3 + w] = v;
  }
  named_bar_sync(6, 96);
  if (qt == 0)
    for (int t = 0; t < 2; ++t)
      st_release_u64(sync + 1 + t * kMaxCtas + c, ((E + 1) << 32) | max(max(red[t * 3], red[t * 3 + 1]), red[t * 3 + 2]));
  // ---- B: every CTA's partial of this launch (polled in parallel, relaxed) -> the tensor amax -> g
  uint32_t pa[2] = {0u, 0u};
  for (int t = 0; t < 2; ++t)
    for (int i = qt; i < G; i += 96) {
      unsigned long long v;
      while (((v = ld_relaxed_u64(sync + 1 + t * kMaxCtas + i)) >> 32) != E + 1) __nanosleep(64);
      pa[t] = max(pa[t], (uint32_t)v);
    }
  named_bar_sync(6, 96);  // every CTA's partial is in (red[] is free again)
  for (int t = 0; t < 2; ++t) {
    const uint32_t v = warp_max_u32(pa[t]);
    if ((qt & 31) == 0) red[t * 3 + w] = v;
  }
  named_bar_sync(6, 96);
  if (qt < 2) {
    const uint32_t a = max(max(red[qt * 3], red[qt * 3 + 1]), red[qt * 3 + 2]);
    gsh[qt] = a >= 0x7F800000u ? __uint_as_float(0x7FC00000u) : (a == 0 ? 1.0f : __fdiv_rn(__uint_as_float(a), 2688.0f));
  }
  named_bar_sync(6, 96);
  KVQ_TRACE_AP(2);
  // ---- C: quantize [u0, u1) into the slot rows (head-major: row h * head_stride_rows + t)
#ifdef KVQ_AP_EXPERIMENT_NOWORK
  for (int t = 0; t < 0; ++t) {
#else
  for (int t = 0; t < 2; ++t) {
#endif
    const float g = gsh[t];
    if (g != g) continue;  // non-finite tensor: reported, slot bytes undefined (as kv_quantize_append)
    const float rg = __frcp_rn(g);
    const bool exact = !(g >= 0x1p-60f && g <= 0x1p60f);
    const uint8_t* x = static_cast<const uint8_t*>(p.ap_x[t]);
    for (int64_t u = u0 + qt; u < u1; u += 96) {
      float v[1][16];
      unpack_block16<DT>(x + u * kUB, v[0]);
      uint32_t sb[1], w0[1], w1[1];
      const uint32_t flags = exact ? 1u : quantize_blocks_fast<1, false>(v, g, rg, sb, w0, w1);
      if (flags) quantize_block16_exact<false>(v[0], g, sb[0], w0[0], w1[0]);
      const int64_t row = u / kNB;
      const int j = (int)(u - row * kNB);
      const int64_t tt = row / H, h = row - tt * H;
      const int64_t orow = h * p.head_stride_rows + tt;
      *reinterpret_cast<uint2*>(p.ap_codes[t] + orow * (D / 2) + j * 8) = make_uint2(w0[0], w1[0]);
      p.ap_scales[t][orow * kNB + j] = (uint8_t)sb[0];
    }
    if (c == 0 && qt == 0) p.ap_g[t] = g;
  }
  // ---- D: this CTA's bytes are visible device-wide -> done tag; CTA 0 advances the launch epoch
  KVQ_TRACE_AP(3);
  __threadfence();
  named_bar_sync(6, 96);
  if (qt == 0) st_release_u64(sync + 1 + 2 * kMaxCtas + c, E + 1);
  if (c == 0) {  // every CTA has read E (at its start) and finished: advance the launch epoch
    ap_wait_all_done(sync, G, E, qt, 96);
    named_bar_sync(6, 96);
    KVQ_TRACE_AP(4);
    if (qt == 0) st_release_u64(sync, E + 1);
  }
#undef KVQ_TRACE_AP
}

// SMOOTH (K-smoothing, reading Z20): the cache holds K_bar = K - m per key row,
// and the score is restored exactly as q.k = q.k_bar + m_j sum_u q_u -- a rank-1 term added in
// fp32 to the scaled MMA scores before the row max, from the fp32 row sum of the (rounded) Q row
// and the key means of the tile (one coalesced load per softmax thread, shared through smem).
template <int D, bool NVFP4, bool MMA_BF16, bool SMOOTH, bool QSPLIT, bool APPEND = false>
__global__ void __launch_bounds__(kThreads, 1) attn_ws_kernel(const __grid_constant__ AttnParams p) {
  using SM = WsSmem<D, QSPLIT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // tile bases: Q_i = sbase + i*T, K_b = sbase + (2+b)*T, V_b = sbase + (4+b)*T
  const uint32_t sbase = smem_u32(smem);
  constexpr uint32_t kT = SM::kTile;
#define SQ(i) (sbase + (uint32_t)(i) * kT)
#define SK(b) (sbase + (2u + (uint32_t)(b)) * kT)
#define SV(b) (sbase + (4u + (uint32_t)(b)) * kT)
#define SQL(i) (sbase + (uint32_t)((i) ? SM::kQL1 : SM::kQL0))
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
  uint64_t* kfull = bars + 0;   // [2] dequant -> MMA, per K^ buffer
  uint64_t* vfull = bars + 2;   // [2]
  uint64_t* kempty = bars + 4;  // [2] MMA -> dequant
  uint64_t* vempty = bars + 6;  // [2]
  uint64_t* sfull = bars + 8;   // [2] MMA -> softmax WG i (S_i ready; PV_i(prev) done)
  uint64_t* pfull = bars + 10;  // [2] softmax WG i -> MMA (P_i written, O_i rescaled)
  uint64_t* ofull = bars + 12;  // [2] MMA -> softmax WG i (last PV_i of a piece done)
  uint64_t* qfull = bars + 14;  // [2] softmax WG i -> MMA (Q_i tile of a piece loaded)
  uint64_t* sfree = bars + 16;  // [2] softmax WG i -> MMA (S_i loaded to registers; kRotate only)
  uint64_t* ofree = bars + 18;  // [2] MMA -> softmax WG i (PV_i of a tile done: O_i may be rescaled; kRotate)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 20);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int H = p.H;
  const int n = count_tiles(p);
  const int G = gridDim.x, c = blockIdx.x;
  const Sched sch = make_sched(p, n, G);

  if (warp == 12) tmem_alloc(tslot, 512);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(kfull + b, NVFP4 ? 128 : 1);  // dequant: one arrival per key row; bf16 KV: the TMA issuer
      mbar_init(vfull + b, NVFP4 ? 128 : 1);
      mbar_init(kempty + b, 1);
      mbar_init(vempty + b, 1);
      mbar_init(sfull + b, 1);
      mbar_init(pfull + b, kSplitRows ? 256 : 128);  // split rows: both halves of every row arrive
      mbar_init(ofull + b, 1);
      mbar_init(qfull + b, 128);
      mbar_init(sfree + b, 128);
      mbar_init(ofree + b, 1);
    }
    fence_mbar_init();
    if (APPEND) {
      *reinterpret_cast<unsigned long long*>(smem + SM::kAp) = ld_acquire_u64(p.ap_sync);
      if (p.trace != nullptr) {  // debug: per-CTA start time (ns)
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        p.trace[1024 + 2 * kMaxCtas + blockIdx.x] = t0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // fused append: this launch's epoch, read by thread 0 before any CTA can finish (fused_append_role);
  // each role re-reads it from shared memory where it needs it, so it does not occupy registers
  auto launch_epoch = [&]() { return *reinterpret_cast<const volatile unsigned long long*>(smem + SM::kAp); };
  // Pieces of this CTA and their processing order.  APPEND: a first piece that starts inside a unit is
  // that unit's tail -- it ends with the unit's last key tiles, the current chunk's -- so it is
  // processed last, long after the append has finished; every role walks the same order.
  int npc = 0;
  bool defer = false;
  if (APPEND) {
    Piece t;
    while (get_piece(sch, c, npc, t)) ++npc;
    if (npc > 1) {
      get_piece(sch, c, 0, t);
      defer = t.tb > 0;
    }
  }
  auto next_piece = [&](int kk, Piece& pc) -> bool {
    if (!APPEND) return get_piece(sch, c, kk, pc);
    if (kk >= npc) return false;
    get_piece(sch, c, defer ? (kk + 1) % npc : kk, pc);
    return true;
  };

  if (warp < 8) {
   if constexpr (kSplitRows) {
    // ================================================================ softmax, split rows (kSplitRows)
    reg_alloc<APPEND ? kRegSoftmaxAp : kRegSoftmax>();
    const int half = warp >> 2;  // this warpgroup's key columns of every row: [64 half, 64 half + 64)
    const int row = tid & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    float* pmax = reinterpret_cast<float*>(smem + SM::kXch);  // [2 step parities][2 halves][128]
    float* qinf = pmax + 2 * 2 * 128;                          // [2 tiles][128][3]
    float* lsum = qinf + 2 * 128 * 3;                          // [2 tiles][2 halves][128]
    int g = 0;     // key-tile counter (barrier parity; both query tiles advance together)
    int step = 0;  // (key tile, query tile) steps: exchange-buffer parity
    const float sl2 = p.q_scale ? p.scale_log2 * __ldg(p.q_scale) : p.scale_log2;
    bool gcur_ok = false;  // APPEND: the appended slot's g, loaded once it is in place
    float gk_cur = 1.0f, gv_cur = 1.0f;
    Piece pc;
    for (int k = 0; next_piece(k, pc); ++k) {
      const int h = pc.unit / p.qpairs, q0 = (pc.unit - h * p.qpairs) * 256;
      {  // warpgroup `half` loads query tile `half` and publishes each row's scales for both halves
        const int tq = q0 + 128 * half + row;
        const QRow qr = load_q_row<D, MMA_BF16, SMOOTH, QSPLIT>(SQ(half), SQL(half), row, p.Q, p.q_dtype,
                                                                (int64_t)tq * H + h, tq < p.Tq, p.status);
        float* q3 = qinf + (half * 128 + row) * 3;
        q3[0] = qr.qsum * sl2;
        q3[1] = sl2 * qr.qscale;  // this row's exponent scale (Q was scaled by 1/qscale)
        q3[2] = qr.nonfinite ? 1.0f : 0.0f;
        fence_proxy_async_smem();
        mbar_arrive(qfull + half);
      }
      named_bar_sync(8, 256);
      float sl2q[2], qsb[2], m_run[2], l_run[2], gv_run[2];
      bool rrep[2];
#pragma unroll
      for (int qi = 0; qi < 2; ++qi) {
        const float* q3 = qinf + (qi * 128 + row) * 3;
        qsb[qi] = q3[0];
        sl2q[qi] = q3[1];
        rrep[qi] = q3[2] != 0.0f;
        m_run[qi] = -INFINITY;
        l_run[qi] = 0.0f;
        gv_run[qi] = 1.0f;
      }
      TileIter it;
      tile_seek(p, pc.tb, it);
      for (int j = 0; j < pc.te - pc.tb; ++j, ++g, tile_next(p, it)) {
        const AttnSeg& sg = p.seg[it.seg];
        const int lo = max(sg.begin - it.t0, 0), hi = min(sg.end - it.t0, 128);
        float gk = 1.0f, gv = 1.0f;
        if (NVFP4) {
          if (APPEND && sg.slot == p.ap_slot) {  // g of the slot appended by this launch: after CTA 0's done tag
            if (!gcur_ok) {
              const unsigned long long Ec = *reinterpret_cast<const volatile unsigned long long*>(smem + SM::kAp);
              while (ld_relaxed_u64(p.ap_sync + 1 + 2 * kMaxCtas) != Ec + 1) __nanosleep(64);
              asm volatile("fence.acq_rel.gpu;" ::: "memory");
              gk_cur = ld_relaxed_f32(p.ap_g);
              gv_cur = ld_relaxed_f32(p.ap_g + 1);
              gcur_ok = true;
            }
            gk = gk_cur;
            gv = gv_cur;
          } else {
            gk = __ldg(p.g + 2 * sg.slot);
            gv = __ldg(p.g + 2 * sg.slot + 1);
          }
        }
        float mean_r = 0.0f;  // SMOOTH: key `row`'s mean, loaded by half 0, shared through smem
        if (SMOOTH && half == 0 && row >= lo && row < hi)
          mean_r = __ldg(p.mean_k + (int64_t)h * p.head_stride_rows + (int64_t)sg.slot * p.T_pad + it.t0 + row);
#pragma unroll  // the per-tile-pair state (m_run[qi], ...) stays in registers
        for (int qi = 0; qi < 2; ++qi, ++step) {
          const uint32_t tS = tmem + 128 * qi + lane_off;
          const uint32_t tO = tmem + 256 + 128 * qi + lane_off;
          const float cs = gk * sl2q[qi];
          KVQ_TRACE(g, 3 * qi + 0);
          mbar_wait(sfull + qi, g & 1);
          KVQ_TRACE(g, 3 * qi + 1);
          tc_fence_after();
          uint32_t s[64];
          KVQ_TMEM_LD32(tS + 64 * half, s);
          KVQ_TMEM_LD32(tS + 64 * half + 32, (s + 32));
          if (SMOOTH && qi == 0 && half == 0)
            (reinterpret_cast<float*>(smem + SM::kMean) + (j & 1) * 128)[row] = mean_r;
          tmem_ld_wait();
          KVQ_TRACE_SM(g, 12);
          if (SMOOTH) {  // y = s * cs + m_j * sum(q) * scale_log2 (log2 units), in place
            if (qi == 0) named_bar_sync(8, 256);  // the tile's key means are in place
            const float* mbuf = reinterpret_cast<const float*>(smem + SM::kMean) + (j & 1) * 128 + 64 * half;
            const uint64_t cs2s = f32x2_pack(cs, cs), qsb2 = f32x2_pack(qsb[qi], qsb[qi]);
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
              const float2 m2 = reinterpret_cast<const float2*>(mbuf)[kk];
              const uint64_t b2 = fmul2(f32x2_pack(m2.x, m2.y), qsb2);
              const uint64_t y2 = ffma2(f32x2_pack(__uint_as_float(s[2 * kk]), __uint_as_float(s[2 * kk + 1])), cs2s, b2);
              float y0, y1;
              f32x2_unpack(y2, y0, y1);
              s[2 * kk] = __float_as_uint(y0);
              s[2 * kk + 1] = __float_as_uint(y1);
            }
          }
          // this half's row max over valid keys (column 64 half + kk)
          const int clo = lo - 64 * half, chi = hi - 64 * half;
          if (clo > 0 || chi < 64) {
#pragma unroll
            for (int kk = 0; kk < 64; ++kk)
              if (kk < clo || kk >= chi) s[kk] = __float_as_uint(-INFINITY);
          }
          float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
          for (int kk = 0; kk < 64; kk += 8) {
            mx0 = fmax3(mx0, __uint_as_float(s[kk]), __uint_as_float(s[kk + 1]));
            mx1 = fmax3(mx1, __uint_as_float(s[kk + 2]), __uint_as_float(s[kk + 3]));
            mx2 = fmax3(mx2, __uint_as_float(s[kk + 4]), __uint_as_float(s[kk + 5]));
            mx3 = fmax3(mx3, __uint_as_float(s[kk + 6]), __uint_as_float(s[kk + 7]));
          }
          float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
          // the row's max = max of both halves' (double-buffered by step parity)
          pmax[((step & 1) * 2 + half) * 128 + row] = mx;
          named_bar_sync(8, 256);
          mx = fmaxf(mx, pmax[((step & 1) * 2 + (half ^ 1)) * 128 + row]);
          // lazy max, identical in both halves (same inputs): see the per-tile design
          const float m_tile = SMOOTH ? mx : mx * cs;
          const float m_new = (j == 0 || m_tile > m_run[qi] + kLazyLog2) ? fmaxf(m_run[qi], m_tile) : m_run[qi];
          const float alpha = ex2_approx(m_run[qi] - m_new);
          KVQ_TRACE_SM(g, 13);
          const float cse = SMOOTH ? 1.0f : cs;
          const uint64_t cs2 = f32x2_pack(cse, cse), mneg2 = f32x2_pack(-m_new, -m_new);
          uint64_t acc0 = 0, acc1 = 0;
          float la[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int kk = 0; kk < 32; ++kk) {
            const uint64_t x2 = ffma2(f32x2_pack(__uint_as_float(s[2 * kk]), __uint_as_float(s[2 * kk + 1])), cs2, mneg2);
            float x0, x1, p0, p1;
            f32x2_unpack(x2, x0, x1);
            if ((kk & 7) < kPolyPairs) {
              exp2_poly_pair(x0, x1, p0, p1);
            } else {
              p0 = ex2_approx(x0);
              p1 = ex2_approx(x1);
            }
            const uint32_t pk = MMA_BF16 ? pack_bf162(p0, p1) : pack_half2(p0, p1);
            s[kk] = pk;
            if (MMA_BF16) {
              const uint64_t r2 = f32x2_pack(__uint_as_float(pk << 16), __uint_as_float(pk & 0xFFFF0000u));
              if (kk & 1) acc1 = fadd2(acc1, r2);
              else acc0 = fadd2(acc0, r2);
            } else {
              asm("{ .reg .b16 l, h;\n mov.b32 {l, h}, %4;\n add.rn.f32.f16 %0, l, %0;\n add.rn.f32.f16 %1, h, %1;\n}"
                  : "+f"(la[(kk & 1) * 2]), "+f"(la[(kk & 1) * 2 + 1]) : "f"(0.0f), "f"(0.0f), "r"(pk));
            }
          }
          float a0, a1, b0, b1;
          f32x2_unpack(acc0, a0, a1);
          f32x2_unpack(acc1, b0, b1);
          l_run[qi] = l_run[qi] * alpha + ((a0 + a1) + (b0 + b1)) + ((la[0] + la[1]) + (la[2] + la[3]));
          KVQ_TRACE_SM(g, 14);
          // P of this half's 64 keys = 32 fp16x2 columns at [32 half, +32) of S_qi (the other half has
          // loaded its S: both passed the barrier above)
          KVQ_TMEM_ST32(tS + 32 * half, s);
          if (j > 0) {  // O_qi (this half's D/2 columns) in units of the current chunk's g_V
            const float f = alpha * (gv_run[qi] / gv);
            if (!__all_sync(0xffffffffu, f == 1.0f)) {
              const uint64_t f2 = f32x2_pack(f, f);
              uint32_t* o = s + 32;  // the upper half of s[] is free once P is packed
#pragma unroll
              for (int cc = 0; cc < D / 64; ++cc) {
                const uint32_t ta = tO + (D / 2) * half + 32 * cc;
                KVQ_TMEM_LD32(ta, o);
                tmem_ld_wait();
#pragma unroll
                for (int kk = 0; kk < 32; kk += 2) {
                  float x0, x1;
                  f32x2_unpack(fmul2(f32x2_pack(__uint_as_float(o[kk]), __uint_as_float(o[kk + 1])), f2), x0, x1);
                  o[kk] = __float_as_uint(x0);
                  o[kk + 1] = __float_as_uint(x1);
                }
                KVQ_TMEM_ST32(ta, o);
              }
            }
          }
          gv_run[qi] = gv;
          m_run[qi] = m_new;
          tmem_st_wait();
          KVQ_TRACE_SM(g, 15);
          tc_fence_before();
          mbar_arrive(pfull + qi);
          KVQ_TRACE(g, 3 * qi + 2);
        }
      }
      // ---- piece epilogue: combine the halves' row sums (fixed order: half 0 + half 1)
#pragma unroll
      for (int qi = 0; qi < 2; ++qi) lsum[(qi * 2 + half) * 128 + row] = l_run[qi];
      named_bar_sync(8, 256);
#pragma unroll
      for (int qi = 0; qi < 2; ++qi) {
        const float l_tot = lsum[(qi * 2) * 128 + row] + lsum[(qi * 2 + 1) * 128 + row];
        const int t = q0 + 128 * qi + row;
        const uint32_t tO = tmem + 256 + 128 * qi + lane_off;
        // score range (reading Z25), as in the per-tile design
        if (half == 0 && !(fabsf(m_run[qi]) < kScoreRangeLog2) && !rrep[qi] && t < p.Tq)
          report_status(p.status, -7 /* KVQ_ERANGE */, (unsigned long long)(((int64_t)t * H + h) * D));
        mbar_wait(ofull + qi, k & 1);
        tc_fence_after();
        const float f = pc.full ? gv_run[qi] / l_tot : gv_run[qi];
        float* wsO = p.ws + (size_t)pc.slot * p.ws_slot_floats + (size_t)(128 * qi + row) * D;
        if (!pc.full && t < p.Tq && half == 0) {
          float* wml = p.ws + (size_t)pc.slot * p.ws_slot_floats + 256 * D;
          wml[128 * qi + row] = m_run[qi];
          wml[256 + 128 * qi + row] = l_tot;
        }
#pragma unroll
        for (int cc = 0; cc < D / 64; ++cc) {  // this half's D/2 columns, 32 at a time
          const int col = (D / 2) * half + 32 * cc;
          uint32_t o[32];
          KVQ_TMEM_LD32(tO + col, o);
          tmem_ld_wait();
          if (t < p.Tq) {
            if (!pc.full) {
              float4* dst = reinterpret_cast<float4*>(wsO + col);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                dst[kk] = make_float4(__uint_as_float(o[4 * kk]) * f, __uint_as_float(o[4 * kk + 1]) * f,
                                      __uint_as_float(o[4 * kk + 2]) * f, __uint_as_float(o[4 * kk + 3]) * f);
            } else {
              const int64_t base = ((int64_t)t * H + h) * D + col;
              if (p.out_dtype == DT_FP32) {
                float4* dst = reinterpret_cast<float4*>((float*)p.O + base);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                  dst[kk] = make_float4(__uint_as_float(o[4 * kk]) * f, __uint_as_float(o[4 * kk + 1]) * f,
                                        __uint_as_float(o[4 * kk + 2]) * f, __uint_as_float(o[4 * kk + 3]) * f);
              } else {
                uint4* dst = reinterpret_cast<uint4*>((__nv_bfloat16*)p.O + base);
                if (p.o_peer[0] != nullptr) {  // f4 direct: straight into the owning rank's O shard
                  const int r = t / p.o_Ts;
                  dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o_peer[r]) +
                                                 ((int64_t)(t - r * p.o_Ts) * p.o_H + p.o_h0 + h) * D + col);
                }
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  dst[kk] = make_uint4(pack_bf162(__uint_as_float(o[8 * kk]) * f, __uint_as_float(o[8 * kk + 1]) * f),
                                       pack_bf162(__uint_as_float(o[8 * kk + 2]) * f, __uint_as_float(o[8 * kk + 3]) * f),
                                       pack_bf162(__uint_as_float(o[8 * kk + 4]) * f, __uint_as_float(o[8 * kk + 5]) * f),
                                       pack_bf162(__uint_as_float(o[8 * kk + 6]) * f, __uint_as_float(o[8 * kk + 7]) * f));
              }
            }
          }
        }
      }
    }
   } else {
    // ================================================================ softmax WG (tile qi)
    reg_alloc<APPEND ? kRegSoftmaxAp : kRegSoftmax>();
    const int qi = warp >> 2;
    const int row = tid & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + 128 * qi + lane_off;
    const uint32_t tO = tmem + 256 + 128 * qi + lane_off;
    int g = 0;  // global tile counter (barrier parity)
    // exponent scale (log2 units); NVFP4-exchanged Q carries g_Q (device scalar) into it
    const float sl2 = p.q_scale ? p.scale_log2 * __ldg(p.q_scale) : p.scale_log2;
    bool gcur_ok = false;  // APPEND: the appended slot's g, loaded once it is in place
    float gk_cur = 1.0f, gv_cur = 1.0f;
    Piece pc;
    for (int k = 0; next_piece(k, pc); ++k) {
      const int h = pc.unit / p.qpairs, q0 = (pc.unit - h * p.qpairs) * 256;
      const int t = q0 + 128 * qi + row;
      const QRow qr = load_q_row<D, MMA_BF16, SMOOTH, QSPLIT>(SQ(qi), SQL(qi), row, p.Q, p.q_dtype,
                                                              (int64_t)t * H + h, t < p.Tq, p.status);
      const uint64_t qsb2 = f32x2_pack(qr.qsum * sl2, qr.qsum * sl2);
      const float sl2q = sl2 * qr.qscale;  // this row's exponent scale (Q was scaled by 1/qscale)
      const bool range_reported = qr.nonfinite;
      fence_proxy_async_smem();
      mbar_arrive(qfull + qi);
      float m_run = -INFINITY, l_run = 0.0f, gv_run = 1.0f;
      TileIter it;
      tile_seek(p, pc.tb, it);
      for (int j = 0; j < pc.te - pc.tb; ++j, ++g, tile_next(p, it)) {
        const AttnSeg& sg = p.seg[it.seg];
        const int lo = max(sg.begin - it.t0, 0), hi = min(sg.end - it.t0, 128);
        float gk = 1.0f, gv = 1.0f;
        if (NVFP4) {
          if (APPEND && sg.slot == p.ap_slot) {  // g of the slot appended by this launch: after CTA 0's done tag
            if (!gcur_ok) {
              const unsigned long long Ec = *reinterpret_cast<const volatile unsigned long long*>(smem + SM::kAp);
              while (ld_relaxed_u64(p.ap_sync + 1 + 2 * kMaxCtas) != Ec + 1) __nanosleep(64);
              asm volatile("fence.acq_rel.gpu;" ::: "memory");
              gk_cur = ld_relaxed_f32(p.ap_g);
              gv_cur = ld_relaxed_f32(p.ap_g + 1);
              gcur_ok = true;
            }
            gk = gk_cur;
            gv = gv_cur;
          } else {
            gk = __ldg(p.g + 2 * sg.slot);
            gv = __ldg(p.g + 2 * sg.slot + 1);
          }
        }
        const float cs = gk * sl2q;
        float mean_r = 0.0f;  // SMOOTH: this thread's key of the tile
        if (SMOOTH && row >= lo && row < hi)
          mean_r = __ldg(p.mean_k + (int64_t)h * p.head_stride_rows + (int64_t)sg.slot * p.T_pad + it.t0 + row);
        KVQ_TRACE(g, 3 * qi + 0);
        mbar_wait(sfull + qi, g & 1);
        KVQ_TRACE(g, 3 * qi + 1);
        tc_fence_after();
        uint32_t s[128];
        uint32_t tSa = tS, tSb = tS + 64;  // S keys 0-63 / 64-127; P goes to tSb (kRotate) or tS
        if (kRotate) {
          uint32_t ra, rb;
          sp_regions(2 * j + qi, ra, rb);
          tSa = tmem + 64u * ra + lane_off;
          tSb = tmem + 64u * rb + lane_off;
        }
        KVQ_TMEM_LD32(tSa, s);
        KVQ_TMEM_LD32(tSa + 32, (s + 32));
        KVQ_TMEM_LD32(tSb, (s + 64));
        KVQ_TMEM_LD32(tSb + 32, (s + 96));
        if (SMOOTH) {  // share the tile's key means within the warpgroup (double-buffered)
          float* mbuf = reinterpret_cast<float*>(smem + SM::kMean) + (qi * 2 + (j & 1)) * 128;
          mbuf[row] = mean_r;
          asm volatile("bar.sync %0, 128;" ::"r"(1 + qi) : "memory");
        }
        tmem_ld_wait();
        if (kRotate) {
          tc_fence_before();
          mbar_arrive(sfree + qi);  // S_i(j) is in registers: its region a may take the next QK
        }
        KVQ_TRACE_SM(g, 12);
        if (SMOOTH) {  // y = s * cs + m_j * sum(q) * scale_log2  (log2 units), in place
          const float* mbuf = reinterpret_cast<const float*>(smem + SM::kMean) + (qi * 2 + (j & 1)) * 128;
          const uint64_t cs2s = f32x2_pack(cs, cs);
#pragma unroll
          for (int kk = 0; kk < 64; ++kk) {
            const float2 m2 = reinterpret_cast<const float2*>(mbuf)[kk];
            const uint64_t b2 = fmul2(f32x2_pack(m2.x, m2.y), qsb2);
            const uint64_t y2 = ffma2(f32x2_pack(__uint_as_float(s[2 * kk]), __uint_as_float(s[2 * kk + 1])), cs2s, b2);
            float y0, y1;
            f32x2_unpack(y2, y0, y1);
            s[2 * kk] = __float_as_uint(y0);
            s[2 * kk + 1] = __float_as_uint(y1);
          }
        }
        // row max over valid keys (raw scores: the scale cs > 0 commutes with max)
        if (lo != 0 || hi != 128) {
#pragma unroll
          for (int kk = 0; kk < 128; ++kk)
            if (kk < lo || kk >= hi) s[kk] = __float_as_uint(-INFINITY);
        }
#if KVQ_MAX_TREE
        // 3-input max tree (depth 5: 128 -> 43 -> 15 -> 5 -> 2 -> 1), every level independent
        float t43[43];
#pragma unroll
        for (int i = 0; i < 42; ++i)
          t43[i] = fmax3(__uint_as_float(s[3 * i]), __uint_as_float(s[3 * i + 1]), __uint_as_float(s[3 * i + 2]));
        t43[42] = fmaxf(__uint_as_float(s[126]), __uint_as_float(s[127]));
        float t15[15];
#pragma unroll
        for (int i = 0; i < 14; ++i) t15[i] = fmax3(t43[3 * i], t43[3 * i + 1], t43[3 * i + 2]);
        t15[14] = t43[42];
        const float t5_0 = fmax3(t15[0], t15[1], t15[2]), t5_1 = fmax3(t15[3], t15[4], t15[5]),
                    t5_2 = fmax3(t15[6], t15[7], t15[8]), t5_3 = fmax3(t15[9], t15[10], t15[11]),
                    t5_4 = fmax3(t15[12], t15[13], t15[14]);
        const float mx = fmaxf(fmax3(t5_0, t5_1, t5_2), fmaxf(t5_3, t5_4));
#else
        // four independent 3-input max chains
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int kk = 0; kk < 128; kk += 8) {
          mx0 = fmax3(mx0, __uint_as_float(s[kk]), __uint_as_float(s[kk + 1]));
          mx1 = fmax3(mx1, __uint_as_float(s[kk + 2]), __uint_as_float(s[kk + 3]));
          mx2 = fmax3(mx2, __uint_as_float(s[kk + 4]), __uint_as_float(s[kk + 5]));
          mx3 = fmax3(mx3, __uint_as_float(s[kk + 6]), __uint_as_float(s[kk + 7]));
        }
        const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
#endif
#ifdef KVQ_EXPERIMENT_NO_MAX  // timing experiments only (wrong results)
        const float m_new = j > 0 ? m_run : mx * cs;
#else
        // Lazy max (FA4-style): the reference point moves only when the tile max exceeds it by more
        // than kLazyLog2 (P <= 2^kLazyLog2, far inside fp16); otherwise O needs no rescale.  The row
        // sum l is taken from the fp16-ROUNDED P (the weights the PV MMA actually uses), so the
        // normalisation stays exactly consistent for peaked rows.
        const float m_tile = SMOOTH ? mx : mx * cs;
        const float m_new = (j == 0 || m_tile > m_run + kLazyLog2) ? fmaxf(m_run, m_tile) : m_run;
#endif
        const float alpha = ex2_approx(m_run - m_new);
        KVQ_TRACE_SM(g, 13);
        // p = 2^(s * cs - m) with packed fp32x2 FFMA; l sums the fp16-rounded p (two packed chains)
        const float cse = SMOOTH ? 1.0f : cs;  // SMOOTH: s already holds the scaled, restored score
        const uint64_t cs2 = f32x2_pack(cse, cse), mneg2 = f32x2_pack(-m_new, -m_new);
        uint64_t acc0 = 0, acc1 = 0;
        float la[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int kk = 0; kk < 64; ++kk) {
          const uint64_t x2 = ffma2(f32x2_pack(__uint_as_float(s[2 * kk]), __uint_as_float(s[2 * kk + 1])), cs2, mneg2);
          float x0, x1, p0, p1;
          f32x2_unpack(x2, x0, x1);
          if ((kk & 7) < kPolyPairs) {  // a fixed share of the exponentials on the FMA pipe
            exp2_poly_pair(x0, x1, p0, p1);
          } else {
            p0 = ex2_approx(x0);
            p1 = ex2_approx(x1);
          }
          const uint32_t pk = MMA_BF16 ? pack_bf162(p0, p1) : pack_half2(p0, p1);
          s[kk] = pk;
          if (kEarlySttm && kk == 31) KVQ_TMEM_ST32(kRotate ? tSb : tS, s);  // keys 0-63 final: store now
#if defined(KVQ_SUM_UNROUNDED)
          if (kk & 1) acc1 = fadd2(acc1, f32x2_pack(p0, p1));
          else acc0 = fadd2(acc0, f32x2_pack(p0, p1));
#elif !defined(KVQ_EXPERIMENT_NO_SUM)
          // mixed-precision adds (FHADD: fp32 += fp16 lane) of the rounded P, four chains
          if (MMA_BF16) {  // bf16 -> fp32 is exact bit placement (no native fp32 += bf16): FADD2 of the pair
            const uint64_t r2 = f32x2_pack(__uint_as_float(pk << 16), __uint_as_float(pk & 0xFFFF0000u));
            if (kk & 1) acc1 = fadd2(acc1, r2);
            else acc0 = fadd2(acc0, r2);
          } else {
            asm("{ .reg .b16 l, h;\n mov.b32 {l, h}, %4;\n add.rn.f32.f16 %0, l, %0;\n add.rn.f32.f16 %1, h, %1;\n}"
                : "+f"(la[(kk & 1) * 2]), "+f"(la[(kk & 1) * 2 + 1]) : "f"(0.0f), "f"(0.0f), "r"(pk));
          }
#endif
        }
        float a0, a1, b0, b1;
        f32x2_unpack(acc0, a0, a1);
        f32x2_unpack(acc1, b0, b1);
        l_run = l_run * alpha + ((a0 + a1) + (b0 + b1)) + ((la[0] + la[1]) + (la[2] + la[3]));
        KVQ_TRACE_SM(g, 14);
        if (!kEarlySttm) KVQ_TMEM_ST32(kRotate ? tSb : tS, s);
        KVQ_TMEM_ST32((kRotate ? tSb : tS) + 32, (s + 32));
        // O_i is kept in units of the current chunk's g_V: rescale by alpha * g_V,prev / g_V,new.
        // Without kRotate PV_i(j-1) is complete here (issued before QK_i(j), whose commit we waited on);
        // with it, the rescale waits for PV_i(j-1)'s own commit (`ofree`).
#ifdef KVQ_EXPERIMENT_NO_RESCALE
        if (false) {
#else
        if (j > 0) {
#endif
          // (gv is the tile's slot scale, uniform: the IEEE division only runs on a chunk change)
          const float f = gv == gv_run ? alpha : alpha * (gv_run / gv);
          if (!__all_sync(0xffffffffu, f == 1.0f)) {
            if (kRotate) {  // this tile's QK no longer orders PV_i(j-1) before us: wait for it
              mbar_wait(ofree + qi, (g - 1) & 1);
              tc_fence_after();
            }
            const uint64_t f2 = f32x2_pack(f, f);
#pragma unroll
            for (int cc = 0; cc < D / 32; ++cc) {  // one 32-column chunk per TMEM round trip
              uint32_t* o = s + 64;
              KVQ_TMEM_LD32(tO + 32 * cc, o);
              tmem_ld_wait();
#pragma unroll
              for (int kk = 0; kk < 32; kk += 2) {
                float x0, x1;
                f32x2_unpack(fmul2(f32x2_pack(__uint_as_float(o[kk]), __uint_as_float(o[kk + 1])), f2), x0, x1);
                o[kk] = __float_as_uint(x0);
                o[kk + 1] = __float_as_uint(x1);
              }
              KVQ_TMEM_ST32(tO + 32 * cc, o);
            }
          }
        }
        gv_run = gv;
        m_run = m_new;
        tmem_st_wait();
        KVQ_TRACE_SM(g, 15);
        tc_fence_before();
        mbar_arrive(pfull + qi);
        KVQ_TRACE(g, 3 * qi + 2);
      }
      // ---- piece epilogue
      // Score range (reading Z25): the scores come out of an fp32 accumulation whose absolute error
      // grows with their magnitude (~|score| 2^-24 sqrt(d)), while softmax weights depend on score
      // DIFFERENCES; a row whose running max reaches 2^12 log2 units in magnitude (or is non-finite)
      // is KVQ_ERANGE, index = the query row's first element, and its O is undefined.  (m_run is
      // within kLazyLog2 of the row's true max, so checking it once per piece sees every such row.)
      if (!(fabsf(m_run) < kScoreRangeLog2) && !range_reported && t < p.Tq)
        report_status(p.status, -7 /* KVQ_ERANGE */, (unsigned long long)(((int64_t)t * H + h) * D));
      mbar_wait(ofull + qi, k & 1);
      tc_fence_after();
      const float f = pc.full ? gv_run / l_run : gv_run;
      float* wsO = p.ws + (size_t)pc.slot * p.ws_slot_floats + (size_t)(128 * qi + row) * D;
      if (!pc.full && t < p.Tq) {
        float* wml = p.ws + (size_t)pc.slot * p.ws_slot_floats + 256 * D;
        wml[128 * qi + row] = m_run;
        wml[256 + 128 * qi + row] = l_run;
      }
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        KVQ_TMEM_LD32(tO + 32 * cc, o);
        tmem_ld_wait();
        if (t < p.Tq) {
          if (!pc.full) {
            float4* dst = reinterpret_cast<float4*>(wsO + 32 * cc);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              dst[kk] = make_float4(__uint_as_float(o[4 * kk]) * f, __uint_as_float(o[4 * kk + 1]) * f,
                                    __uint_as_float(o[4 * kk + 2]) * f, __uint_as_float(o[4 * kk + 3]) * f);
          } else {
            const int64_t base = ((int64_t)t * H + h) * D + 32 * cc;
            if (p.out_dtype == DT_FP32) {
              float4* dst = reinterpret_cast<float4*>((float*)p.O + base);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                dst[kk] = make_float4(__uint_as_float(o[4 * kk]) * f, __uint_as_float(o[4 * kk + 1]) * f,
                                      __uint_as_float(o[4 * kk + 2]) * f, __uint_as_float(o[4 * kk + 3]) * f);
            } else {
              uint4* dst = reinterpret_cast<uint4*>((__nv_bfloat16*)p.O + base);
              if (p.o_peer[0] != nullptr) {  // f4 direct: straight into the owning rank's O shard
                const int r = t / p.o_Ts;
                dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o_peer[r]) +
                                               ((int64_t)(t - r * p.o_Ts) * p.o_H + p.o_h0 + h) * D + 32 * cc);
              }
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                dst[kk] = make_uint4(pack_bf162(__uint_as_float(o[8 * kk]) * f, __uint_as_float(o[8 * kk + 1]) * f),
                                     pack_bf162(__uint_as_float(o[8 * kk + 2]) * f, __uint_as_float(o[8 * kk + 3]) * f),
                                     pack_bf162(__uint_as_float(o[8 * kk + 4]) * f, __uint_as_float(o[8 * kk + 5]) * f),
                                     pack_bf162(__uint_as_float(o[8 * kk + 6]) * f, __uint_as_float(o[8 * kk + 7]) * f));
            }
          }
        }
      }
    }
   }
  } else if (warp < 12) {
    // ================================================================ dequant WG
    reg_dealloc<APPEND ? kRegDequantAp : kRegDequant>();
    const int r = tid - 256;  // key row within the tile
    int g = 0;
    bool ap_ready = false;  // APPEND: every CTA's share of the appended slot is in place
    Piece pc;
    for (int k = 0; next_piece(k, pc); ++k) {
      const int h = pc.unit / p.qpairs;
      TileIter it;
      tile_seek(p, pc.tb, it);
      for (int j = pc.tb; j < pc.te; ++j, ++g, tile_next(p, it)) {
        const AttnSeg& sg = p.seg[it.seg];
        const int b = SM::buf(g);
        const uint32_t par = SM::empty_par(g);
#ifdef KVQ_EXPERIMENT_NO_DEQUANT  // timing experiments only (wrong results): K^/V^ tiles never written
        if (NVFP4) {
          if (g >= SM::kNBuf) mbar_wait(kempty + b, par);
          mbar_arrive(kfull + b);
          if (g >= SM::kNBuf) mbar_wait(vempty + b, par);
          mbar_arrive(vfull + b);
        } else
#endif
        if (NVFP4) {
          const int64_t crow = (int64_t)h * p.head_stride_rows + (int64_t)sg.slot * p.T_pad + it.t0 + r;
          PackedRow<D> pk, pv;
          if (APPEND && sg.slot == p.ap_slot) {  // the chunk being appended by this launch
            if (!ap_ready) {
              unsigned long long t0 = 0, t1;
              if (r == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
              ap_wait_all_done(p.ap_sync, G, launch_epoch(), r, 128);
              named_bar_sync(5, 128);
              if (r == 0 && p.trace != nullptr) {  // debug: per-CTA (start of the wait, its length) in ns
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                p.trace[1024 + 2 * c] = t0;
                p.trace[1024 + 2 * c + 1] = t1 - t0;
              }
              ap_ready = true;
            }
            load_packed_row<D, true>(pk, p.codes_k + crow * (D / 2), p.scales_k + crow * (D / 16));
            load_packed_row<D, true>(pv, p.codes_v + crow * (D / 2), p.scales_v + crow * (D / 16));
          } else {
            load_packed_row<D>(pk, p.codes_k + crow * (D / 2), p.scales_k + crow * (D / 16));
            load_packed_row<D>(pv, p.codes_v + crow * (D / 2), p.scales_v + crow * (D / 16));
          }
          if (g >= SM::kNBuf) mbar_wait(kempty + b, par);
          store_dequant_row<D>(SK(b), r, pk);
          fence_proxy_async_smem();
          mbar_arrive(kfull + b);
          if (r == 0) KVQ_TRACE(g, 6);
          if (g >= SM::kNBuf) mbar_wait(vempty + b, par);
          store_dequant_row<D>(SV(b), r, pv);
          fence_proxy_async_smem();
          mbar_arrive(vfull + b);
          if (r == 0) KVQ_TRACE(g, 7);
        } else if (r == 0) {
          // bf16-KV mode: one thread (warp 8) lands each 128-key K tile with TMA, another (warp 9)
          // each V tile, so neither stream waits on the other's buffer (D/64 panels of 128 rows x
          // 128 B, 128B-swizzled = the K-major SW128 layout; keys past n_keys are zeros)
          constexpr uint32_t kBytes = 128u * D * 2u;
          if (g >= SM::kNBuf) mbar_wait(kempty + b, par);
          mbar_arrive_expect_tx(kfull + b, kBytes);
#pragma unroll
          for (int pn = 0; pn < D / 64; ++pn) tma_load_3d(SK(b) + 16384u * pn, &p.tmap_k, 64 * pn, h, it.t0, kfull + b);
        } else if (r == 32) {
          constexpr uint32_t kBytes = 128u * D * 2u;
          if (g >= SM::kNBuf) mbar_wait(vempty + b, par);
          mbar_arrive_expect_tx(vfull + b, kBytes);
#pragma unroll
          for (int pn = 0; pn < D / 64; ++pn) tma_load_3d(SV(b) + 16384u * pn, &p.tmap_v, 64 * pn, h, it.t0, vfull + b);
        }
      }
    }
  } else {
    reg_dealloc<APPEND ? kRegMmaAp : kRegMma>();
  }
  if (warp == 12) {
    // ================================================================ MMA issuer warp
    // The whole warp runs this loop converged (descriptors stay in uniform registers); one elected
    // lane issues each unrolled group of tcgen05.mma and its commits.  Descriptor bases are
    // precomputed; the k-step offsets are compile-time adds to the start-address field.
    constexpr uint32_t kIdS = umma_idesc_f16(128, 128, MMA_BF16 ? 1 : 0, 0, 0);
    constexpr uint32_t kIdS64 = umma_idesc_f16(128, 64, MMA_BF16 ? 1 : 0, 0, 0);
    constexpr uint32_t kIdO = umma_idesc_f16(128, D, MMA_BF16 ? 1 : 0, 0, 1);
    const uint64_t dQ0 = umma_desc_sw128(SQ(0), 16, 1024), dQ1 = umma_desc_sw128(SQ(1), 16, 1024);
    const uint64_t dL0 = umma_desc_sw128(SQL(0), 16, 1024), dL1 = umma_desc_sw128(SQL(1), 16, 1024);
    const uint64_t dK0 = umma_desc_sw128(SK(0), 16, 1024), dK1 = umma_desc_sw128(SK(1), 16, 1024);
    const uint64_t dV0 = umma_desc_sw128(SV(0), 16384, 1024), dV1 = umma_desc_sw128(SV(1), 16384, 1024);
    auto issue_qk = [&](int qi, int b) {
      const uint64_t da = qi ? dQ1 : dQ0, db = b ? dK1 : dK0;
      const uint32_t dt = tmem + 128u * qi;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          umma_ss(dt, da + off, db + off, kIdS, kk > 0 ? 1u : 0u);
        }
        if (QSPLIT) {  // + Q_lo K^T into the same accumulator
          const uint64_t dl = qi ? dL1 : dL0;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
            umma_ss(dt, dl + off, db + off, kIdS, 1u);
          }
        }
      }
      __syncwarp();
    };
    // kRotate: keys [64 half, 64 half + 64) of the K tile into the 64-column TMEM region `reg`
    auto issue_qk_half = [&](int qi, int b, int half, uint32_t reg) {
      const uint64_t da = qi ? dQ1 : dQ0, db = (b ? dK1 : dK0) + (uint64_t)((8192 * half) >> 4);
      const uint32_t dt = tmem + 64u * reg;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          umma_ss(dt, da + off, db + off, kIdS64, kk > 0 ? 1u : 0u);
        }
        if (QSPLIT) {
          const uint64_t dl = qi ? dL1 : dL0;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
            umma_ss(dt, dl + off, db + off, kIdS64, 1u);
          }
        }
      }
      __syncwarp();
    };
    // P_i at TMEM column pcol (kRotate: its region b; else S_i's first 64 columns)
    auto issue_pv = [&](int qi, int b, bool first, uint32_t pcol) {
      const uint64_t db = b ? dV1 : dV0;
      const uint32_t dt = tmem + 256u + 128u * qi, ta = tmem + pcol;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(dt, ta + 8 * kk, db + (uint64_t)((kk * 2048) >> 4), kIdO, (!first || kk > 0) ? 1u : 0u);
      }
      __syncwarp();
    };
    auto tc_commit = [&](uint64_t* bar) {
      if (elect_one()) kvq::tc_commit(bar);
      __syncwarp();
    };
    auto qk_rot = [&](int qi, int b, int kq) {  // the kq-th QK of the piece (tile qi) into its regions
      uint32_t ra, rb;
      sp_regions(kq, ra, rb);
      issue_qk_half(qi, b, 0, ra);
      issue_qk_half(qi, b, 1, rb);
    };
    auto p_col = [&](int kq) -> uint32_t {
      uint32_t ra, rb;
      sp_regions(kq, ra, rb);
      return 64u * rb;
    };
    int g = 0;
    Piece pc;
    for (int k = 0; next_piece(k, pc); ++k) {
      const int np = pc.te - pc.tb;
      mbar_wait(qfull + 0, k & 1);
      mbar_wait(qfull + 1, k & 1);
      mbar_wait(kfull + SM::buf(g), SM::full_par(g));
      tc_fence_after();
      if (kRotate) qk_rot(0, SM::buf(g), 0);
      else issue_qk(0, SM::buf(g));
      tc_commit(sfull + 0);
      if (kRotate) qk_rot(1, SM::buf(g), 1);
      else issue_qk(1, SM::buf(g));
      tc_commit(sfull + 1);
      tc_commit(kempty + SM::buf(g));
      for (int j = 0; j < np; ++j) {
        const int gj = g + j, b = SM::buf(gj), bn = SM::buf(gj + 1);
        const bool more = j + 1 < np;
        if (kRotate) {
          // Four issues per tile pair, each as soon as its inputs are ready (polled: the whole warp reads
          // lane 0's non-blocking barrier tests), in two rounds so that every QK follows the PV whose P
          // region it reuses:
          //   [A] QK_0(j+1): region a = R0 held S_1(j) (j >= 1; j = 0: S_0(0), and S_1(0)'s R2 is its b) ->
          //       needs softmax_1 to have loaded S_1(j); region b = P_1(j-1)'s (PV_1(j-1) issued last round)
          //   [B] PV_0(j): needs P_0(j) and V(j)
          //   [C] QK_1(j+1): a = R0 held S_0(j+1) -> needs softmax_0 to have loaded it; b = P_0(j)'s ([B])
          //   [D] PV_1(j): needs P_1(j)
          auto ready = [&](bool c) { return __shfl_sync(0xffffffffu, c ? 1 : 0, 0) != 0; };
          bool doneA = !more, doneB = false;
          while (!(doneA && doneB)) {
            if (!doneA && ready(mbar_test(kfull + bn, SM::full_par(gj + 1)) &&
                                (j != 0 || mbar_test(sfree + 0, gj & 1)) && mbar_test(sfree + 1, gj & 1))) {
              tc_fence_after();
              KVQ_TRACE(gj + 1, 9);
              qk_rot(0, bn, 2 * j + 2);
              tc_commit(sfull + 0);
              doneA = true;
            }
            if (!doneB && ready(mbar_test(vfull + b, SM::full_par(gj)) && mbar_test(pfull + 0, gj & 1))) {
              tc_fence_after();
              KVQ_TRACE(gj, 8);
              issue_pv(0, b, j == 0, p_col(2 * j));
              tc_commit(ofree + 0);
              if (!more) tc_commit(ofull + 0);
              doneB = true;
            }
          }
          bool doneC = !more, doneD = false;
          while (!(doneC && doneD)) {
            if (!doneC && ready(mbar_test(sfree + 0, (gj + 1) & 1))) {
              tc_fence_after();
              qk_rot(1, bn, 2 * j + 3);
              KVQ_TRACE(gj + 1, 11);
              tc_commit(sfull + 1);
              tc_commit(kempty + bn);
              doneC = true;
            }
            if (!doneD && ready(mbar_test(pfull + 1, gj & 1))) {
              tc_fence_after();
              KVQ_TRACE(gj, 10);
              issue_pv(1, b, j == 0, p_col(2 * j + 1));
              tc_commit(vempty + b);
              tc_commit(ofree + 1);
              if (!more) tc_commit(ofull + 1);
              doneD = true;
            }
          }
          continue;
        }
        mbar_wait(vfull + b, SM::full_par(gj));
        mbar_wait(pfull + 0, gj & 1);
        tc_fence_after();
        KVQ_TRACE(gj, 8);
        issue_pv(0, b, j == 0, 0u);
        if (more) {
          mbar_wait(kfull + bn, SM::full_par(gj + 1));
          tc_fence_after();
          KVQ_TRACE(gj + 1, 9);
          issue_qk(0, bn);
          tc_commit(sfull + 0);
        } else {
          tc_commit(ofull + 0);
        }
        mbar_wait(pfull + 1, gj & 1);
        tc_fence_after();
        KVQ_TRACE(gj, 10);
        issue_pv(1, b, j == 0, 128u);
        tc_commit(vempty + b);
        if (more) {
          issue_qk(1, bn);
          KVQ_TRACE(gj + 1, 11);
          tc_commit(sfull + 1);
          tc_commit(kempty + bn);
        } else {
          tc_commit(ofull + 1);
        }
      }
      g += np;
    }
  }
  if (APPEND && warp >= 13) {  // the MMA warpgroup's three spare warps quantize this CTA's share
    const unsigned long long E = launch_epoch();
    if (p.ap_dtype == DT_BF16) fused_append_role<D, DT_BF16>(p, smem + SM::kAp, tid - 13 * 32, E);
    else fused_append_role<D, DT_FP32>(p, smem + SM::kAp, tid - 13 * 32, E);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 12) tmem_dealloc(tmem, 512);
#undef SQ
#undef SK
#undef SV
#undef SQL
}

// ---------------------------------------------------------------------------------------------
// v2 (d = 128, NVFP4 cache, bf16 queries, plain mode): 64-key tiles so that each query tile's P has
// TMEM columns of its own -- S_i [64 i, +64), P_i [128 + 32 i, +32), O_i [256 + 128 i, +128) -- and
// QK_i(j+1) is issued as soon as softmax_i(j) has loaded S_i(j) into registers (the `sfree` barrier),
// overlapping the next scores with this tile's softmax.  The tensor core then runs
// QK0(j) QK1(j) PV0(j-1) PV1(j-1) ...; softmax_i(j) waits for PV_i(j-1) (`pempty`) only before it
// writes P_i(j) and rescales O_i.  Dequant: 64 threads per tensor (one key row each).
constexpr int kV2Keys = 64;
struct V2Smem {
  static constexpr int kQ = 128 * 128 * 2;   // one 128-query tile (bytes)
  static constexpr int kKV = 64 * 128 * 2;   // one 64-key tile
  static constexpr int kQ0 = 0, kQ1 = kQ;
  static constexpr int kK0 = 2 * kQ, kK1 = kK0 + kKV, kV0 = kK1 + kKV, kV1 = kV0 + kKV;
  static constexpr int kBar = kV1 + kKV;
  static constexpr int kBytes = kBar + 24 * 8 + 16 + 1024;
};

KVQ_DEV uint32_t chunk_addr64(uint32_t base, int r, int c) {  // 64-row K-major SW128 tile
  return base + (uint32_t)(c >> 3) * 8192u + sw128_off(r, c & 7);
}

template <int D>
KVQ_DEV void store_dequant_row64(uint32_t base, int r, const PackedRow<D>& pr) {
#pragma unroll
  for (int j = 0; j < D / 16; ++j) {
    const uint32_t sb = (pr.s[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    const uint32_t s2 = f16x2_from_e4m3x2(sb | (sb << 8));
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int wi = 2 * j + half;
      const uint4 q = pr.c[wi >> 2];
      const uint32_t w = (wi & 3) == 0 ? q.x : (wi & 3) == 1 ? q.y : (wi & 3) == 2 ? q.z : q.w;
      uint32_t o[4];
      dequant_word_f16(w, s2, o);
      st_shared_v4(chunk_addr64(base, r, wi), o[0], o[1], o[2], o[3]);
    }
  }
}

KVQ_DEV int count_tiles64(const AttnParams& p) {
  int n = 0;
  for (int s = 0; s < p.nseg; ++s) n += ((p.seg[s].end + 63) >> 6) - (p.seg[s].begin >> 6);
  return n;
}
KVQ_DEV void tile_seek64(const AttnParams& p, int tb, TileIter& it) {
  int s = 0;
  for (; s < p.nseg; ++s) {
    const int nt = ((p.seg[s].end + 63) >> 6) - (p.seg[s].begin >> 6);
    if (tb < nt) break;
    tb -= nt;
  }
  it.seg = s;
  it.t0 = (p.seg[s].begin & ~63) + 64 * tb;
}
KVQ_DEV void tile_next64(const AttnParams& p, TileIter& it) {
  it.t0 += 64;
  if (it.t0 < p.seg[it.seg].end) return;
  if (++it.seg >= p.nseg) return;
  it.t0 = p.seg[it.seg].begin & ~63;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_v2_kernel(const __grid_constant__ AttnParams p) {
  static_assert(D == 128, "v2: d = 128");
  using SM = V2Smem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
#define V2Q(i) (sbase + SM::kQ0 + (uint32_t)(i) * SM::kQ)
#define V2K(b) (sbase + SM::kK0 + (uint32_t)(b) * SM::kKV)
#define V2V(b) (sbase + SM::kV0 + (uint32_t)(b) * SM::kKV)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
  uint64_t* kfull = bars + 0;    // [2] dequant -> MMA (64 arrivals)
  uint64_t* vfull = bars + 2;    // [2]
  uint64_t* kempty = bars + 4;   // [2] MMA -> dequant
  uint64_t* vempty = bars + 6;   // [2]
  uint64_t* sfull = bars + 8;    // [2] MMA -> softmax i: S_i(j) ready
  uint64_t* sfree = bars + 10;   // [2] softmax i -> MMA: S_i(j) loaded, its columns may be overwritten
  uint64_t* pfull = bars + 12;   // [2] softmax i -> MMA: P_i(j) written, O_i rescaled
  uint64_t* pempty = bars + 14;  // [2] MMA -> softmax i: PV_i(j) done (P_i free, O_i stable)
  uint64_t* ofull = bars + 16;   // [2] MMA -> softmax i: last PV_i of a piece done
  uint64_t* qfull = bars + 18;   // [2] softmax i -> MMA: Q_i of a piece loaded
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 20);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int H = p.H;
  const int n = count_tiles64(p);
  const int G = gridDim.x, c = blockIdx.x;
  const Sched sch = make_sched(p, n, G);

  if (warp == 12) tmem_alloc(tslot, 512);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(kfull + b, 64);
      mbar_init(vfull + b, 64);
      mbar_init(kempty + b, 1);
      mbar_init(vempty + b, 1);
      mbar_init(sfull + b, 1);
      mbar_init(sfree + b, 128);
      mbar_init(pfull + b, 128);
      mbar_init(pempty + b, 1);
      mbar_init(ofull + b, 1);
      mbar_init(qfull + b, 128);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp < 8) {
    // ================================================================ softmax WG (query tile qi)
    reg_alloc<kRegSoftmax>();
    const int qi = warp >> 2;
    const int row = tid & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + 64 * qi + lane_off;
    const uint32_t tP = tmem + 128 + 32 * qi + lane_off;
    const uint32_t tO = tmem + 256 + 128 * qi + lane_off;
    const float sl2 = p.scale_log2;
    int g = 0;   // tiles processed (barrier parity)
    int kk = 0;  // pieces processed
    Piece pc;
    for (int k = 0; get_piece(sch, c, k, pc); ++k, ++kk) {
      const int h = pc.unit / p.qpairs, q0 = (pc.unit - h * p.qpairs) * 256;
      const int t = q0 + 128 * qi + row;
      const float sl2q = sl2 * load_q_row<D, false, false, false>(V2Q(qi), V2Q(qi), row, p.Q, p.q_dtype,
                                                                   (int64_t)t * H + h, t < p.Tq, p.status).qscale;
      fence_proxy_async_smem();
      mbar_arrive(qfull + qi);
      float m_run = -INFINITY, l_run = 0.0f, gv_run = 1.0f;
      TileIter it;
      tile_seek64(p, pc.tb, it);
      for (int j = 0; j < pc.te - pc.tb; ++j, ++g, tile_next64(p, it)) {
        const AttnSeg& sg = p.seg[it.seg];
        const int lo = max(sg.begin - it.t0, 0), hi = min(sg.end - it.t0, kV2Keys);
        const float gk = __ldg(p.g + 2 * sg.slot), gv = __ldg(p.g + 2 * sg.slot + 1);
        const float cs = gk * sl2q;
        mbar_wait(sfull + qi, g & 1);
        tc_fence_after();
        uint32_t s[64];
        KVQ_TMEM_LD32(tS, s);
        KVQ_TMEM_LD32(tS + 32, (s + 32));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(sfree + qi);  // QK_i(j+1) may now overwrite S_i
        if (lo != 0 || hi != kV2Keys) {
#pragma unroll
          for (int q = 0; q < 64; ++q)
            if (q < lo || q >= hi) s[q] = __float_as_uint(-INFINITY);
        }
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int q = 0; q < 64; q += 8) {
          mx0 = fmax3(mx0, __uint_as_float(s[q]), __uint_as_float(s[q + 1]));
          mx1 = fmax3(mx1, __uint_as_float(s[q + 2]), __uint_as_float(s[q + 3]));
          mx2 = fmax3(mx2, __uint_as_float(s[q + 4]), __uint_as_float(s[q + 5]));
          mx3 = fmax3(mx3, __uint_as_float(s[q + 6]), __uint_as_float(s[q + 7]));
        }
        const float m_tile = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * cs;
        const float m_new = (j == 0 || m_tile > m_run + kLazyLog2) ? fmaxf(m_run, m_tile) : m_run;
        const float alpha = ex2_approx(m_run - m_new);
        const uint64_t cs2 = f32x2_pack(cs, cs), mneg2 = f32x2_pack(-m_new, -m_new);
        float la[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint64_t x2 = ffma2(f32x2_pack(__uint_as_float(s[2 * q]), __uint_as_float(s[2 * q + 1])), cs2, mneg2);
          float x0, x1, p0, p1;
          f32x2_unpack(x2, x0, x1);
          if ((q & 7) < kPolyPairs) {
            exp2_poly_pair(x0, x1, p0, p1);
          } else {
            p0 = ex2_approx(x0);
            p1 = ex2_approx(x1);
          }
          const uint32_t pk = pack_half2(p0, p1);
          s[q] = pk;
          asm("{ .reg .b16 l, h;\n mov.b32 {l, h}, %4;\n add.rn.f32.f16 %0, l, %0;\n add.rn.f32.f16 %1, h, %1;\n}"
              : "+f"(la[(q & 1) * 2]), "+f"(la[(q & 1) * 2 + 1]) : "f"(0.0f), "f"(0.0f), "r"(pk));
        }
        l_run = l_run * alpha + ((la[0] + la[1]) + (la[2] + la[3]));
        // PV_i(j-1) done: P_i free, O_i stable (the first tile of a piece waits for the previous piece's)
        if (g > 0) mbar_wait(pempty + qi, (g - 1) & 1);
        tc_fence_after();
        KVQ_TMEM_ST32(tP, s);
        if (j > 0) {
          const float f = alpha * (gv_run / gv);
          if (!__all_sync(0xffffffffu, f == 1.0f)) {
            const uint64_t f2 = f32x2_pack(f, f);
            uint32_t o[64];
#pragma unroll
            for (int cc = 0; cc < D / 32; cc += 2) {
              KVQ_TMEM_LD32(tO + 32 * cc, o);
              KVQ_TMEM_LD32(tO + 32 * (cc + 1), (o + 32));
              tmem_ld_wait();
#pragma unroll
              for (int q = 0; q < 64; q += 2) {
                float x0, x1;
                f32x2_unpack(fmul2(f32x2_pack(__uint_as_float(o[q]), __uint_as_float(o[q + 1])), f2), x0, x1);
                o[q] = __float_as_uint(x0);
                o[q + 1] = __float_as_uint(x1);
              }
              KVQ_TMEM_ST32(tO + 32 * cc, o);
              KVQ_TMEM_ST32(tO + 32 * (cc + 1), (o + 32));
            }
          }
        }
        gv_run = gv;
        m_run = m_new;
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(pfull + qi);
      }
      // ---- piece epilogue
      mbar_wait(ofull + qi, kk & 1);
      tc_fence_after();
      const float f = pc.full ? gv_run / l_run : gv_run;
      float* wsO = p.ws + (size_t)pc.slot * p.ws_slot_floats + (size_t)(128 * qi + row) * D;
      if (!pc.full && t < p.Tq) {
        float* wml = p.ws + (size_t)pc.slot * p.ws_slot_floats + 256 * D;
        wml[128 * qi + row] = m_run;
        wml[256 + 128 * qi + row] = l_run;
      }
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        KVQ_TMEM_LD32(tO + 32 * cc, o);
        tmem_ld_wait();
        if (t < p.Tq) {
          if (!pc.full) {
            float4* dst = reinterpret_cast<float4*>(wsO + 32 * cc);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              dst[q] = make_float4(__uint_as_float(o[4 * q]) * f, __uint_as_float(o[4 * q + 1]) * f,
                                   __uint_as_float(o[4 * q + 2]) * f, __uint_as_float(o[4 * q + 3]) * f);
          } else {
            const int64_t base = ((int64_t)t * H + h) * D + 32 * cc;
            if (p.out_dtype == DT_FP32) {
              float4* dst = reinterpret_cast<float4*>((float*)p.O + base);
#pragma unroll
              for (int q = 0; q < 8; ++q)
                dst[q] = make_float4(__uint_as_float(o[4 * q]) * f, __uint_as_float(o[4 * q + 1]) * f,
                                     __uint_as_float(o[4 * q + 2]) * f, __uint_as_float(o[4 * q + 3]) * f);
            } else {
              uint4* dst = reinterpret_cast<uint4*>((__nv_bfloat16*)p.O + base);
#pragma unroll
              for (int q = 0; q < 4; ++q)
                dst[q] = make_uint4(pack_bf162(__uint_as_float(o[8 * q]) * f, __uint_as_float(o[8 * q + 1]) * f),
                                    pack_bf162(__uint_as_float(o[8 * q + 2]) * f, __uint_as_float(o[8 * q + 3]) * f),
                                    pack_bf162(__uint_as_float(o[8 * q + 4]) * f, __uint_as_float(o[8 * q + 5]) * f),
                                    pack_bf162(__uint_as_float(o[8 * q + 6]) * f, __uint_as_float(o[8 * q + 7]) * f));
            }
          }
        }
      }
    }
  } else if (warp < 12) {
    // ================================================================ dequant WG: 64 K rows + 64 V rows
    reg_dealloc<kRegDequant>();
    const int r = (tid - 256) & 63;
    const bool is_v = tid - 256 >= 64;
    uint64_t* full = is_v ? vfull : kfull;
    uint64_t* empty = is_v ? vempty : kempty;
    const uint8_t* codes = is_v ? p.codes_v : p.codes_k;
    const uint8_t* scales = is_v ? p.scales_v : p.scales_k;
    int g = 0;
    Piece pc;
    for (int k = 0; get_piece(sch, c, k, pc); ++k) {
      const int h = pc.unit / p.qpairs;
      TileIter it;
      tile_seek64(p, pc.tb, it);
      for (int j = pc.tb; j < pc.te; ++j, ++g, tile_next64(p, it)) {
        const AttnSeg& sg = p.seg[it.seg];
        const int b = g & 1;
        const int64_t crow = (int64_t)h * p.head_stride_rows + (int64_t)sg.slot * p.T_pad + it.t0 + r;
        PackedRow<D> pr;
        load_packed_row<D>(pr, codes + crow * (D / 2), scales + crow * (D / 16));
        if (g >= 2) mbar_wait(empty + b, ((g >> 1) - 1) & 1);
        store_dequant_row64<D>(is_v ? V2V(b) : V2K(b), r, pr);
        fence_proxy_async_smem();
        mbar_arrive(full + b);
      }
    }
  } else {
    reg_dealloc<kRegMma>();
  }
  if (warp == 12) {
    // ================================================================ MMA issuer warp
    constexpr uint32_t kIdS = umma_idesc_f16(128, kV2Keys, 0, 0, 0);
    constexpr uint32_t kIdO = umma_idesc_f16(128, D, 0, 0, 1);
    const uint64_t dQ0 = umma_desc_sw128(V2Q(0), 16, 1024), dQ1 = umma_desc_sw128(V2Q(1), 16, 1024);
    const uint64_t dK0 = umma_desc_sw128(V2K(0), 16, 1024), dK1 = umma_desc_sw128(V2K(1), 16, 1024);
    const uint64_t dV0 = umma_desc_sw128(V2V(0), 8192, 1024), dV1 = umma_desc_sw128(V2V(1), 8192, 1024);
    auto issue_qk = [&](int qi, int b) {
      const uint64_t da = qi ? dQ1 : dQ0, db = b ? dK1 : dK0;
      const uint32_t dt = tmem + 64u * qi;
      if (elect_one()) {
#pragma unroll
        for (int q = 0; q < D / 16; ++q)
          umma_ss(dt, da + (uint64_t)(((q >> 2) * 16384 + (q & 3) * 32) >> 4),
                  db + (uint64_t)(((q >> 2) * 8192 + (q & 3) * 32) >> 4), kIdS, q > 0 ? 1u : 0u);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int qi, int b, bool first) {
      const uint64_t db = b ? dV1 : dV0;
      const uint32_t dt = tmem + 256u + 128u * qi, ta = tmem + 128u + 32u * qi;
      if (elect_one()) {
#pragma unroll
        for (int q = 0; q < kV2Keys / 16; ++q)
          umma_ts(dt, ta + 8 * q, db + (uint64_t)((q * 2048) >> 4), kIdO, (!first || q > 0) ? 1u : 0u);
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) kvq::tc_commit(bar);
      __syncwarp();
    };
    auto pv_pair = [&](int t, bool first, bool last) {  // PV of global tile t for both query tiles
      const int bt = t & 1;
      mbar_wait(vfull + bt, (t >> 1) & 1);
      mbar_wait(pfull + 0, t & 1);
      tc_fence_after();
      issue_pv(0, bt, first);
      commit(pempty + 0);
      if (last) commit(ofull + 0);
      mbar_wait(pfull + 1, t & 1);
      tc_fence_after();
      issue_pv(1, bt, first);
      commit(pempty + 1);
      if (last) commit(ofull + 1);
      commit(vempty + bt);
    };
    int g = 0;
    Piece pc;
    for (int k = 0; get_piece(sch, c, k, pc); ++k) {
      const int np = pc.te - pc.tb;
      mbar_wait(qfull + 0, k & 1);
      mbar_wait(qfull + 1, k & 1);
      for (int j = 0; j < np; ++j) {
        const int gj = g + j, b = gj & 1;
        mbar_wait(kfull + b, (gj >> 1) & 1);
        if (gj > 0) mbar_wait(sfree + 0, (gj - 1) & 1);
        tc_fence_after();
        issue_qk(0, b);
        commit(sfull + 0);
        if (gj > 0) mbar_wait(sfree + 1, (gj - 1) & 1);
        tc_fence_after();
        issue_qk(1, b);
        commit(sfull + 1);
        commit(kempty + b);
        if (j > 0) pv_pair(gj - 1, j == 1, false);
      }
      pv_pair(g + np - 1, np == 1, true);
      g += np;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 12) tmem_dealloc(tmem, 512);
#undef V2Q
#undef V2K
#undef V2V
}

// Merge the partial pieces of every split unit: O = sum_p 2^(m_p - m) O_p / sum_p 2^(m_p - m) l_p,
// pieces in increasing CTA order (deterministic).  A unit is split exactly when a CTA range boundary
// falls strictly inside it; CTA b of this kernel handles the boundary of attention CTA b (if it is
// the first boundary inside its unit), so only split units are touched.  Thread = (row, 4 columns).
#ifndef KVQ_COMBINE_SPLIT
#define KVQ_COMBINE_SPLIT 4
#endif
constexpr int kCombineSplit = KVQ_COMBINE_SPLIT;  // CTAs per split unit (row blocks): the merge is per-SM bandwidth bound

template <int D>
__global__ void __launch_bounds__(512) combine_kernel(const __grid_constant__ AttnParams p, int n) {
  const int G = p.grid;
  const Sched sch = make_sched(p, n, G);
  const int b = blockIdx.x + 1;  // boundary between attention CTAs b-1 and b
  const int sb = range_begin(sch, b);
  if (sb % n == 0) return;                                   // boundary on a unit edge: no split
  const int unit = sb / n;
  const int s0 = unit * n, s1 = s0 + n;
  if (range_begin(sch, b - 1) > s0) return;                 // an earlier boundary owns this unit
  const int c0 = b - 1;                                      // CTA holding the unit's first piece
  const bool c0_first = range_begin(sch, c0) == s0;         // ... as its first piece?
  int c1 = b;
  while (c1 + 1 < G && range_begin(sch, c1 + 1) < s1) ++c1;  // last CTA with a piece of the unit
  const int h = unit / p.qpairs, q0 = (unit - h * p.qpairs) * 256;
  constexpr int kTpr = D / 4;  // threads per row
  constexpr int kRows = 256 / kCombineSplit;  // rows of the unit merged by this CTA (blockIdx.y)
  for (int i = threadIdx.x; i < kRows * kTpr; i += blockDim.x) {
    const int rr = blockIdx.y * kRows + i / kTpr, c4 = i % kTpr;
    const int t = q0 + rr;
    if (t >= p.Tq) continue;
    float m = -INFINITY;
    for (int cc = c0; cc <= c1; ++cc) {
      const int slot = (cc == c0 && !c0_first) ? 2 * cc + 1 : 2 * cc;  // first piece = c0's last; others = their first
      m = fmaxf(m, p.ws[(size_t)slot * p.ws_slot_floats + 256 * D + rr]);
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float l = 0.0f;
    for (int cc = c0; cc <= c1; ++cc) {
      const int slot = (cc == c0 && !c0_first) ? 2 * cc + 1 : 2 * cc;
      const float* base = p.ws + (size_t)slot * p.ws_slot_floats;
      const float w = exp2f(base[256 * D + rr] - m);
      l += w * base[256 * D + 256 + rr];
      const float4 o = reinterpret_cast<const float4*>(base + (size_t)rr * D)[c4];
      acc.x += w * o.x; acc.y += w * o.y; acc.z += w * o.z; acc.w += w * o.w;
    }
    const float inv = 1.0f / l;
    const int64_t ob = ((int64_t)t * p.H + h) * D + 4 * c4;
    if (p.out_dtype == DT_FP32) {
      *reinterpret_cast<float4*>((float*)p.O + ob) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    } else {
      __nv_bfloat16* dst = (__nv_bfloat16*)p.O + ob;
      if (p.o_peer[0] != nullptr) {  // f4 direct: straight into the owning rank's O shard
        const int r = t / p.o_Ts;
        dst = reinterpret_cast<__nv_bfloat16*>(p.o_peer[r]) + ((int64_t)(t - r * p.o_Ts) * p.o_H + p.o_h0 + h) * D + 4 * c4;
      }
      *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf162(acc.x * inv, acc.y * inv), pack_bf162(acc.z * inv, acc.w * inv));
    }
  }
}

template <int D, bool NVFP4, bool MMA_BF16, bool SMOOTH = false, bool QSPLIT = false, bool APPEND = false>
cudaError_t launch_t(AttnParams p, cudaStream_t st) {
  auto kern = attn_ws_kernel<D, NVFP4, MMA_BF16, SMOOTH, QSPLIT, APPEND>;
  const int smem = WsSmem<D, QSPLIT>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  p.qpairs = (p.Tq + 255) / 256;
  p.units = p.qpairs * p.H;
  // persistent stream-K grid when a workspace is available, else one CTA per unit
  int n = 0;
  for (int s = 0; s < p.nseg; ++s) n += ((p.seg[s].end + 127) >> 7) - (p.seg[s].begin >> 7);
  if (n == 0 || p.units == 0) return cudaSuccess;
  if ((int64_t)p.units * n >= (int64_t)1 << 31) return cudaErrorInvalidValue;  // 32-bit step indices (Sched)
  int G = p.units;
  bool split = false;
  if (p.ws != nullptr && p.ws_slots >= 2) {
    G = p.ws_slots / 2 < p.max_ctas ? p.ws_slots / 2 : p.max_ctas;
    const int64_t W = (int64_t)p.units * n;
    if (G > W / 2) G = (int)(W / 2);  // at least two (unit, tile) steps per CTA
    if (G < 1) G = 1;
    p.full_units = p.hybrid ? (p.units / G) * G : 0;
    const int64_t Wr = (int64_t)(p.units - p.full_units) * n;  // stream-K remainder
    split = Wr > 0 && ((Wr % G != 0) || ((Wr / G) % n != 0));
  } else {
    p.full_units = 0;
  }
  p.grid = G;
  p.ws_slot_floats = 256 * D + 512;
  if (APPEND) {  // every CTA exchanges its shard amax with all others: co-residency guaranteed or no launch
    if (p.ws == nullptr || G > kMaxCtas) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p);
  } else {
    kern<<<G, kThreads, smem, st>>>(p);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess || !split) return e;
  if (G > 1) combine_kernel<D><<<dim3(G - 1, kCombineSplit), 512, 0, st>>>(p, n);  // per range boundary
  return cudaGetLastError();
}

// v2 is opt-in (environment KVQ_ATTN_V2=1): correct (parity tests), but 945 us against v1's 850 on
// the Wan layer -- the per-tile softmax overheads double with 64-key tiles
bool attn_v2_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("KVQ_ATTN_V2");
    return e != nullptr && e[0] == '1';
  }();
  return on;
}

cudaError_t launch_v2(AttnParams p, cudaStream_t st) {
  auto kern = attn_v2_kernel<128>;
  const int smem = V2Smem::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  p.qpairs = (p.Tq + 255) / 256;
  p.units = p.qpairs * p.H;
  int n = 0;
  for (int s = 0; s < p.nseg; ++s) n += ((p.seg[s].end + 63) >> 6) - (p.seg[s].begin >> 6);
  if (n == 0 || p.units == 0) return cudaSuccess;
  if ((int64_t)p.units * n >= (int64_t)1 << 31) return cudaErrorInvalidValue;
  int G = p.units;
  bool split = false;
  if (p.ws != nullptr && p.ws_slots >= 2) {
    G = p.ws_slots / 2 < p.max_ctas ? p.ws_slots / 2 : p.max_ctas;
    const int64_t W = (int64_t)p.units * n;
    if (G > W / 2) G = (int)(W / 2);
    if (G < 1) G = 1;
    split = (W % G != 0) || ((W / G) % n != 0);
  }
  p.full_units = 0;
  p.grid = G;
  p.ws_slot_floats = 256 * 128 + 512;
  kern<<<G, kThreads, smem, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess || !split) return e;
  if (G > 1) combine_kernel<128><<<dim3(G - 1, kCombineSplit), 512, 0, st>>>(p, n);
  return cudaGetLastError();
}

template <int D, bool SMOOTH>
cudaError_t launch_nvfp4(const AttnParams& p, cudaStream_t st) {
  if (p.q_dtype == DT_FP32) return launch_t<D, true, false, SMOOTH, true>(p, st);
  if (D == 128 && !SMOOTH && p.q_dtype == DT_BF16 && p.q_scale == nullptr && p.o_peer[0] == nullptr && attn_v2_enabled())
    return launch_v2(p, st);
  return launch_t<D, true, false, SMOOTH>(p, st);
}

template <int D>
void touch_attention(cudaFuncAttributes* a) {
  cudaFuncGetAttributes(a, attn_ws_kernel<D, true, false, false, false>);
  cudaFuncGetAttributes(a, attn_ws_kernel<D, true, false, true, false>);
  cudaFuncGetAttributes(a, attn_ws_kernel<D, true, false, false, true>);
  cudaFuncGetAttributes(a, attn_ws_kernel<D, true, false, true, true>);
  cudaFuncGetAttributes(a, combine_kernel<D>);
}

}  // namespace

// module load of the NVFP4 attention kernels (see preload_quant_kernels)
cudaError_t preload_attention_kernels() {
  cudaFuncAttributes a;
  touch_attention<128>(&a);
  touch_attention<64>(&a);
  return cudaGetLastError();
}

// chunk attention with the chunk's quantize/append fused into the launch (plain NVFP4 mode, bf16 Q)
cudaError_t launch_attention_append(const AttnParams& p, cudaStream_t st) {
  return p.d == 128 ? launch_t<128, true, false, false, false, true>(p, st) : launch_t<64, true, false, false, false, true>(p, st);
}

cudaError_t launch_attention(const AttnParams& p, bool nvfp4_kv, cudaStream_t st) {
  if (nvfp4_kv && p.mean_k) return p.d == 128 ? launch_nvfp4<128, true>(p, st) : launch_nvfp4<64, true>(p, st);
  if (nvfp4_kv) return p.d == 128 ? launch_nvfp4<128, false>(p, st) : launch_nvfp4<64, false>(p, st);
  return p.d == 128 ? launch_t<128, false, true>(p, st) : launch_t<64, false, true>(p, st);
}

}  // namespace kvq
