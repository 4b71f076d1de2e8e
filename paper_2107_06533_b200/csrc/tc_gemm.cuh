// Split-precision tcgen05 "TN" tile engine shared by the factor SYRK, the blocked
// sweep-inverse trailing update and the two preconditioning GEMMs.
//
//   D[i][j] = sum_k A[a_row + i][k] * B[b_row + j][k]      (128 x 128 tile, fp32 in TMEM)
//
// Each operand is stored in HBM as two planes [2][rows][ld] (hi, lo) of a
// split-precision pair, K contiguous (K-major).  Three MMAs per K step,
// hi*hi + hi*lo + lo*hi, recover fp32-class accuracy on the tensor cores:
//   Kind::BF16 (kind::f16, bf16 planes): |x - hi - lo| <= 2^-18|x|  (factors, preconditioning)
//   Kind::TF32 (kind::tf32, tf32 planes): |x - hi - lo| <= 2^-22|x|  (inverse updates)
// One TMA producer lane, one MMA-issuing lane, all four warps drain TMEM in the epilogue.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace spd {

constexpr int kStages = 3;
constexpr uint32_t kTileBytes = 128 * 128;  // 128 rows x 128 B (64 bf16 or 32 fp32), SWIZZLE_128B
constexpr uint32_t kStageBytes = 4 * kTileBytes;
constexpr size_t kTcSmemBytes = kStages * kStageBytes + 1024 /*align slack*/ + 256 /*barriers*/;

struct TcItem {
  int32_t a_map, b_map;  // indices into the tensor-map array
  int32_t a_row, b_row;  // operand row offsets (tensor-map dim 1)
  int32_t k0, nk;        // first K element, number of K blocks
  int32_t epi;           // index into the epilogue table
  int32_t flags;         // kSameAB | kMirror
  int32_t out_r, out_c;  // D[i][j] -> target element (out_c + j, out_r + i) (transposed store)
  int32_t m_valid, n_valid;
  int32_t o2_row;  // row offset of the optional second target (TcEpi::out2)
  int32_t b_koff;  // K-major items: B's K coordinate = A's + b_koff (operands in different K columns)
};
constexpr int32_t kSameAB = 1;  // B tile == A tile (diagonal SYRK tile): load once
constexpr int32_t kMirror = 2;  // also update target (out_r + i, out_c + j) (symmetric off-diagonal tile)
constexpr int32_t kMnMajor = 8;  // operands are MN-major split planes [2][K][ld] (bf16 only): each
                                 // 16-KB tile is two 64(MN) x 64(K) TMA boxes at (row, k), (row + 64, k)
constexpr int32_t kF32Rows = 16;  // (kF32 engines) operands are fp32 rows [M][d] read straight from the
                                 // activations by TMA (tensor maps in the F32Maps kernel parameter, a_map /
                                 // b_map index it); converter warps split them into the bf16 hi/lo MN-major
                                 // planes per K block of 32 rows: no staging pass
// fp16 operand classes (TcEpi::dscale[c] is the power-of-two scale of class c): flags bits 8-9 the A
// operand's class, 10-11 the B operand's, 12-13 the out2 planes'.  D carries s_A s_B; the epilogue
// multiplies alpha by 1 / (s_A s_B) and stores out2 planes of (C * s_out2).
constexpr int kScaleShiftA = 8, kScaleShiftB = 10, kScaleShiftO = 12;
SPD_DEV float scale_of(const float* ds, int32_t flags, int shift) { return ds[(flags >> shift) & 3]; }
constexpr int32_t kIm2col = 32;  // (with kMnMajor) operand tiles come from im2col-mode TMA loads of the staged
                                 // NHWC activation planes (TcRun::i2c[map] describes the convolution)
constexpr int32_t kOut2Rows = 4;  // out2 row-style: out2[(o2_row + i) * ld2 + j]; else transposed:
                                  // out2[(o2_row + j) * ld2 + i] (coalesced along the TMEM lanes)

enum EpiMode : int32_t {
  kAxpby = 0,      // out = beta*out + alpha*D   (fp32 target)
  kSplitBf16 = 1,  // out planes (bf16) <- split(alpha*D)
  kSplitTf32 = 2,  // out planes (fp32, tf32-exact) <- split(alpha*D)
  kPackedUpper = 3,  // packed upper triangle of a d x d symmetric target (run.out, run.d):
                     //   P = run.wscale * (run.decay * P + (1 - run.decay) * run.alpha * D), i <= j only
  kUpdate = 4,       // out += run.alpha * D (transposed store; the weight update W -= lr * P)
  kSplitF16 = 5,     // out planes (fp16) <- split(alpha * D * s_out[j]), transposed store like kSplitTf32, with
                     // s_out[j] = scale of bound(gmax * amax_b[b_row + j]) written to rs_out (row scaled planes)
};

// fp32-rows operand maps, passed by value (the activation pointers change between runs; a kernel
// parameter needs no device copy and is captured into CUDA graphs with the launch)
constexpr int kMaxF32Maps = 40;
struct F32Maps {
  CUtensorMap m[kMaxF32Maps];
};
struct NoF32Maps {};
template <bool B>
using F32Param = typename std::conditional<B, F32Maps, NoF32Maps>::type;
constexpr uint32_t kF32Bk = 32;                           // K rows per fp32 stage
constexpr uint32_t kF32Plane = 128 * kF32Bk * 2;          // one bf16 plane of a 128 x 32 tile (8 KB)
constexpr uint32_t kF32Tile = 128 * kF32Bk * 4;           // one fp32 tile (16 KB)
static_assert(4 * kF32Plane + 2 * kF32Tile == 4 * 128 * 128, "an fp32-rows stage reuses a bf16 stage's bytes");

// Per-launch arguments (kernel parameters, not table entries): what changes between runs.
// One channels-last convolution's im2col operand (kIm2col items): the staged hi / lo activation
// planes [2][N*H*W][C], one NHWC tensor map per plane (maps[a_map + p]; output positions past the
// batch are TMA out-of-bounds zeros), column index (tap, channel) = (r * kw + s) * C + c.
struct Im2colGeom {
  int32_t C, kw, taps, Wo, HoWo, N;
  int32_t stride_w, stride_h, pad_w, pad_h, dil_w, dil_h;
};

struct TcRun {
  void* out;     // kPackedUpper target (packed buffer)
  int64_t d;     // matrix dimension of the packed target
  float alpha;   // scale of D (1/M for factors)
  float decay;   // running-average weight of the old value (0: never read)
  float wscale;  // final scale (1/P)
  int32_t pad_;
  Probe* probe;  // launch probe (spdkfac_stats_set_probes) or nullptr
  const Im2colGeom* i2c = nullptr;  // per tensor map (kIm2col items)
};

struct TcEpi {
  void* out;
  int64_t ld;            // row stride (elements) of the target
  int64_t plane_stride;  // elements between hi and lo planes (split modes)
  float alpha, beta;
  int32_t mode;
  int32_t o2_f16;  // out2 planes: 0 = tf32 (fp32 storage), 1 = fp16 scaled by dscale[0]
  // optional second target (kAxpby only): split planes, row (a_row + i), column j:
  // out2[(a_row + i) * ld2 + j] = hi(alpha*D), out2[... + plane2] = lo(alpha*D)
  void* out2;
  int64_t ld2, plane2;
  int32_t c_map;  // kCTile kernels: 2-D tensor map of the fp32 target (box 128 x 128)
  int32_t pad2_;
  // optional per-target operand-class scales in device memory (kAxpby / kCTile; see kScaleShiftA)
  const float* dscale;
  // optional per-row operand scales (fp16 planes of row r hold x * s[r]): D[i][j] carries
  // rs_a[a_row + i] * rs_b[b_row + j], divided out in kAxpby / kUpdate / kSplitF16
  const float* rs_a;
  const float* rs_b;
  // kSplitF16: the bound of output row j (column j of D) is gmax[0] * amax_b[b_row + j]
  const float* gmax;
  const float* amax_b;
  float* rs_out;
};

// power-of-two scale s with |x s| <= 2^13 for |x| <= bound (fp16 planes: 8x headroom below 65504)
__device__ __forceinline__ float f16_scale(float bound) {
  int e = 0;
  if (bound > 0.f && isfinite(bound)) frexpf(bound, &e);  // bound <= 2^e
  e = max(min(e, 100), -100);
  return ldexpf(1.f, 13 - e);
}

// Epilogue of one 32-column chunk of the accumulator tile: thread row i (TMEM lane),
// values v[t] = D[i][c*32 + t].  All global reads of a chunk are issued before any
// store (independent addresses), so read-modify-write targets pay one memory latency
// per chunk, not per element.
__device__ __forceinline__ void epilogue_chunk(const TcItem& it, const TcEpi& ep, const TcRun& run, int i, int c,
                                               const float (&v)[32]) {
  const bool row_ok = i < it.m_valid;
  const int64_t ri = int64_t(it.out_r) + i;
  const int jn = it.n_valid - c * 32;  // valid columns in this chunk (may exceed 32)
  if (ep.mode == kAxpby) {
    float alpha =
        ep.dscale ? ep.alpha / (scale_of(ep.dscale, it.flags, kScaleShiftA) * scale_of(ep.dscale, it.flags, kScaleShiftB))
                  : ep.alpha;
    float v_[32];  // per-row unscaled values (fp16 row-scaled operands)
    if (ep.rs_a) {
      alpha /= ep.rs_a[it.a_row + (row_ok ? i : 0)];
#pragma unroll
      for (int t = 0; t < 32; ++t) v_[t] = (t < jn) ? v[t] / ep.rs_b[it.b_row + c * 32 + t] : 0.f;
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) v_[t] = v[t];
    }
    float* out = static_cast<float*>(ep.out);
    float* base = out + (int64_t(it.out_c) + c * 32) * ep.ld + ri;  // transposed: column j -> row of target
    float old[32];
    if (ep.beta != 0.f) {
#pragma unroll
      for (int t = 0; t < 32; ++t) old[t] = (row_ok && t < jn) ? base[int64_t(t) * ep.ld] : 0.f;
    }
#pragma unroll
    for (int t = 0; t < 32; ++t)
      if (row_ok && t < jn) base[int64_t(t) * ep.ld] = (ep.beta != 0.f ? ep.beta * old[t] : 0.f) + alpha * v_[t];
    if (it.flags & kMirror) {  // same values, target row ri, 32 contiguous columns
      float* rowp = out + ri * ep.ld + it.out_c + c * 32;
      if (ep.beta != 0.f) {
#pragma unroll
        for (int t = 0; t < 32; ++t) old[t] = (row_ok && t < jn) ? rowp[t] : 0.f;
      }
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (row_ok && t < jn) rowp[t] = (ep.beta != 0.f ? ep.beta * old[t] : 0.f) + alpha * v_[t];
    }
    if (ep.out2 != nullptr && row_ok && ep.o2_f16) {  // fp16 planes of (C * s)
      const float sc = scale_of(ep.dscale, it.flags, kScaleShiftO);
      __half* o2b = static_cast<__half*>(ep.out2);
      if (it.flags & kOut2Rows) {
        __half* o2 = o2b + (int64_t(it.o2_row) + i) * ep.ld2 + c * 32;
#pragma unroll
        for (int t = 0; t < 32; t += 8) {
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            __half h0, l0, h1, l1;
            split_f16(alpha * v_[t + 2 * u], sc, h0, l0);
            split_f16(alpha * v_[t + 2 * u + 1], sc, h1, l1);
            hw[u] = uint32_t(__half_as_ushort(h0)) | (uint32_t(__half_as_ushort(h1)) << 16);
            lw[u] = uint32_t(__half_as_ushort(l0)) | (uint32_t(__half_as_ushort(l1)) << 16);
          }
          *reinterpret_cast<uint4*>(o2 + t) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(o2 + ep.plane2 + t) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
      } else {
        __half* o2 = o2b + (int64_t(it.o2_row) + c * 32) * ep.ld2 + i;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          if (t < jn) {
            __half h, l;
            split_f16(alpha * v_[t], sc, h, l);
            o2[int64_t(t) * ep.ld2] = h;
            o2[int64_t(t) * ep.ld2 + ep.plane2] = l;
          }
        }
      }
    } else if (ep.out2 != nullptr && row_ok) {
      if (it.flags & kOut2Rows) {
        float* o2 = static_cast<float*>(ep.out2) + (int64_t(it.o2_row) + i) * ep.ld2 + c * 32;
#pragma unroll
        for (int t = 0; t < 32; t += 4) {
          float h[4], l[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) split_tf32(alpha * v_[t + u], h[u], l[u]);
          *reinterpret_cast<float4*>(o2 + t) = make_float4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<float4*>(o2 + ep.plane2 + t) = make_float4(l[0], l[1], l[2], l[3]);
        }
      } else {
        float* o2 = static_cast<float*>(ep.out2) + (int64_t(it.o2_row) + c * 32) * ep.ld2 + i;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          if (t < jn) {
            float h, l;
            split_tf32(alpha * v_[t], h, l);
            o2[int64_t(t) * ep.ld2] = h;
            o2[int64_t(t) * ep.ld2 + ep.plane2] = l;
          }
        }
      }
    }
  } else if (ep.mode == kSplitBf16) {
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(ep.out);
    const int64_t o0 = (int64_t(it.out_c) + c * 32) * ep.ld + ri;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (row_ok && t < jn) {
        __nv_bfloat16 h, l;
        split_bf16(ep.alpha * v[t], h, l);
        out[o0 + int64_t(t) * ep.ld] = h;
        out[o0 + int64_t(t) * ep.ld + ep.plane_stride] = l;
      }
    }
  } else if (ep.mode == kSplitTf32) {
    float* out = static_cast<float*>(ep.out);
    const int64_t o0 = (int64_t(it.out_c) + c * 32) * ep.ld + ri;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (row_ok && t < jn) {
        float h, l;
        split_tf32(ep.alpha * v[t], h, l);
        out[o0 + int64_t(t) * ep.ld] = h;
        out[o0 + int64_t(t) * ep.ld + ep.plane_stride] = l;
      }
    }
  } else if (ep.mode == kUpdate) {
    float* out = static_cast<float*>(ep.out);
    float* base = out + (int64_t(it.out_c) + c * 32) * ep.ld + ri;  // transposed: column j -> row of target
    float old[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) old[t] = (row_ok && t < jn) ? base[int64_t(t) * ep.ld] : 0.f;
    const float ra = ep.rs_a ? 1.f / ep.rs_a[it.a_row + (row_ok ? i : 0)] : 1.f;
#pragma unroll
    for (int t = 0; t < 32; ++t)
      if (row_ok && t < jn) {
        const float x = ep.rs_a ? v[t] * ra / ep.rs_b[it.b_row + c * 32 + t] : v[t];
        base[int64_t(t) * ep.ld] = fmaf(run.alpha, x, old[t]);
      }
  } else if (ep.mode == kSplitF16) {  // fp16 planes of the output rows j, each with its own scale
    __half* out = static_cast<__half*>(ep.out);
    const int64_t o0 = (int64_t(it.out_c) + c * 32) * ep.ld + ri;
    const float ra = ep.alpha / ep.rs_a[it.a_row + (row_ok ? i : 0)];
    const float g = ep.gmax[0];
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (row_ok && t < jn) {
        const int jb = it.b_row + c * 32 + t;
        const float so = f16_scale(g * ep.amax_b[jb]);
        if (i == 0) ep.rs_out[it.out_c + c * 32 + t] = so;  // the same value from every CTA of this column
        __half h, l;
        split_f16(v[t] * ra / ep.rs_b[jb], so, h, l);
        out[o0 + int64_t(t) * ep.ld] = h;
        out[o0 + int64_t(t) * ep.ld + ep.plane_stride] = l;
      }
    }
  } else {  // kPackedUpper: global row gi = out_r + i, columns gj = out_c + c*32 + t, keep gj >= gi
    // target / dim / scale from the epilogue table (factor groups) or the run arguments (single plan)
    float* out = static_cast<float*>(ep.out ? ep.out : run.out);
    const int64_t gi = ri, d = ep.out ? ep.ld : run.d;
    const float alpha = ep.out ? ep.alpha : run.alpha;
    const int64_t gj0 = int64_t(it.out_c) + c * 32;
    float* rowp = out + gi * (2 * d - gi + 1) / 2 - gi;  // packed index of (gi, gj) = rowp + gj
    float old[32];
    if (run.decay != 0.f) {
#pragma unroll
      for (int t = 0; t < 32; ++t) old[t] = (row_ok && t < jn && gj0 + t >= gi) ? rowp[gj0 + t] : 0.f;
    }
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (row_ok && t < jn && gj0 + t >= gi) {
        const float fresh = alpha * v[t];
        const float nv = run.decay != 0.f ? run.decay * old[t] + (1.f - run.decay) * fresh : fresh;
        rowp[gj0 + t] = run.wscale * nv;
      }
    }
  }
}

// Persistent, warp-specialised tile engine: grid <= #SMs, CTA b processes items b, b+grid, ...
//   warp 0      TMA producer (one lane), kStages-deep smem ring
//   warp 1      MMA issuer (one lane) + TMEM owner; two 128-column accumulators so the
//               next tile's MMAs run while the epilogue drains the previous one
//   warps 2..5  epilogue (warp w drains TMEM lanes [32 (w % 4), +32))
// kCTile (template): the epilogue target is a fp32 matrix reached through a 2-D tensor
// map (TcEpi::c_map): the producer TMA-loads the 128x128 target tile into shared memory
// while the tile's MMAs run, the epilogue applies out = beta*out + alpha*D^T there
// (lanes walk contiguous smem -> conflict-free) and one thread TMA-stores it back.  Used
// for the read-modify-write inverse updates, where per-thread loads left the kernel
// latency-bound at ~2 TB/s.
// kCTile target tiles move as 32-row slices through a ring of two 16-KB slots, loaded and
// stored by one epilogue thread: after slice u is stored it loads slice u + 2 (of this tile,
// or the first slices of the CTA's next tile, which then land during that tile's mainloop).
// The TMA producer only streams operands, and the small ring leaves room for 3 operand
// stages (2 x 64 KB in flight while one is consumed).
constexpr int kCSliceRows = 32;
constexpr int kCSlices = 128 / kCSliceRows;
constexpr int kCRing = 2;
constexpr uint32_t kCSliceBytes = kCSliceRows * 128 * 4;
template <int kSt>
constexpr size_t tc_smem_bytes(bool ctile) {
  return size_t(kSt) * kStageBytes + (ctile ? kCRing * kCSliceBytes : 0) + 1024 + 256;
}

// kAcc > 0: chunked accumulation.  tcgen05.mma accumulates into TMEM with truncation (measured on
// B200: a positive K = 4608 tf32 sum comes out 3.3e-5 low, ~2^-24 per accumulating MMA), which a
// long K chain turns into a biased relative error; the preconditioning GEMMs (K = d_in <= 4608,
// heavy cancellation when the gradient lies in a rank-deficient factor's span) need better.  With
// kAcc, each item's K range is cut into chunks of kAcc K blocks, every chunk is accumulated afresh
// in a TMEM buffer (the two buffers alternate per chunk) and the epilogue warps add the chunks
// into a 128-float register accumulator per row with round-to-nearest fp32 adds.
// kF32: four extra warps (6..9) convert kF32Rows items' fp32 tiles to bf16 hi/lo planes in place
// (the factor SYRK of row-layout members: linear inputs, channels-last output gradients, 1x1 conv
// inputs); the MMA warp waits on their conv[] barrier instead of the TMA's full[].
template <Kind K, int kSt, bool kCTile, int kAcc = 0, bool kF32 = false>
__global__ void __launch_bounds__(kF32 ? 320 : 192, 1)
    tc3_gemm_kernel(const CUtensorMap* __restrict__ maps, const TcItem* __restrict__ items,
                    const TcEpi* __restrict__ epis, const TcRun run, int n_items,
                    const __grid_constant__ F32Param<kF32> fm) {
  static_assert(kAcc == 0 || !kCTile, "chunked accumulation is for register epilogues");
  static_assert(!kF32 || K == Kind::BF16, "fp32-rows operands feed the bf16 SYRK");
  constexpr int BK = is_16bit(K) ? 64 : 32;  // one 128-byte swizzle row of K
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  float* ctile = reinterpret_cast<float*>(smem + kSt * kStageBytes);  // kCRing x [32][128] (kCTile)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSt * kStageBytes + (kCTile ? kCRing * kCSliceBytes : 0));
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;  // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint64_t* cfull = tempty + 2;     // [kCRing] C slice landed
  uint64_t* conv = cfull + kCRing;  // [kSt] (kF32) converted bf16 planes ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv + kSt);

  const int warp = warp_id();
  const int lane = lane_id();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    for (int q = 0; q < kCRing; ++q) mbar_init(&cfull[q], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (kAcc > 0) tmem_alloc<512>(tmem_slot);  // + the chunk-sum accumulator
    else tmem_alloc<256>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  probe_start(run.probe);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      uint32_t g = 0, t = 0;
      int last_a = -1, last_b = -1;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
        const TcItem it = items[item];
        const bool same = (it.flags & kSameAB) != 0;
        if constexpr (kF32) {
          if (it.flags & kF32Rows) {  // fp32 rows: [32 K rows][128 MN] tiles behind the bf16 planes
            const CUtensorMap* am = &fm.m[it.a_map];
            const CUtensorMap* bm = &fm.m[it.b_map];
            for (int kb = 0; kb < it.nk; ++kb, ++g) {
              const uint32_t s = g % kSt;
              mbar_wait(&empty[s], ((g / kSt) & 1) ^ 1);
              mbar_expect_tx(&full[s], same ? kF32Tile : 2 * kF32Tile);
              uint8_t* st = smem + s * kStageBytes + 4 * kF32Plane;
              const int kc = it.k0 + kb * int(kF32Bk);
              tma_load_2d(st, am, &full[s], it.a_row, kc);
              if (!same) tma_load_2d(st + kF32Tile, bm, &full[s], it.b_row, kc);
            }
            continue;
          }
        }
        const CUtensorMap* am = maps + it.a_map;
        const CUtensorMap* bm = maps + it.b_map;
        if (it.a_map != last_a) {
          tmap_acquire(am), last_a = it.a_map;
          if (it.flags & kIm2col) tmap_acquire(am + 1);  // the lo plane's map
        }
        if (!same && it.b_map != last_b) {
          tmap_acquire(bm), last_b = it.b_map;
          if (it.flags & kIm2col) tmap_acquire(bm + 1);
        }
        const uint32_t bytes = same ? 2 * kTileBytes : 4 * kTileBytes;
        for (int kb = 0; kb < it.nk; ++kb, ++g) {
          const uint32_t s = g % kSt;
          mbar_wait(&empty[s], ((g / kSt) & 1) ^ 1);
          mbar_expect_tx(&full[s], bytes);
          uint8_t* st = smem + s * kStageBytes;
          const int kc = it.k0 + kb * BK;
          if (it.flags & kIm2col) {  // 64 output positions x 64 (tap, channel) columns per box
            const Im2colGeom ga = run.i2c[it.a_map];
            const int n0 = kc / ga.HoWo, rem = kc - n0 * ga.HoWo, ho = rem / ga.Wo, wo = rem - ho * ga.Wo;
            const int bw = wo * ga.stride_w - ga.pad_w, bh = ho * ga.stride_h - ga.pad_h;
            auto load_half = [&](uint8_t* dst, const CUtensorMap* mp, int mn, int p) {
              int tap = mn / ga.C;
              const int c0 = mn - tap * ga.C;
              tap = tap < ga.taps ? tap : ga.taps - 1;  // columns past d: any valid box (masked outputs)
              const int r = tap / ga.kw, q = tap - r * ga.kw;
              tma_load_im2col_4d(dst, mp + p, &full[s], c0, bw, bh, n0, uint16_t(q * ga.dil_w), uint16_t(r * ga.dil_h));
            };
#pragma unroll
            for (int p = 0; p < 2; ++p) {
              load_half(st + p * kTileBytes, am, it.a_row, p);
              load_half(st + p * kTileBytes + kTileBytes / 2, am, it.a_row + 64, p);
              if (!same) {
                load_half(st + (2 + p) * kTileBytes, bm, it.b_row, p);
                load_half(st + (2 + p) * kTileBytes + kTileBytes / 2, bm, it.b_row + 64, p);
              }
            }
          } else if (it.flags & kMnMajor) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
              tma_load_3d(st + p * kTileBytes, am, &full[s], it.a_row, kc, p);
              tma_load_3d(st + p * kTileBytes + kTileBytes / 2, am, &full[s], it.a_row + 64, kc, p);
              if (!same) {
                tma_load_3d(st + (2 + p) * kTileBytes, bm, &full[s], it.b_row, kc, p);
                tma_load_3d(st + (2 + p) * kTileBytes + kTileBytes / 2, bm, &full[s], it.b_row + 64, kc, p);
              }
            }
          } else {
            tma_load_3d(st, am, &full[s], kc, it.a_row, 0);
            tma_load_3d(st + kTileBytes, am, &full[s], kc, it.a_row, 1);
            if (!same) {
              tma_load_3d(st + 2 * kTileBytes, bm, &full[s], kc + it.b_koff, it.b_row, 0);
              tma_load_3d(st + 3 * kTileBytes, bm, &full[s], kc + it.b_koff, it.b_row, 1);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc_k = make_idesc<K>(128, 128);
      constexpr uint32_t idesc_mn = idesc_k | (1u << 15) | (1u << 16);  // transpose A and B
      uint32_t g = 0, t = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const TcItem it = items[item];
        const bool same = (it.flags & kSameAB) != 0;
        const int nch = kAcc ? max(1, (it.nk + kAcc - 1) / max(kAcc, 1)) : 1;
        for (int ch = 0; ch < nch; ++ch, ++t) {
        const uint32_t buf = t & 1, use = t >> 1;
        mbar_wait(&tempty[buf], (use & 1) ^ 1);  // epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t acc = tmem + buf * 128;
        const int kb0 = kAcc ? ch * kAcc : 0, kb1 = kAcc ? min(it.nk, kb0 + kAcc) : it.nk;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const uint32_t s = g % kSt;
          const uint32_t first = uint32_t(kb - kb0);  // 0: this chunk starts a fresh accumulator
          uint8_t* st = smem + s * kStageBytes;
          if (kF32 && (it.flags & kF32Rows)) {  // bf16 planes converted from fp32 rows, 32 K rows
            mbar_wait(&conv[s], (g / kSt) & 1);
            tc_fence_after();
            const uint64_t ahi = make_sdesc_sw128_mn_lbo(st, kF32Plane / 2);
            const uint64_t alo = make_sdesc_sw128_mn_lbo(st + kF32Plane, kF32Plane / 2);
            const uint64_t bhi = same ? ahi : make_sdesc_sw128_mn_lbo(st + 2 * kF32Plane, kF32Plane / 2);
            const uint64_t blo = same ? alo : make_sdesc_sw128_mn_lbo(st + 3 * kF32Plane, kF32Plane / 2);
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {  // 16 K rows = two 1024-B atoms per instruction
              const uint64_t off = uint64_t(kk * (2048 >> 4));
              umma<K>(acc, ahi + off, bhi + off, idesc_mn, (first | kk) != 0);
              umma<K>(acc, ahi + off, blo + off, idesc_mn, 1u);
              umma<K>(acc, alo + off, bhi + off, idesc_mn, 1u);
            }
            tc_commit(&empty[s]);
            continue;
          }
          mbar_wait(&full[s], (g / kSt) & 1);
          tc_fence_after();
          if (K == Kind::BF16 && (it.flags & kMnMajor)) {
            const uint64_t ahi = make_sdesc_sw128_mn(st);
            const uint64_t alo = make_sdesc_sw128_mn(st + kTileBytes);
            const uint64_t bhi = same ? ahi : make_sdesc_sw128_mn(st + 2 * kTileBytes);
            const uint64_t blo = same ? alo : make_sdesc_sw128_mn(st + 3 * kTileBytes);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // 16 K rows = two 1024-B atoms per instruction
              const uint64_t off = uint64_t(kk * (2048 >> 4));
              umma<K>(acc, ahi + off, bhi + off, idesc_mn, (first | kk) != 0);
              umma<K>(acc, ahi + off, blo + off, idesc_mn, 1u);
              umma<K>(acc, alo + off, bhi + off, idesc_mn, 1u);
            }
          } else {
            const uint64_t ahi = make_sdesc_sw128(st);
            const uint64_t alo = make_sdesc_sw128(st + kTileBytes);
            const uint64_t bhi = same ? ahi : make_sdesc_sw128(st + 2 * kTileBytes);
            const uint64_t blo = same ? alo : make_sdesc_sw128(st + 3 * kTileBytes);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // 4 x 32 B of K per 128-B swizzle row
              const uint64_t off = uint64_t(kk * 2);
              umma<K>(acc, ahi + off, bhi + off, idesc_k, (first | kk) != 0);
              umma<K>(acc, ahi + off, blo + off, idesc_k, 1u);
              umma<K>(acc, alo + off, bhi + off, idesc_k, 1u);
            }
          }
          tc_commit(&empty[s]);  // smem slot free once these MMAs retire
        }
        tc_commit(&tfull[buf]);
        }
      }
    }
    __syncwarp();
  } else if (kF32 && warp >= 6) {  // ---- fp32 -> bf16 hi/lo converters (warps 6..9)
    if constexpr (kF32) {
      const int ct = int(threadIdx.x) - 192;  // 0..127
      uint32_t g = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const TcItem it = items[item];
        if (!(it.flags & kF32Rows)) {  // keep conv[s]'s phases in step with the slot's uses: arrive once
          for (int kb = 0; kb < it.nk; ++kb, ++g) {  // the TMA data landed (never ahead of the MMA)
            const uint32_t s = g % kSt;
            mbar_wait(&full[s], (g / kSt) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[s]);
          }
          continue;
        }
        const bool same = (it.flags & kSameAB) != 0;
        for (int kb = 0; kb < it.nk; ++kb, ++g) {
          const uint32_t s = g % kSt;
          mbar_wait(&full[s], (g / kSt) & 1);
          uint8_t* st = smem + s * kStageBytes;
          const float* src = reinterpret_cast<const float*>(st + 4 * kF32Plane);
#pragma unroll 1
          for (int op = 0; op < (same ? 1 : 2); ++op) {
            uint8_t* hi = st + 2 * op * kF32Plane;  // A: planes 0, 1; B: planes 2, 3
#pragma unroll
            for (int u = 0; u < 8; ++u) {  // 1024 float4 of a [32][128] fp32 tile, 8 per thread
              const int idx = ct + 128 * u, k = idx >> 5, mn = (idx & 31) << 2;
              const float4 x = *reinterpret_cast<const float4*>(src + op * (kF32Tile / 4) + k * 128 + mn);
              __nv_bfloat16 h[4], l[4];
              split_bf16(x.x, h[0], l[0]);
              split_bf16(x.y, h[1], l[1]);
              split_bf16(x.z, h[2], l[2]);
              split_bf16(x.w, h[3], l[3]);
              // MN-major SWIZZLE_128B: half mn / 64 at +4 KB, row k at k * 128 B, 16-B chunk
              // ((mn % 64) / 8) ^ (k % 8), element (mn % 8) * 2 B
              const uint32_t off = uint32_t(mn >> 6) * (kF32Plane / 2) + uint32_t(k) * 128u +
                                   (uint32_t(((mn & 63) >> 3) ^ (k & 7)) << 4) + uint32_t(mn & 7) * 2u;
              uint2 hv, lv;
              hv.x = uint32_t(__bfloat16_as_ushort(h[0])) | (uint32_t(__bfloat16_as_ushort(h[1])) << 16);
              hv.y = uint32_t(__bfloat16_as_ushort(h[2])) | (uint32_t(__bfloat16_as_ushort(h[3])) << 16);
              lv.x = uint32_t(__bfloat16_as_ushort(l[0])) | (uint32_t(__bfloat16_as_ushort(l[1])) << 16);
              lv.y = uint32_t(__bfloat16_as_ushort(l[2])) | (uint32_t(__bfloat16_as_ushort(l[3])) << 16);
              *reinterpret_cast<uint2*>(hi + off) = hv;
              *reinterpret_cast<uint2*>(hi + kF32Plane + off) = lv;
            }
          }
          fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core's reads
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[s]);
        }
      }
    }
    __syncwarp();
  } else {  // ---- epilogue warps 2..5
    const int quad = warp & 3;
    const int i = quad * 32 + lane;
    const bool cio = kCTile && warp == 2 && lane == 0;  // the C-slice loader / storer
    // slice u of this CTA = slice u % kCSlices of its (u / kCSlices)-th item: rows
    // out_c + kCSliceRows * h of the target, columns out_r ..
    auto load_slice = [&](uint32_t u) {
      const int item = int(blockIdx.x + (u / kCSlices) * gridDim.x);
      if (item >= n_items) return;
      const TcItem it2 = items[item];
      const CUtensorMap* cm = maps + epis[it2.epi].c_map;
      tmap_acquire(cm);
      const uint32_t q = u % kCRing;
      mbar_expect_tx(&cfull[q], kCSliceBytes);
      tma_load_2d(ctile + q * (kCSliceBytes / 4), cm, &cfull[q], it2.out_r,
                  it2.out_c + kCSliceRows * int(u % kCSlices));
    };
    if constexpr (kCTile) {
      if (cio)
        for (uint32_t u = 0; u < kCRing; ++u) load_slice(u);
    }
    uint32_t t = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++t) {
      const TcItem it = items[item];
      const TcEpi ep = epis[it.epi];
      if constexpr (kAcc > 0) {  // sum the item's chunks in TMEM columns [256, 384), then one epilogue
        const int nch = max(1, (it.nk + kAcc - 1) / kAcc);
        const uint32_t lane_off = uint32_t(quad * 32) << 16;
        for (int ch = 0; ch < nch; ++ch, ++t) {
          const uint32_t buf = t & 1, use = t >> 1;
          mbar_wait(&tfull[buf], use & 1);
          tc_fence_after();
          const bool last = ch == nch - 1;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float v[32];
            if (it.nk > 0) {
              tmem_ld_32x32b_x32(tmem + buf * 128 + lane_off + uint32_t(c * 32), v);
            } else {
#pragma unroll
              for (int u = 0; u < 32; ++u) v[u] = 0.f;
            }
            if (ch > 0) {  // round-to-nearest fp32 adds of the chunk partial sums
              float a[32];
              tmem_ld_32x32b_x32(tmem + 256 + lane_off + uint32_t(c * 32), a);
#pragma unroll
              for (int u = 0; u < 32; ++u) v[u] += a[u];
            }
            if (!last) {
              tmem_st_32x32b_x32(tmem + 256 + lane_off + uint32_t(c * 32), v);
            } else if (c * 32 < it.n_valid) {
              epilogue_chunk(it, ep, run, i, c, v);
            }
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);  // TMEM buffer drained: the next chunk may use it
        }
        --t;  // the item loop header advances t past the item's last chunk
        continue;
      }
      const uint32_t buf = t & 1, use = t >> 1;
      const float calpha = (kCTile && ep.dscale) ? ep.alpha / (scale_of(ep.dscale, it.flags, kScaleShiftA) *
                                                                  scale_of(ep.dscale, it.flags, kScaleShiftB))
                                                 : ep.alpha;
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        if (!kCTile && c * 32 >= it.n_valid) break;  // uniform (kCTile targets are whole 128-tiles)
        float v[32];
        if (it.nk > 0) {
          tmem_ld_32x32b_x32(tmem + buf * 128 + (uint32_t(quad * 32) << 16) + uint32_t(c * 32), v);
        } else {
#pragma unroll
          for (int u = 0; u < 32; ++u) v[u] = 0.f;
        }
        if constexpr (kCTile) {  // slice h: slot[j][i] = beta * slot[j][i] + alpha * D[i][j]
          static_assert(kCSliceRows % 32 == 0, "a TMEM chunk of 32 columns lies in one C slice");
          const int h = (c * 32) / kCSliceRows, r0 = (c * 32) % kCSliceRows;
          const uint32_t u2 = kCSlices * t + h, q = u2 % kCRing;
          if (r0 == 0) mbar_wait(&cfull[q], (u2 / kCRing) & 1);
          float* col = ctile + q * (kCSliceBytes / 4) + r0 * 128 + i;
#pragma unroll
          for (int u = 0; u < 32; ++u) col[u * 128] = ep.beta * col[u * 128] + calpha * v[u];
          if (r0 + 32 == kCSliceRows) {  // slice complete: store it, then reuse the slot
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (cio) {
              tma_store_2d(maps + ep.c_map, ctile + q * (kCSliceBytes / 4), it.out_r, it.out_c + kCSliceRows * h);
              tma_store_commit_and_wait_read();
              load_slice(u2 + kCRing);
            }
          }
        } else {
          epilogue_chunk(it, ep, run, i, c, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);  // TMEM drained: MMA may reuse this accumulator
    }
  }
  tc_fence_before();
  __syncthreads();
  probe_stop(run.probe);
  if (warp == 1) {
    if constexpr (kAcc > 0) tmem_free<512>(tmem);
    else tmem_free<256>(tmem);
  }
}


// ------------------------------------------------------------------ CTA-pair engine
// cta_group::2 variant for the symmetric factor SYRK (bf16 split planes, MN-major): a
// cluster of two CTAs computes one 256 x 256 super tile = 2 x 2 blocks of 128.  CTA r
// stages A block (a_row + 128 r) and B block (b_row + 128 r) of every K slab (the same
// 64-KB stage layout as the single-CTA engine, signalled on the leader's barrier); the
// leader issues M = 256, N = 256 MMAs that read both CTAs' shared memory, and each CTA's
// TMEM receives its 128 rows x 256 columns.  Per SM this halves the operand bytes per MMA
// cycle (the single-CTA SYRK sat at ~40% tensor-pipe activity waiting on TMA).
struct TcPairItem {
  int32_t map;           // operand tensor map (A and B both come from it: symmetric factor)
  int32_t a_row, b_row;  // MN coordinates of CTA 0's A and B blocks (CTA 1: +128)
  int32_t k0, nk;
  int32_t epi;
  int32_t flags;         // kSameAB: diagonal super tile, B blocks == A blocks
  int32_t out_r[2];      // per CTA rank: target row offset
  int32_t out_c[4];      // per (rank, half) at [2 r + h]: target column offset, -1 = no store
  int32_t m_valid[2], n_valid[2];
  int32_t pad_;
};

constexpr size_t kPairSmemBytes = size_t(kStages) * kStageBytes + 1024 + 256;

template <int kSt>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    tc3_pair_kernel(const CUtensorMap* __restrict__ maps, const TcPairItem* __restrict__ items,
                    const TcEpi* __restrict__ epis, const TcRun run, int n_items) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSt * kStageBytes);
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;  // [2]
  uint64_t* tempty = tfull + 2;   // [2] (leader: 8 arrivals = 4 epilogue warps x 2 CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const uint32_t pair = cluster_idx(), npairs = cluster_count();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  probe_start(run.probe);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs), completion on the leader's full[s]
      uint32_t g = 0;
      int last = -1;
      for (int item = int(pair); item < n_items; item += int(npairs)) {
        const TcPairItem it = items[item];
        const bool same = (it.flags & kSameAB) != 0;
        const CUtensorMap* m = maps + it.map;
        if (it.map != last) tmap_acquire(m), last = it.map;
        const int ar = it.a_row + 128 * int(rank), br = it.b_row + 128 * int(rank);
        const uint32_t bytes = 2u * (same ? 2 * kTileBytes : 4 * kTileBytes);  // both CTAs
        for (int kb = 0; kb < it.nk; ++kb, ++g) {
          const uint32_t s = g % kSt;
          mbar_wait(&empty[s], ((g / kSt) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], bytes);
          const uint32_t fb = mapa_shared(&full[s], 0);
          uint8_t* st = smem + s * kStageBytes;
          const int kc = it.k0 + kb * 64;
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            tma_load_3d_pair(st + p * kTileBytes, m, fb, ar, kc, p);
            tma_load_3d_pair(st + p * kTileBytes + kTileBytes / 2, m, fb, ar + 64, kc, p);
            if (!same) {
              tma_load_3d_pair(st + (2 + p) * kTileBytes, m, fb, br, kc, p);
              tma_load_3d_pair(st + (2 + p) * kTileBytes + kTileBytes / 2, m, fb, br + 64, kc, p);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---- MMA issuer (leader only)
      constexpr uint32_t idesc = make_idesc<Kind::BF16>(256, 256) | (1u << 15) | (1u << 16);
      uint32_t g = 0, t = 0;
      for (int item = int(pair); item < n_items; item += int(npairs), ++t) {
        const TcPairItem it = items[item];
        const bool same = (it.flags & kSameAB) != 0;
        const uint32_t buf = t & 1, use = t >> 1;
        mbar_wait(&tempty[buf], (use & 1) ^ 1);  // both CTAs drained this accumulator
        tc_fence_after();
        const uint32_t acc = tmem + buf * 256;
        for (int kb = 0; kb < it.nk; ++kb, ++g) {
          const uint32_t s = g % kSt;
          mbar_wait(&full[s], (g / kSt) & 1);
          tc_fence_after();
          uint8_t* st = smem + s * kStageBytes;
          const uint64_t ahi = make_sdesc_sw128_mn(st);
          const uint64_t alo = make_sdesc_sw128_mn(st + kTileBytes);
          const uint64_t bhi = same ? ahi : make_sdesc_sw128_mn(st + 2 * kTileBytes);
          const uint64_t blo = same ? alo : make_sdesc_sw128_mn(st + 3 * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t off = uint64_t(kk * (2048 >> 4));
            umma_pair_bf16(acc, ahi + off, bhi + off, idesc, (kb | kk) != 0);
            umma_pair_bf16(acc, ahi + off, blo + off, idesc, 1u);
            umma_pair_bf16(acc, alo + off, bhi + off, idesc, 1u);
          }
          tc_commit_pair(&empty[s], 3);  // both CTAs' stage s free once these retire
        }
        tc_commit_pair(&tfull[buf], 3);
      }
    }
    __syncwarp();
  } else {  // ---- epilogue warps 2..5 (both CTAs): rows 128 r + i of the super tile
    const int quad = warp & 3;
    const int i = quad * 32 + lane;
    const uint32_t tempty_leader0 = mapa_shared(&tempty[0], 0);
    uint32_t t = 0;
    for (int item = int(pair); item < n_items; item += int(npairs), ++t) {
      const TcPairItem it = items[item];
      const TcEpi ep = epis[it.epi];
      const uint32_t buf = t & 1, use = t >> 1;
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const int32_t occ[2] = {rank ? it.out_c[2] : it.out_c[0], rank ? it.out_c[3] : it.out_c[1]};
      const int32_t orr = rank ? it.out_r[1] : it.out_r[0];
      const int32_t mv = rank ? it.m_valid[1] : it.m_valid[0];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int oc = occ[h];
        if (oc < 0) continue;  // uniform: lower-triangle or padding block
        TcItem ti{};
        ti.out_r = orr;
        ti.out_c = oc;
        ti.m_valid = mv;
        ti.n_valid = it.n_valid[h];
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          if (c * 32 >= ti.n_valid) break;
          float v[32];
          if (it.nk > 0) {
            tmem_ld_32x32b_x32(tmem + buf * 256 + (uint32_t(quad * 32) << 16) + uint32_t(h * 128 + c * 32), v);
          } else {
#pragma unroll
            for (int u = 0; u < 32; ++u) v[u] = 0.f;
          }
          epilogue_chunk(ti, ep, run, i, c, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + buf * 8);  // leader's tempty[buf]
    }
  }
  tc_fence_before();
  cluster_sync();  // the peer's TMEM / smem are read by the leader's MMAs until the end
  probe_stop(run.probe);
  if (warp == 1) tmem_free_pair<512>(tmem);
}


// ------------------------------------------------------------------ CTA-pair C-tile engine
// cta_group::2 variant of the kCTile engine for the blocked inverse's trailing update (tf32 split
// planes, K-major): a cluster of two CTAs computes a 256 x 256 super tile D = A B^T, A = 256 panel
// rows (two 128-blocks, one per CTA), B = 256 panel rows (two 128-blocks, one per CTA), i.e. four
// 128 x 128 target tiles that share their K range.  Each CTA stages only its own A and B blocks per
// K slab (the same 64-KB stage as the single-CTA engine) and the leader's M = N = 256 MMAs read both
// CTAs' shared memory, so per SM the operand bytes per MMA cycle halve -- the single-CTA update ran
// at ~30% tensor-pipe, fed from L2 / DRAM.  CTA r's TMEM holds super-tile rows [128 r, +128) x 256
// columns = its two target tiles h = 0, 1, which it read-modify-writes through the C-slice ring.
struct TcPairCItem {
  int32_t a_map, b_map;  // operand tensor maps
  int32_t a_row, b_row;  // operand rows of CTA 0's blocks (CTA 1: +128)
  int32_t k0, nk;        // first K element, number of 32-wide K blocks
  int32_t epi;           // epilogue table entry (kAxpby on a C-tile target: alpha, beta, c_map)
  int32_t out_r[2];      // per CTA rank: target column offset (the M block)
  int32_t out_c[2];      // per tile h: target row offset (the N block)
  int32_t flags;         // fp16 operand classes (kScaleShiftA / B; TcEpi::dscale)
};

constexpr size_t kPairCSmemBytes = size_t(kStages) * kStageBytes + kCRing * kCSliceBytes + 1024 + 256;

template <int kSt, Kind K = Kind::TF32>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    tc3_pair_ctile_kernel(const CUtensorMap* __restrict__ maps, const TcPairCItem* __restrict__ items,
                          const TcEpi* __restrict__ epis, const TcRun run, int n_items) {
  constexpr int BKp = is_16bit(K) ? 64 : 32;  // K elements per 128-byte operand row
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  float* ctile = reinterpret_cast<float*>(smem + kSt * kStageBytes);  // kCRing x [32][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSt * kStageBytes + kCRing * kCSliceBytes);
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;  // [2]
  uint64_t* tempty = tfull + 2;   // [2] (leader: 8 arrivals = 4 epilogue warps x 2 CTAs)
  uint64_t* cfull = tempty + 2;   // [kCRing] C slice landed (own CTA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfull + kCRing);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const uint32_t pair = cluster_idx(), npairs = cluster_count();
  if (warp == 0 && lane == 0) {
    for (int st = 0; st < kSt; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    for (int q = 0; q < kCRing; ++q) mbar_init(&cfull[q], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  probe_start(run.probe);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs), completion on the leader's full[s]
      uint32_t g = 0;
      int last_a = -1, last_b = -1;
      for (int item = int(pair); item < n_items; item += int(npairs)) {
        const TcPairCItem it = items[item];
        const CUtensorMap* am = maps + it.a_map;
        const CUtensorMap* bm = maps + it.b_map;
        if (it.a_map != last_a) tmap_acquire(am), last_a = it.a_map;
        if (it.b_map != last_b) tmap_acquire(bm), last_b = it.b_map;
        const int ar = it.a_row + 128 * int(rank), br = it.b_row + 128 * int(rank);
        for (int kb = 0; kb < it.nk; ++kb, ++g) {
          const uint32_t st = g % kSt;
          mbar_wait(&empty[st], ((g / kSt) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&full[st], 2u * 4u * kTileBytes);  // both CTAs' A, B hi / lo
          const uint32_t fb = mapa_shared(&full[st], 0);
          uint8_t* sp = smem + st * kStageBytes;
          const int kc = it.k0 + kb * BKp;
          tma_load_3d_pair(sp, am, fb, kc, ar, 0);
          tma_load_3d_pair(sp + kTileBytes, am, fb, kc, ar, 1);
          tma_load_3d_pair(sp + 2 * kTileBytes, bm, fb, kc, br, 0);
          tma_load_3d_pair(sp + 3 * kTileBytes, bm, fb, kc, br, 1);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---- MMA issuer (leader only)
      constexpr uint32_t idesc = make_idesc<K>(256, 256);
      uint32_t g = 0, t = 0;
      for (int item = int(pair); item < n_items; item += int(npairs), ++t) {
        const TcPairCItem it = items[item];
        const uint32_t buf = t & 1, use = t >> 1;
        mbar_wait(&tempty[buf], (use & 1) ^ 1);  // both CTAs drained this accumulator
        tc_fence_after();
        const uint32_t acc = tmem + buf * 256;
        for (int kb = 0; kb < it.nk; ++kb, ++g) {
          const uint32_t st = g % kSt;
          mbar_wait(&full[st], (g / kSt) & 1);
          tc_fence_after();
          uint8_t* sp = smem + st * kStageBytes;
          const uint64_t ahi = make_sdesc_sw128(sp), alo = make_sdesc_sw128(sp + kTileBytes);
          const uint64_t bhi = make_sdesc_sw128(sp + 2 * kTileBytes), blo = make_sdesc_sw128(sp + 3 * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // 4 x 32 B of K per 128-B swizzle row
            const uint64_t off = uint64_t(kk * 2);
            if constexpr (is_16bit(K)) {
              umma_pair_bf16(acc, ahi + off, bhi + off, idesc, (kb | kk) != 0);  // (kind::f16; fp16 via idesc)
              umma_pair_bf16(acc, ahi + off, blo + off, idesc, 1u);
              umma_pair_bf16(acc, alo + off, bhi + off, idesc, 1u);
            } else {
              umma_pair_tf32(acc, ahi + off, bhi + off, idesc, (kb | kk) != 0);
              umma_pair_tf32(acc, ahi + off, blo + off, idesc, 1u);
              umma_pair_tf32(acc, alo + off, bhi + off, idesc, 1u);
            }
          }
          tc_commit_pair(&empty[st], 3);  // both CTAs' stage free once these retire
        }
        tc_commit_pair(&tfull[buf], 3);
      }
    }
    __syncwarp();
  } else {  // ---- epilogue warps 2..5 (both CTAs): rows 128 rank + i of the super tile
    const int quad = warp & 3;
    const int i = quad * 32 + lane;
    const bool cio = warp == 2 && lane == 0;  // the C-slice loader / storer of this CTA
    const uint32_t tempty_leader0 = mapa_shared(&tempty[0], 0);
    constexpr int kSl = 2 * kCSlices;  // C slices per item: tile h = 0 then h = 1
    // slice u of this CTA: slice (u % kCSlices) of tile ((u / kCSlices) % 2) of its (u / kSl)-th item
    auto load_slice = [&](uint32_t u) {
      const int item = int(pair + (u / kSl) * npairs);
      if (item >= n_items) return;
      const TcPairCItem it2 = items[item];
      const CUtensorMap* cm = maps + epis[it2.epi].c_map;
      tmap_acquire(cm);
      const uint32_t q = u % kCRing;
      const int hh = int((u / kCSlices) % 2);
      mbar_expect_tx(&cfull[q], kCSliceBytes);
      tma_load_2d(ctile + q * (kCSliceBytes / 4), cm, &cfull[q], rank ? it2.out_r[1] : it2.out_r[0],
                  (hh ? it2.out_c[1] : it2.out_c[0]) + kCSliceRows * int(u % kCSlices));
    };
    if (cio)
      for (uint32_t u = 0; u < kCRing; ++u) load_slice(u);
    uint32_t t = 0;
    for (int item = int(pair); item < n_items; item += int(npairs), ++t) {
      const TcPairCItem it = items[item];
      const TcEpi ep = epis[it.epi];
      const float calpha = ep.dscale ? ep.alpha / (scale_of(ep.dscale, it.flags, kScaleShiftA) *
                                                   scale_of(ep.dscale, it.flags, kScaleShiftB))
                                     : ep.alpha;
      const uint32_t buf = t & 1, use = t >> 1;
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 2 * kCSlices; ++c) {  // 32-column chunk c of this CTA's 256 columns
        float v[32];
        tmem_ld_32x32b_x32(tmem + buf * 256 + (uint32_t(quad * 32) << 16) + uint32_t(c * 32), v);
        const uint32_t u2 = kSl * t + c, q = u2 % kCRing;
        mbar_wait(&cfull[q], (u2 / kCRing) & 1);
        float* col = ctile + q * (kCSliceBytes / 4) + i;  // slot[j][i] = beta slot[j][i] + alpha D[i][j]
#pragma unroll
        for (int uu = 0; uu < 32; ++uu) col[uu * 128] = ep.beta * col[uu * 128] + calpha * v[uu];
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (cio) {  // slice complete: store it, then reuse the slot
          const int hh = c / kCSlices;
          tma_store_2d(maps + ep.c_map, ctile + q * (kCSliceBytes / 4), rank ? it.out_r[1] : it.out_r[0],
                       (hh ? it.out_c[1] : it.out_c[0]) + kCSliceRows * (c % kCSlices));
          tma_store_commit_and_wait_read();
          load_slice(u2 + kCRing);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + buf * 8);  // leader's tempty[buf]
    }
  }
  tc_fence_before();
  cluster_sync();  // the peer's TMEM / smem are read by the leader's MMAs until the end
  probe_stop(run.probe);
  if (warp == 1) tmem_free_pair<512>(tmem);
}

}  // namespace spd
