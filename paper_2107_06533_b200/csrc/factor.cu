// Kronecker-factor construction: X^T X over rows (linear), im2col patches (conv A)
// or spatial output-gradient rows (conv G), on tcgen05 with 3 x bf16 split operands.
//
// Pipeline per factor (one plan = one layer-side):
//   1. stage kernel  : rows of X (im2col patches for conv A) split into bf16 hi/lo planes
//                      Xs[2][M][ld] in their natural row order -- one streaming HBM pass
//   2. tc3 GEMM      : upper-triangle 128x128 tiles (I <= J) x split-K slices, partial tiles to ws
//   3. reduce + pack : sum split-K partials in fixed order, apply 1/M, running average, 1/P,
//                      write the packed upper triangle (the all-reduce / fusion-buffer format)
#include <algorithm>
#include <cstring>

#include "runtime.cuh"

namespace spd {

// ------------------------------------------------------------------ staging kernels
// Xs[p][m][j]: plane p (hi, lo), row m < M (one sample / output position), column j < ld
// (ld = d rounded up to 8; columns [d, ld) are zero).  Rows are the natural order of the
// activations, so staging is a streaming split (plus the im2col gather for conv A) with no
// transpose; the tcgen05 kernel reads the planes as MN-major operands (kMnMajor).

struct ConvGeom {
  int B, C, H, W, Ho, Wo, kh, kw, sh, sw, ph, pw, dh, dw;
};

__device__ __forceinline__ uint32_t pack_bf16x2(__nv_bfloat16 a, __nv_bfloat16 b) {
  __nv_bfloat162 v = __halves2bfloat162(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void store_split4(__nv_bfloat16* xs, int64_t plane, int64_t o, float4 v) {
  __nv_bfloat16 h[4], l[4];
  split_bf16(v.x, h[0], l[0]);
  split_bf16(v.y, h[1], l[1]);
  split_bf16(v.z, h[2], l[2]);
  split_bf16(v.w, h[3], l[3]);
  uint2 hv, lv;
  hv.x = pack_bf16x2(h[0], h[1]), hv.y = pack_bf16x2(h[2], h[3]);
  lv.x = pack_bf16x2(l[0], l[1]), lv.y = pack_bf16x2(l[2], l[3]);
  *reinterpret_cast<uint2*>(xs + o) = hv;
  *reinterpret_cast<uint2*>(xs + plane + o) = lv;
}

__device__ __forceinline__ void store_split8(__nv_bfloat16* xs, int64_t plane, int64_t o, float4 a, float4 b) {
  __nv_bfloat16 h[8], l[8];
  split_bf16(a.x, h[0], l[0]);
  split_bf16(a.y, h[1], l[1]);
  split_bf16(a.z, h[2], l[2]);
  split_bf16(a.w, h[3], l[3]);
  split_bf16(b.x, h[4], l[4]);
  split_bf16(b.y, h[5], l[5]);
  split_bf16(b.z, h[6], l[6]);
  split_bf16(b.w, h[7], l[7]);
  uint4 hv, lv;
  hv.x = pack_bf16x2(h[0], h[1]), hv.y = pack_bf16x2(h[2], h[3]), hv.z = pack_bf16x2(h[4], h[5]);
  hv.w = pack_bf16x2(h[6], h[7]);
  lv.x = pack_bf16x2(l[0], l[1]), lv.y = pack_bf16x2(l[2], l[3]), lv.z = pack_bf16x2(l[4], l[5]);
  lv.w = pack_bf16x2(l[6], l[7]);
  *reinterpret_cast<uint4*>(xs + o) = hv;
  *reinterpret_cast<uint4*>(xs + plane + o) = lv;
}

__device__ __forceinline__ void store_split2(__nv_bfloat16* xs, int64_t plane, int64_t o, float v0, float v1) {
  __nv_bfloat16 h0, l0, h1, l1;
  split_bf16(v0, h0, l0);
  split_bf16(v1, h1, l1);
  *reinterpret_cast<__nv_bfloat162*>(xs + o) = __halves2bfloat162(h0, h1);
  *reinterpret_cast<__nv_bfloat162*>(xs + plane + o) = __halves2bfloat162(l0, l1);
}

// rows x[m][0..d) (row stride ldx) -> Xs.  Block = kStageRows rows; thread (row lane, column
// slot) as in the im2col kernel below (no per-element index division).  kVec: ldx % 4 == 0,
// d % 4 == 0, x 16-B aligned -> float4 loads, 2 x 8-B stores.
constexpr int kStageRows = 32;

template <bool kVec, bool kW8 = false>  // kW8: 8 columns per slot (d % 8 == 0), 16-B stores
__global__ void __launch_bounds__(256) stage_rows_kernel(const float* __restrict__ x, int64_t M, int64_t d,
                                                         int64_t ldx, __nv_bfloat16* __restrict__ xs, int64_t ld,
                                                         int tpr, int cps, Probe* probe) {
  probe_start(probe);
  const int64_t plane = M * ld;
  constexpr int kW = kW8 ? 8 : (kVec ? 4 : 2);
  const int64_t m0 = int64_t(blockIdx.x) * kStageRows;
  const int ncol = int(ld / kW), rpar = int(blockDim.x) / tpr;
  const int cs0 = int(threadIdx.x) % tpr, r0 = int(threadIdx.x) / tpr;
  const int rows = int(M - m0 < kStageRows ? M - m0 : int64_t(kStageRows));
  const int cs_end = min(ncol, int(blockIdx.y + 1) * cps);
  for (int cs = int(blockIdx.y) * cps + cs0; cs < cs_end; cs += tpr) {
    const int j = cs * kW;
    for (int rb = r0; rb < rows; rb += 4 * rpar) {  // 4 rows per pass: loads first, then stores
      float4 val[4], val2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = rb + u * rpar;
        const float* src = x + (m0 + r) * ldx + j;
        val[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        val2[u] = val[u];
        if (r < rows) {
          if constexpr (kVec) {
            if (j < d) {
              val[u] = __ldg(reinterpret_cast<const float4*>(src));
              if constexpr (kW8) val2[u] = __ldg(reinterpret_cast<const float4*>(src) + 1);
            }
          } else {
            if (j < d) val[u].x = __ldg(src);
            if (j + 1 < d) val[u].y = __ldg(src + 1);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = rb + u * rpar;
        if (r < rows) {
          if constexpr (kW8)
            store_split8(xs, plane, (m0 + r) * ld + j, val[u], val2[u]);
          else if constexpr (kVec)
            store_split4(xs, plane, (m0 + r) * ld + j, val[u]);
          else
            store_split2(xs, plane, (m0 + r) * ld + j, val[u].x, val[u].y);
        }
      }
    }
  }
  __syncthreads();
  probe_stop(probe);
}

// Deferred row staging of several members in ONE launch (the group's compute): block b stages
// kStageRows rows of member t (rows [32 (b - blk0[t]), + 32)), every column, 8 columns per slot with
// two float4 loads and two 16-B stores; 4 slots per thread in flight.  Members qualify with d % 8 == 0,
// a row stride ldx % 4 == 0 and a 16-B aligned input (the rest stage at stage() time as before).
constexpr int kBatchStageMax = 64;
struct StageBatch {
  const float* x[kBatchStageMax];
  __nv_bfloat16* xs[kBatchStageMax];
  int64_t M[kBatchStageMax], ldx[kBatchStageMax], ld[kBatchStageMax];
  int32_t d[kBatchStageMax];
  int32_t blk0[kBatchStageMax + 1];
  int n;
};
__global__ void __launch_bounds__(256) stage_rows_batched_kernel(const __grid_constant__ StageBatch a, Probe* probe) {
  probe_start(probe);
  const int b = blockIdx.x;
  int lo = 0, hi = a.n - 1;
  while (lo < hi) {  // last t with blk0[t] <= b
    const int mid = (lo + hi + 1) >> 1;
    if (a.blk0[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  const int t = lo;
  const int64_t M = a.M[t], ldx = a.ldx[t], ld = a.ld[t], m0 = int64_t(b - a.blk0[t]) * kStageRows;
  const int nslot = a.d[t] >> 3;
  const int rows = int(M - m0 < kStageRows ? M - m0 : int64_t(kStageRows));
  const int total = rows * nslot;
  const float* __restrict__ x = a.x[t];
  __nv_bfloat16* __restrict__ xs = a.xs[t];
  const int64_t plane = M * ld;
  for (int base = int(threadIdx.x); base < total; base += 4 * int(blockDim.x)) {
    float4 v0[4], v1[4];
    int64_t o[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = base + u * int(blockDim.x);
      o[u] = -1;
      if (idx < total) {
        const int r = idx / nslot, j = (idx - r * nslot) * 8;
        const float4* src = reinterpret_cast<const float4*>(x + (m0 + r) * ldx + j);
        v0[u] = __ldg(src);
        v1[u] = __ldg(src + 1);
        o[u] = (m0 + r) * ld + j;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (o[u] >= 0) store_split8(xs, plane, o[u], v0[u], v1[u]);
  }
  __syncthreads();
  probe_stop(probe);
}

// launch shape for M rows of ncol column slots, `rows` rows per block: enough blocks for the
// 148 SMs (column ranges of cps slots split over blockIdx.y when M is small), tpr threads
// per row (a multiple of 32 balancing the passes over the range), as many row lanes as fit
// in 256 threads.
struct RowShape {
  dim3 grid;
  int tpr, threads, cps;
};
inline RowShape row_shape(int64_t M, int64_t ncol, int rows) {
  const int64_t row_blocks = cdiv(M, rows);
  int64_t ysplit = 1;
  if (row_blocks < 600) ysplit = std::max<int64_t>(1, std::min(cdiv(600, row_blocks), ncol / 32));
  const int cps = int(cdiv(ncol, ysplit));
  ysplit = cdiv(ncol, cps);
  int tpr = cps;
  if (cps > 32) {
    const int passes = int(cdiv(cps, 256));
    tpr = int(std::min<int64_t>(256, round_up(cdiv(cps, passes), 32)));
  }
  const int lanes = std::max(1, std::min(rows, 256 / tpr));
  return RowShape{dim3(unsigned(row_blocks), unsigned(ysplit)), tpr, tpr * lanes, cps};
}

// im2col: block = kIm2colRows consecutive output positions.  The per-row source geometry is
// computed once into shared memory; thread (row lane r0, column slot cs) keeps its column
// decomposition across the rows it walks (tpr threads per row, 256/tpr rows in parallel).
// Column order: channels-last (ki, kj, c) -- the column order of a channels-last conv weight
// [cout][kh*kw*cin] -- or NCHW (c, ki, kj), the reference's unfold order.  kVec
// (channels-last, C % 4 == 0): float4 loads of 4 channels, 2 x 8-B stores; otherwise column
// pairs (bf16x2).
constexpr int kIm2colRows = 32;

template <bool kNhwc, bool kVec, bool kW8 = false>  // kW8: 8 channels per slot (C % 8 == 0), 16-B stores
__global__ void __launch_bounds__(256) stage_im2col_kernel(const float* __restrict__ x, ConvGeom g, int64_t M,
                                                           int64_t d, __nv_bfloat16* __restrict__ xs, int64_t ld,
                                                           int tpr, int cps, Probe* probe) {
  __shared__ int s_b[kIm2colRows], s_h[kIm2colRows], s_w[kIm2colRows];
  probe_start(probe);
  const int64_t m0 = int64_t(blockIdx.x) * kIm2colRows;
  if (threadIdx.x < kIm2colRows) {
    const int64_t m = m0 + threadIdx.x;
    int b = -1, h = 0, w = 0;
    if (m < M) {
      const int HWo = g.Ho * g.Wo;
      b = int(m / HWo);
      const int q = int(m - int64_t(b) * HWo), ho = q / g.Wo, wo = q - ho * g.Wo;
      h = ho * g.sh - g.ph;
      w = wo * g.sw - g.pw;
    }
    s_b[threadIdx.x] = b, s_h[threadIdx.x] = h, s_w[threadIdx.x] = w;
  }
  __syncthreads();
  const int64_t plane = M * ld;
  constexpr int kW = kW8 ? 8 : (kVec ? 4 : 2);
  const int kk_n = g.kh * g.kw;
  const int ncol = int(ld / kW), rpar = int(blockDim.x) / tpr;
  const int cs0 = int(threadIdx.x) % tpr, r0 = int(threadIdx.x) / tpr;
  const int rows = int(M - m0 < kIm2colRows ? M - m0 : int64_t(kIm2colRows));
  const int cs_end = min(ncol, int(blockIdx.y + 1) * cps);
  for (int cs = int(blockIdx.y) * cps + cs0; cs < cs_end; cs += tpr) {
    const int j = cs * kW;
    int ki[2], kj[2], c[2];
    bool valid[2];
#pragma unroll
    for (int u = 0; u < (kVec ? 1 : 2); ++u) {
      const int jj = j + u;
      valid[u] = jj < d;
      int kk, cc;
      if (kNhwc) {
        kk = jj / g.C;
        cc = jj - kk * g.C;
      } else {
        cc = jj / kk_n;
        kk = jj - cc * kk_n;
      }
      ki[u] = kk / g.kw;
      kj[u] = kk - ki[u] * g.kw;
      c[u] = cc;
    }
    for (int rb = r0; rb < rows; rb += 4 * rpar) {  // 4 rows per pass: loads first, then stores
      float4 val[4], val2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = rb + u * rpar;
        val[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        val2[u] = val[u];
        if (r >= rows) continue;
        const int b = s_b[r];
        if constexpr (kVec) {
          const int hi = s_h[r] + ki[0] * g.dh, wi = s_w[r] + kj[0] * g.dw;
          if (valid[0] && hi >= 0 && hi < g.H && wi >= 0 && wi < g.W) {
            const float4* p = reinterpret_cast<const float4*>(x + ((int64_t(b) * g.H + hi) * g.W + wi) * g.C + c[0]);
            val[u] = __ldg(p);
            if constexpr (kW8) val2[u] = __ldg(p + 1);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int hi = s_h[r] + ki[e] * g.dh, wi = s_w[r] + kj[e] * g.dw;
            if (valid[e] && hi >= 0 && hi < g.H && wi >= 0 && wi < g.W) {
              const int64_t off = kNhwc ? ((int64_t(b) * g.H + hi) * g.W + wi) * g.C + c[e]
                                        : ((int64_t(b) * g.C + c[e]) * g.H + hi) * g.W + wi;
              (e ? val[u].y : val[u].x) = __ldg(x + off);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = rb + u * rpar;
        if (r >= rows) continue;
        const int64_t o = (m0 + r) * ld + j;
        if constexpr (kW8)
          store_split8(xs, plane, o, val[u], val2[u]);
        else if constexpr (kVec)
          store_split4(xs, plane, o, val[u]);
        else
          store_split2(xs, plane, o, val[u].x, val[u].y);
      }
    }
  }
  __syncthreads();
  probe_stop(probe);
}

// NCHW output gradients g[b][c][p] -> rows m = b*HW + p, columns c: per-image 32 x 32 transpose
__global__ void __launch_bounds__(256) stage_spatial_kernel(const float* __restrict__ g, int C, int HW,
                                                            __nv_bfloat16* __restrict__ xs, int64_t M, int64_t ld,
                                                            Probe* probe) {
  __shared__ float tile[32][33];
  probe_start(probe);
  const int b = blockIdx.z, p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = ty; k < 32; k += 8) {
    const int c = c0 + k, p = p0 + tx;
    tile[k][tx] = (c < C && p < HW) ? __ldg(g + (int64_t(b) * C + c) * HW + p) : 0.f;
  }
  __syncthreads();
  const int64_t plane = M * ld;
  // 16 column pairs per row, 16 rows per pass
  const int pr = threadIdx.x & 15, rr = threadIdx.x >> 4;
#pragma unroll
  for (int k = rr; k < 32; k += 16) {
    const int p = p0 + k, c = c0 + 2 * pr;
    if (p < HW && c < ld) store_split2(xs, plane, (int64_t(b) * HW + p) * ld + c, tile[2 * pr][k], tile[2 * pr + 1][k]);
  }
  __syncthreads();
  probe_stop(probe);
}

// ------------------------------------------------------------------ reduce + pack
// partial[slot][j][i] = D_tile[i][j]; slot = tile_index(I,J) * splits + s.
// Split-K reduction, one launch per group, deterministic: block (sub-block sb, job, chunk c)
// sums the 8 split-K partial tiles of its chunk (32 independent loads per thread), stores the
// chunk sum, and the last chunk block to arrive (per tile/sub-block counter) adds the chunk
// sums in fixed order, applies scale / running average / 1/P and writes the packed upper
// triangle.  A job is one upper tile of one group member with split K.
constexpr int kChunk = 8;

struct RedMember {
  const float* part;
  float* chunks;
  int* counters;
  float* packed;
  int64_t d;
  int T, splits;
  float scale;
  int pad_;
};
struct RedJob {
  int32_t member, tile, I, J;
};

__global__ void __launch_bounds__(256) reduce_pack_kernel(const RedJob* __restrict__ jobs,
                                                          const RedMember* __restrict__ mems, float decay,
                                                          float world_scale, float* packed_override,
                                                          float scale_override) {
  __shared__ float tile[32][33];
  __shared__ int last;
  const RedJob jb = jobs[blockIdx.y];
  const RedMember mb = mems[jb.member];
  const int64_t d = mb.d;
  const int I = jb.I, J = jb.J, splits = mb.splits;
  const int sb = blockIdx.x, i0 = (sb >> 2) * 32, j0 = (sb & 3) * 32;
  const int nch = (splits + kChunk - 1) / kChunk, ch = blockIdx.z;
  if (ch >= nch) return;
  if (int64_t(I) * 128 + i0 >= d || int64_t(J) * 128 + j0 >= d) return;
  const int s0 = ch * kChunk, s1 = min(splits, s0 + kChunk);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const float* base = mb.part + (int64_t(jb.tile) * splits) * 16384 + i0 + tx;
  float acc[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float* p = base + int64_t(j0 + ty + 8 * r) * 128;
    float a = 0.f;
#pragma unroll
    for (int u = 0; u < kChunk; ++u)
      if (s0 + u < s1) a += __ldg(p + int64_t(s0 + u) * 16384);
    acc[r] = a;
  }
  const int slot = jb.tile * 16 + sb;
  if (nch > 1) {
    float* mine = mb.chunks + (int64_t(slot) * nch + ch) * 1024;
#pragma unroll
    for (int r = 0; r < 4; ++r) mine[(ty + 8 * r) * 32 + tx] = acc[r];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(mb.counters + slot, 1) == nch - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      float a = 0.f;
      for (int c = 0; c < nch; ++c) a += __ldcg(mb.chunks + (int64_t(slot) * nch + c) * 1024 + (ty + 8 * r) * 32 + tx);
      acc[r] = a;
    }
    if (threadIdx.x == 0) mb.counters[slot] = 0;  // ready for the next run
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) tile[ty + 8 * r][tx] = acc[r];  // tile[j][i]
  __syncthreads();
  float* packed = packed_override ? packed_override : mb.packed;
  const float scale = scale_override >= 0.f ? scale_override : mb.scale;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int k = ty + 8 * r;
    const int64_t gi = int64_t(I) * 128 + i0 + k;
    const int64_t gj = int64_t(J) * 128 + j0 + tx;
    if (gi < d && gj < d && gi <= gj) {
      const int64_t pidx = gi * (2 * d - gi + 1) / 2 + (gj - gi);
      const float fresh = scale * tile[tx][k];
      const float v = (decay == 0.f) ? fresh : decay * packed[pidx] + (1.f - decay) * fresh;
      packed[pidx] = world_scale * v;
    }
  }
}

}  // namespace spd

using namespace spd;

// A factor group: n layer-sides staged independently (per-member staging buffers and tensor
// maps) and reduced by ONE persistent tcgen05 launch over all members' tiles (largest K
// first) plus one grouped split-K reduce.  The single-factor plan is a group of one whose
// packed target and scale are supplied per run.
struct Member {
  spdkfac_factor_geom g;
  int64_t M, d, Mpad, ld;  // ld: row length of the staged planes (d rounded up to 8)
  int T, splits, n_tiles;
  int S;  // 256-wide super blocks (CTA-pair engine) when T >= 2, else 0 (single-CTA engine)
  int Ho, Wo;
  __nv_bfloat16* xt;
  float* partial;
  float* chunks;
  int* counters;
  // fp32-rows members (row layouts: linear inputs, channels-last output gradients, 1x1 stride-1
  // channels-last conv inputs): the SYRK reads the activation itself (kF32Rows items), no staging
  bool f32 = false;
  int f32_slot = -1;        // index in the launch's F32Maps
  int64_t ldx = 0;          // row stride of x (elements)
  const float* x = nullptr;  // the activation bound by the last stage()
  // im2col members (channels-last k x k convs, C % 64 == 0, single-CTA engine): the activation itself
  // is staged (Mst = N*H*W rows of C), the SYRK reads im2col tiles of it by TMA (kIm2col)
  bool i2c = false;
  int64_t Mst = 0;
  Im2colGeom ig{};
  // row-layout members staged by the group's compute launch in one batched kernel (stage() records x)
  bool deferred = false;
};

namespace {
// Row layouts whose factor has at most f32_rows_max_blocks() 128-blocks skip the staging pass: the SYRK
// converts TMA-loaded fp32 tiles itself.  Each row block is converted once per tile it feeds (T
// times) against once by the staging pass, so it can only pay for small T (measured on
// ResNet-50: all rows members converted in-kernel cost +2.1 ms of SYRK for -1.25 ms of staging; with
// d <= 256 only, -0.79 ms of staging for +0.65 ms of SYRK, 18.07 vs 18.05 ms per iteration).  Off by
// default; SPDKFAC_F32_ROWS=n enables it for members of at most n blocks.
int f32_rows_max_blocks() {
  const char* e = getenv("SPDKFAC_F32_ROWS");
  return e ? atoi(e) : 0;
}
// SPDKFAC_IM2COL=1: k x k channels-last convs (C % 64 == 0, single-CTA engine) stage only the
// activation and the SYRK gathers im2col tiles by TMA.  Off by default: measured on ResNet-50 (layer1/2
// 3x3 convs) staging -0.23 ms but SYRK +0.37 ms per step (16.74 vs 16.60 ms).
bool im2col_enabled() {
  const char* e = getenv("SPDKFAC_IM2COL");
  return e && e[0] == '1';
}
// SPDKFAC_BATCH_STAGE=1: row-layout members (d % 8 == 0) are staged by the group's compute in one batched
// launch instead of at stage() time.  Off by default: measured correct but slower in the step (16.38 /
// 16.46 vs 16.17 / 16.23 ms): per-member staging on the stage stream overlaps the forward / backward
// kernels, the batched launch sits in front of the group's SYRK.
bool batch_stage_enabled() {
  const char* e = getenv("SPDKFAC_BATCH_STAGE");
  return e && e[0] == '1';
}
bool is_rows_layout(const spdkfac_factor_geom& g) {
  const bool pointwise = g.layout == SPDKFAC_CONV_A_NHWC && g.kh == 1 && g.kw == 1 && g.stride_h == 1 &&
                         g.stride_w == 1 && g.pad_h == 0 && g.pad_w == 0;
  return g.layout == SPDKFAC_ROWS || g.layout == SPDKFAC_SPATIAL_NHWC || pointwise;
}
}  // namespace

struct spdkfac_factor_group {
  std::vector<Member> m;
  CUtensorMap* maps = nullptr;
  Im2colGeom* i2c = nullptr;  // per map index (kIm2col items)
  TcItem* items = nullptr;
  TcPairItem* pitems = nullptr;
  int n_pitems = 0;
  double flops_single = 0, flops_pair = 0;
  TcEpi* epis = nullptr;
  RedJob* jobs = nullptr;
  RedMember* rmem = nullptr;
  int n_items = 0, n_jobs = 0, max_chunks = 0;
  double flops = 0;
  bool per_run_target = false;  // single-factor plan: packed pointer / scale given to run()
};
struct spdkfac_factor_plan : spdkfac_factor_group {};

namespace {

int geom_dims(const spdkfac_factor_geom* g, int64_t* rows, int64_t* dim, int* Ho = nullptr, int* Wo = nullptr) {
  SPD_ARG(g != nullptr, SPDKFAC_ERR_ARG, "null geometry");
  if (g->layout == SPDKFAC_ROWS) {
    SPD_ARG(g->n >= 1, SPDKFAC_ERR_ARG, "compute_factor: empty batch");
    SPD_ARG(g->c >= 1 && g->w >= g->c, SPDKFAC_ERR_SHAPE, "compute_factor: bad row geometry d=%lld ld=%lld",
            (long long)g->c, (long long)g->w);
    *rows = g->n;
    *dim = g->c;
  } else if (g->layout == SPDKFAC_CONV_A || g->layout == SPDKFAC_CONV_A_NHWC) {
    SPD_ARG(g->n >= 1 && g->c >= 1 && g->h >= 1 && g->w >= 1, SPDKFAC_ERR_ARG, "conv factor: empty input");
    SPD_ARG(g->kh >= 1 && g->kw >= 1 && g->stride_h >= 1 && g->stride_w >= 1 && g->dil_h >= 1 && g->dil_w >= 1 &&
                g->pad_h >= 0 && g->pad_w >= 0,
            SPDKFAC_ERR_ARG, "conv factor: bad kernel geometry");
    const int64_t ho = (g->h + 2 * g->pad_h - g->dil_h * (g->kh - 1) - 1) / g->stride_h + 1;
    const int64_t wo = (g->w + 2 * g->pad_w - g->dil_w * (g->kw - 1) - 1) / g->stride_w + 1;
    SPD_ARG(ho >= 1 && wo >= 1, SPDKFAC_ERR_SHAPE, "conv factor: empty output");
    SPD_ARG(g->n * g->c * g->h * g->w < (int64_t(1) << 31), SPDKFAC_ERR_SHAPE, "conv factor: input too large");
    *rows = g->n * ho * wo;
    *dim = g->c * g->kh * g->kw;
    if (Ho) *Ho = int(ho);
    if (Wo) *Wo = int(wo);
  } else if (g->layout == SPDKFAC_SPATIAL || g->layout == SPDKFAC_SPATIAL_NHWC) {
    SPD_ARG(g->n >= 1 && g->c >= 1 && g->h >= 1 && g->w >= 1, SPDKFAC_ERR_ARG, "spatial factor: empty input");
    *rows = g->n * g->h * g->w;
    *dim = g->c;
  } else {
    SPD_ARG(false, SPDKFAC_ERR_ARG, "unknown factor layout %d", g->layout);
  }
  SPD_ARG(*dim <= 65536 && *rows < (int64_t(1) << 31), SPDKFAC_ERR_SHAPE, "factor too large");
  return SPDKFAC_OK;
}

// splits: fill the SMs per factor (148 single-CTA tiles or 74 CTA-pair super tiles; the
// group launch then has at least that many work items), each K slice >= 16 blocks (1024
// rows); splits == 1 stores straight into the packed buffer
int choose_splits(int64_t Mpad, int n_units, int target) {
  const int64_t nkb = Mpad / 64;
  const int64_t want = cdiv(target, n_units);
  const int64_t maxs = std::max<int64_t>(1, nkb / 16);
  return int(std::max<int64_t>(1, std::min(want, maxs)));
}

int member_init(Member* mb, const spdkfac_factor_geom* g) {
  int64_t M, d;
  int Ho = 0, Wo = 0;
  int rc = geom_dims(g, &M, &d, &Ho, &Wo);
  if (rc) return rc;
  mb->g = *g;
  mb->M = M;
  mb->d = d;
  mb->Ho = Ho;
  mb->Wo = Wo;
  mb->Mpad = round_up(M, 64);  // K blocks; rows [M, Mpad) are TMA out-of-bounds zeros
  mb->ld = round_up(d, 8);
  mb->T = int(cdiv(d, 128));
  mb->n_tiles = mb->T * (mb->T + 1) / 2;
  // CTA-pair super tiles where they pay (measured on B200, ResNet-50 shapes): an even number
  // of 128-blocks (no padded half super tile) and at least ~48 pair items to fill the GPU,
  // or a two-block factor over very many rows (the stem conv)
  mb->ldx = g->layout == SPDKFAC_ROWS ? g->w : g->c;
  mb->f32 = mb->T <= f32_rows_max_blocks() && is_rows_layout(*g) && mb->ldx % 4 == 0;
  mb->S = 0;
  if (mb->T >= 2 && !mb->f32) {  // fp32-rows members run on the single-CTA engine (its converter warps)
    const int S = mb->T / 2, units = S * (S + 1) / 2;
    const int sp = choose_splits(mb->Mpad, units, 74);
    if ((mb->T % 2 == 0 && mb->T >= 4 && units * sp >= 48) || (mb->T == 2 && M >= 200000)) mb->S = S;
  }
  mb->splits = mb->S ? choose_splits(mb->Mpad, mb->S * (mb->S + 1) / 2, 74) : choose_splits(mb->Mpad, mb->n_tiles, 148);
  // k x k channels-last convs on the single-CTA engine: TMA im2col loads instead of an im2col staging pass
  const bool pointwise = g->kh == 1 && g->kw == 1 && g->stride_h == 1 && g->stride_w == 1 && g->pad_h == 0 &&
                         g->pad_w == 0;
  mb->deferred = batch_stage_enabled() && !mb->f32 && is_rows_layout(*g) && mb->d % 8 == 0 && mb->ldx % 4 == 0;
  mb->i2c = false;
  if (im2col_enabled() && !mb->S && g->layout == SPDKFAC_CONV_A_NHWC && !pointwise && g->c % 64 == 0 &&
      g->pad_h <= 127 && g->pad_w <= 127 && g->stride_h <= 8 && g->stride_w <= 8 &&
      g->pad_h - (g->kh - 1) * g->dil_h >= -128 && g->pad_w - (g->kw - 1) * g->dil_w >= -128 &&
      (g->kw - 1) * g->dil_w < 65536 && (g->kh - 1) * g->dil_h < 65536 && g->n * g->h * g->w < (int64_t(1) << 31)) {
    mb->i2c = true;
    mb->Mst = g->n * g->h * g->w;
    mb->ig = Im2colGeom{int32_t(g->c), g->kw, g->kh * g->kw, Wo, Ho * Wo, int32_t(g->n), g->stride_w, g->stride_h,
                        g->pad_w, g->pad_h, g->dil_w, g->dil_h};
  }
  // every K slice must be non-empty: reduce_pack_kernel sums all `splits` partial slots, and
  // an empty slice would leave its (uninitialised) slot unwritten.  With per = cdiv(nkb, s),
  // cdiv(nkb, per) slices of `per` blocks cover nkb and the last one holds >= 1 block.
  const int64_t nkb = mb->Mpad / 64, per = cdiv(nkb, int64_t(mb->splits));
  mb->splits = int(cdiv(nkb, per));
  return SPDKFAC_OK;
}

// carve one group's workspace (c.base == nullptr: size only)
void group_carve(spdkfac_factor_group* G, Carve& c) {
  int items = 0, pitems = 0, jobs = 0;
  int f32 = 0;
  for (Member& mb : G->m) {
    if (mb.f32 && f32 == kMaxF32Maps) mb.f32 = false;  // the launch carries at most kMaxF32Maps row maps
    mb.xt = mb.f32 ? nullptr : c.take<__nv_bfloat16>(size_t(2) * (mb.i2c ? mb.Mst * mb.g.c : mb.M * mb.ld));
    mb.f32_slot = mb.f32 ? f32++ : -1;
    if (mb.splits > 1) {
      mb.partial = c.take<float>(size_t(mb.n_tiles) * mb.splits * 16384);
      mb.chunks = c.take<float>(size_t(mb.n_tiles) * 16 * cdiv(mb.splits, kChunk) * 1024);
      mb.counters = c.take<int>(size_t(mb.n_tiles) * 16);
      jobs += mb.n_tiles;
    } else {
      mb.partial = nullptr, mb.chunks = nullptr, mb.counters = nullptr;
    }
    if (mb.S)
      pitems += mb.S * (mb.S + 1) / 2 * mb.splits;
    else
      items += mb.n_tiles * mb.splits;
  }
  const size_t n = G->m.size();
  G->maps = c.take<CUtensorMap>(2 * n, 128);  // member k: [2k] (im2col members: [2k] hi, [2k + 1] lo plane)
  G->i2c = c.take<Im2colGeom>(2 * n);
  G->items = c.take<TcItem>(size_t(std::max(items, 1)));
  G->pitems = c.take<TcPairItem>(size_t(std::max(pitems, 1)));
  G->epis = c.take<TcEpi>(n);
  G->jobs = c.take<RedJob>(size_t(std::max(jobs, 1)));
  G->rmem = c.take<RedMember>(n);
  G->n_items = items;
  G->n_pitems = pitems;
  G->n_jobs = jobs;
}

int group_build(spdkfac_factor_group* G, float* const* packed, const float* scales, cudaStream_t s) {
  const int n = int(G->m.size());
  std::vector<CUtensorMap> maps(2 * size_t(n));
  std::vector<Im2colGeom> geo(2 * size_t(n));
  std::vector<TcItem> items;
  std::vector<TcPairItem> pitems;
  std::vector<TcEpi> epis(n);
  std::vector<RedJob> jobs;
  std::vector<RedMember> rmem(n);
  G->max_chunks = 1;
  G->flops = 0;
  G->flops_single = G->flops_pair = 0;
  for (int k = 0; k < n; ++k) {
    Member& mb = G->m[k];
    if (mb.i2c) {  // one im2col map per staged activation plane
      const spdkfac_factor_geom& g = mb.g;
      for (int p = 0; p < 2; ++p) {
        int rc = make_im2col_map_bf16(&maps[2 * k + p], mb.xt + size_t(p) * mb.Mst * g.c, int(g.n), int(g.h),
                                      int(g.w), int(g.c), g.kh, g.kw, g.stride_h, g.stride_w, g.pad_h, g.pad_w,
                                      g.dil_h, g.dil_w);
        if (rc) return rc;
      }
      geo[2 * k] = mb.ig;
    } else if (!mb.f32) {  // staged bf16 planes (fp32-rows members get their map at compute time)
      int rc = make_operand_map_mn(&maps[2 * k], mb.xt, mb.ld, mb.M);
      if (rc) return rc;
    } else {
      SPD_ARG(mb.f32_slot < kMaxF32Maps, SPDKFAC_ERR_ARG, "too many fp32-rows members in one factor group (%d)",
              mb.f32_slot + 1);
      std::memset(&maps[2 * k], 0, sizeof(CUtensorMap));
    }
    G->flops += double(mb.M) * mb.d * (mb.d + 1);
    (mb.S ? G->flops_pair : G->flops_single) += double(mb.M) * mb.d * (mb.d + 1);
    const int64_t nkb = mb.Mpad / 64, per = cdiv(nkb, mb.splits);
    auto tile_index = [&](int I, int J) { return I * mb.T - I * (I - 1) / 2 + (J - I); };
    for (int I = 0; I < mb.T; ++I)
      for (int J = I; J < mb.T; ++J)
        if (mb.splits > 1) jobs.push_back(RedJob{k, tile_index(I, J), I, J});
    for (int s2 = 0; s2 < mb.splits; ++s2) {
      const int64_t kb0 = std::min<int64_t>(nkb, s2 * per), kb1 = std::min<int64_t>(nkb, (s2 + 1) * per);
      if (kb1 <= kb0) continue;
      // target of block tile (I, J): partial slot (split K) or packed-upper position
      auto out_of = [&](int I, int J, int32_t& out_r, int32_t& out_c) {
        if (mb.splits > 1) {
          out_r = 0;
          out_c = (tile_index(I, J) * mb.splits + s2) * 128;
        } else {
          out_r = I * 128;
          out_c = J * 128;
        }
      };
      auto valid = [&](int I) { return int(std::min<int64_t>(128, mb.d - int64_t(I) * 128)); };
      if (mb.S) {
        for (int P = 0; P < mb.S; ++P)
          for (int Q = P; Q < mb.S; ++Q) {
            TcPairItem it{};
            it.map = 2 * k;
            it.a_row = 2 * P * 128;
            it.b_row = 2 * Q * 128;
            it.k0 = int(kb0 * 64);
            it.nk = int(kb1 - kb0);
            it.epi = k;
            it.flags = (P == Q) ? kSameAB : 0;
            for (int r = 0; r < 2; ++r) {
              const int I = 2 * P + r;
              it.m_valid[r] = I < mb.T ? valid(I) : 0;
              it.n_valid[r] = (2 * Q + r) < mb.T ? valid(2 * Q + r) : 0;
              for (int h = 0; h < 2; ++h) {
                const int J = 2 * Q + h;
                int32_t orr = 0, occ = -1;
                if (I < mb.T && J < mb.T && I <= J) out_of(I, J, orr, occ);
                if (occ >= 0) it.out_r[r] = orr;
                it.out_c[2 * r + h] = occ;
              }
            }
            pitems.push_back(it);
          }
      } else {
        for (int I = 0; I < mb.T; ++I)
          for (int J = I; J < mb.T; ++J) {
            TcItem it{};
            it.a_map = mb.f32 ? mb.f32_slot : 2 * k;
            it.b_map = mb.f32 ? mb.f32_slot : 2 * k;
            it.a_row = I * 128;
            it.b_row = J * 128;
            it.k0 = int(kb0 * 64);
            it.nk = int(kb1 - kb0) * (mb.f32 ? 2 : 1);  // fp32-rows stages hold 32 K rows
            it.epi = k;
            it.flags = (mb.f32 ? kF32Rows : kMnMajor) | (mb.i2c ? kIm2col : 0) | (I == J ? kSameAB : 0);
            out_of(I, J, it.out_r, it.out_c);
            it.m_valid = valid(I);
            it.n_valid = valid(J);
            items.push_back(it);
          }
      }
    }
    if (mb.splits > 1) {
      epis[k] = TcEpi{mb.partial, 128, 0, 1.f, 0.f, kAxpby, 0, nullptr, 0, 0};
      G->max_chunks = std::max<int>(G->max_chunks, int(cdiv(mb.splits, kChunk)));
    } else {  // packed target: from the epilogue table (group) or the run arguments (single plan)
      epis[k] = TcEpi{packed ? packed[k] : nullptr, mb.d, 0, scales ? scales[k] : 1.f, 0.f, kPackedUpper, 0,
                      nullptr, 0, 0};
    }
    rmem[k] = RedMember{mb.partial, mb.chunks, mb.counters, packed ? packed[k] : nullptr, mb.d, mb.T, mb.splits,
                        scales ? scales[k] : 1.f, 0};
    if (mb.counters) SPD_CUDA(cudaMemsetAsync(mb.counters, 0, sizeof(int) * size_t(mb.n_tiles) * 16, s));
  }
  // persistent CTAs take items round-robin: longest K first balances the group
  std::stable_sort(items.begin(), items.end(), [](const TcItem& a, const TcItem& b) { return a.nk > b.nk; });
  std::stable_sort(pitems.begin(), pitems.end(),
                   [](const TcPairItem& a, const TcPairItem& b) { return a.nk > b.nk; });
  G->n_items = int(items.size());
  G->n_pitems = int(pitems.size());
  int rc;
  if ((rc = upload(G->maps, maps, s)) || (rc = upload(G->i2c, geo, s)) || (rc = upload(G->items, items, s)) ||
      (rc = upload(G->pitems, pitems, s)) ||
      (rc = upload(G->epis, epis, s)) ||
      (rc = upload(G->jobs, jobs, s)) || (rc = upload(G->rmem, rmem, s)))
    return rc;
  return SPDKFAC_OK;
}

int member_stage(Member& mb, const float* x, cudaStream_t s) {
  const spdkfac_factor_geom& g = mb.g;
  if (mb.deferred && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {  // staged by the group's compute
    mb.x = x;
    return SPDKFAC_OK;
  }
  mb.x = nullptr;  // (an unaligned input of a deferred member is staged right here)
  if (mb.f32) {  // the SYRK reads x itself: bind it (x must stay valid until compute() has run)
    SPD_ARG((reinterpret_cast<uintptr_t>(x) & 15) == 0, SPDKFAC_ERR_ARG, "factor input must be 16-byte aligned");
    mb.x = x;
    return SPDKFAC_OK;
  }
  Probe* pr = stat_begin(kCatFactorStage, s);
  const bool pointwise = g.layout == SPDKFAC_CONV_A_NHWC && g.kh == 1 && g.kw == 1 && g.stride_h == 1 &&
                         g.stride_w == 1 && g.pad_h == 0 && g.pad_w == 0;
  if (mb.i2c) {  // the activation itself, [N*H*W][C] -> [2][N*H*W][C]: the SYRK gathers im2col tiles by TMA
    const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const RowShape rs = row_shape(mb.Mst, g.c / (vec ? 4 : 2), kStageRows);
    if (vec)
      stage_rows_kernel<true><<<rs.grid, rs.threads, 0, s>>>(x, mb.Mst, g.c, g.c, mb.xt, g.c, rs.tpr, rs.cps, pr);
    else
      stage_rows_kernel<false><<<rs.grid, rs.threads, 0, s>>>(x, mb.Mst, g.c, g.c, mb.xt, g.c, rs.tpr, rs.cps, pr);
  } else if (g.layout == SPDKFAC_ROWS || g.layout == SPDKFAC_SPATIAL_NHWC || pointwise) {
    // linear inputs [n][w] (row stride w); channels-last output gradients [b*h*w][C] and the
    // inputs of channels-last 1x1 stride-1 convs: rows [b*h*w][C]
    const int64_t ldx = g.layout == SPDKFAC_ROWS ? g.w : g.c;
    const bool vec = ldx % 4 == 0 && mb.d % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const bool vec8 = vec && mb.d % 8 == 0;
    const RowShape rs = row_shape(mb.M, mb.ld / (vec8 ? 8 : vec ? 4 : 2), kStageRows);
    if (vec8)
      stage_rows_kernel<true, true><<<rs.grid, rs.threads, 0, s>>>(x, mb.M, mb.d, ldx, mb.xt, mb.ld, rs.tpr, rs.cps,
                                                                   pr);
    else if (vec)
      stage_rows_kernel<true><<<rs.grid, rs.threads, 0, s>>>(x, mb.M, mb.d, ldx, mb.xt, mb.ld, rs.tpr, rs.cps, pr);
    else
      stage_rows_kernel<false><<<rs.grid, rs.threads, 0, s>>>(x, mb.M, mb.d, ldx, mb.xt, mb.ld, rs.tpr, rs.cps, pr);
  } else if (g.layout == SPDKFAC_CONV_A_NHWC || g.layout == SPDKFAC_CONV_A) {
    ConvGeom cg{int(g.n), int(g.c), int(g.h), int(g.w), mb.Ho, mb.Wo, g.kh, g.kw, g.stride_h, g.stride_w,
                g.pad_h, g.pad_w, g.dil_h, g.dil_w};
    const bool vec = g.layout == SPDKFAC_CONV_A_NHWC && g.c % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const bool vec8 = vec && g.c % 8 == 0;  // 8 channels of one tap per slot, 16-B stores
    const int64_t ncol = mb.ld / (vec8 ? 8 : vec ? 4 : 2);
    const RowShape rs = row_shape(mb.M, ncol, kIm2colRows);
    if (g.layout == SPDKFAC_CONV_A_NHWC) {
      if (vec8)
        stage_im2col_kernel<true, true, true><<<rs.grid, rs.threads, 0, s>>>(x, cg, mb.M, mb.d, mb.xt, mb.ld, rs.tpr,
                                                                            rs.cps, pr);
      else if (vec)
        stage_im2col_kernel<true, true><<<rs.grid, rs.threads, 0, s>>>(x, cg, mb.M, mb.d, mb.xt, mb.ld, rs.tpr, rs.cps, pr);
      else
        stage_im2col_kernel<true, false><<<rs.grid, rs.threads, 0, s>>>(x, cg, mb.M, mb.d, mb.xt, mb.ld, rs.tpr,
                                                                        rs.cps, pr);
    } else {
      stage_im2col_kernel<false, false><<<rs.grid, rs.threads, 0, s>>>(x, cg, mb.M, mb.d, mb.xt, mb.ld, rs.tpr,
                                                                        rs.cps, pr);
    }
  } else {
    const int hw = int(g.h * g.w);
    dim3 grid(unsigned(cdiv(hw, 32)), unsigned(cdiv(mb.ld, 32)), unsigned(g.n));
    stage_spatial_kernel<<<grid, 256, 0, s>>>(x, int(g.c), hw, mb.xt, mb.M, mb.ld, pr);
  }
  SPD_CHECK_LAUNCH();
  stat_end(kCatFactorStage, s, 0, double(mb.M) * mb.d * 4 + 4.0 * mb.ld * mb.M);
  return SPDKFAC_OK;
}

int group_compute(spdkfac_factor_group* G, float scale, float decay, float world_scale, float* packed,
                  cudaStream_t s) {
  // algorithmic work: sum over members of M * d * (d + 1) flops
  TcRun run{packed, G->m.empty() ? 0 : G->m[0].d, scale, decay, world_scale, 0};
  run.i2c = G->i2c;
  double bytes_single = 0, bytes_pair = 0;
  for (const Member& mb : G->m) (mb.S ? bytes_pair : bytes_single) += 4.0 * (mb.f32 ? mb.d : mb.ld) * mb.M;
  int rc;
  {  // deferred row staging: every such member of the group in one launch per kBatchStageMax members
    StageBatch sb{};
    double sbytes = 0;
    auto flush = [&]() {
      if (sb.n == 0) return;
      sb.blk0[sb.n] = sb.blk0[sb.n - 1] + int(cdiv(sb.M[sb.n - 1], kStageRows));
      Probe* pr = stat_begin(kCatFactorStage, s);
      stage_rows_batched_kernel<<<sb.blk0[sb.n], 256, 0, s>>>(sb, pr);
      stat_end(kCatFactorStage, s, 0, sbytes);
      sb.n = 0, sbytes = 0;
    };
    for (Member& mb : G->m) {
      if (!mb.deferred || !mb.x) continue;
      if (sb.n == kBatchStageMax) flush();
      const int t = sb.n;
      sb.x[t] = mb.x, sb.xs[t] = mb.xt, sb.M[t] = mb.M, sb.ldx[t] = mb.ldx, sb.ld[t] = mb.ld;
      sb.d[t] = int32_t(mb.d);
      sb.blk0[t] = t == 0 ? 0 : sb.blk0[t - 1] + int(cdiv(sb.M[t - 1], kStageRows));
      sbytes += 8.0 * double(mb.M) * mb.d;
      ++sb.n;
      mb.x = nullptr;  // consumed: the next compute needs a new stage()
    }
    flush();
    SPD_CHECK_LAUNCH();
  }
  if (G->n_items) {
    bool any_f32 = false;
    for (const Member& mb : G->m) any_f32 |= mb.f32;
    if (any_f32) {  // fp32 row maps of this run's activations, passed by value with the launch
      F32Maps fm;  // the launch copies it into the kernel parameters
      for (const Member& mb : G->m) {
        if (!mb.f32) continue;
        SPD_ARG(mb.x != nullptr, SPDKFAC_ERR_ARG, "factor member computed before its input was staged");
        if ((rc = make_rows_map_f32(&fm.m[mb.f32_slot], mb.x, mb.M, mb.d, mb.ldx))) return rc;
      }
      run.probe = stat_begin(kCatFactorSyrk, s);
      if ((rc = launch_tc3_f32(G->maps, G->items, G->epis, G->n_items, s, run, fm))) return rc;
    } else {
      run.probe = stat_begin(kCatFactorSyrk, s);
      if ((rc = launch_tc3(Kind::BF16, G->maps, G->items, G->epis, G->n_items, s, run))) return rc;
    }
    stat_end(kCatFactorSyrk, s, G->flops_single, bytes_single);
  }
  if (G->n_pitems) {
    run.probe = stat_begin(kCatFactorSyrk, s);
    if ((rc = launch_tc3_pair(G->maps, G->pitems, G->epis, G->n_pitems, s, run))) return rc;
    stat_end(kCatFactorSyrk, s, G->flops_pair, bytes_pair);
  }
  if (G->n_jobs == 0) return SPDKFAC_OK;
  dim3 rgrid(16, unsigned(G->n_jobs), unsigned(G->max_chunks));
  stat_begin(kCatFactorReduce, s);
  reduce_pack_kernel<<<rgrid, 256, 0, s>>>(G->jobs, G->rmem, decay, world_scale,
                                           G->per_run_target ? packed : nullptr,
                                           G->per_run_target ? scale : -1.f);
  SPD_CHECK_LAUNCH();
  stat_end(kCatFactorReduce, s, 0, 0);
  return SPDKFAC_OK;
}

}  // namespace

extern "C" {

int spdkfac_factor_dims(const spdkfac_factor_geom* g, int64_t* rows, int64_t* dim) {
  return geom_dims(g, rows, dim);
}

size_t spdkfac_factor_workspace_size(const spdkfac_factor_geom* g) {
  spdkfac_factor_group G;
  G.m.resize(1);
  if (member_init(&G.m[0], g) != SPDKFAC_OK) return 0;
  Carve c(nullptr, 0);
  group_carve(&G, c);
  return c.used + 256;
}

int spdkfac_factor_plan_create(spdkfac_factor_plan** out, const spdkfac_factor_geom* g, void* ws, size_t ws_bytes,
                               void* stream) {
  SPD_ARG(out != nullptr, SPDKFAC_ERR_ARG, "null plan out");
  auto* p = new spdkfac_factor_plan();
  p->m.resize(1);
  int rc = member_init(&p->m[0], g);
  if (rc) {
    delete p;
    return rc;
  }
  Carve c(ws, ws_bytes);
  group_carve(p, c);
  if (!c.ok() || ws == nullptr) {
    delete p;
    set_error("factor workspace too small: need %zu bytes, got %zu", c.used, ws_bytes);
    return SPDKFAC_ERR_ARG;
  }
  p->per_run_target = true;
  if ((rc = group_build(p, nullptr, nullptr, static_cast<cudaStream_t>(stream)))) {
    delete p;
    return rc;
  }
  *out = p;
  return SPDKFAC_OK;
}

int spdkfac_factor_plan_stage(spdkfac_factor_plan* p, const float* x, void* stream) {
  SPD_ARG(p && x, SPDKFAC_ERR_ARG, "null argument");
  return member_stage(p->m[0], x, static_cast<cudaStream_t>(stream));
}

int spdkfac_factor_plan_compute(spdkfac_factor_plan* p, float scale, float decay, float world_scale, float* packed,
                                void* stream) {
  SPD_ARG(p && packed, SPDKFAC_ERR_ARG, "null argument");
  return group_compute(p, scale, decay, world_scale, packed, static_cast<cudaStream_t>(stream));
}

int spdkfac_factor_plan_run(spdkfac_factor_plan* p, const float* x, float scale, float decay, float world_scale,
                            float* packed, void* stream) {
  int rc = spdkfac_factor_plan_stage(p, x, stream);
  if (rc) return rc;
  return spdkfac_factor_plan_compute(p, scale, decay, world_scale, packed, stream);
}

void spdkfac_factor_plan_destroy(spdkfac_factor_plan* p) { delete p; }

size_t spdkfac_factor_group_workspace_size(int n, const spdkfac_factor_geom* geoms) {
  if (n < 1 || !geoms) return 0;
  spdkfac_factor_group G;
  G.m.resize(n);
  for (int k = 0; k < n; ++k)
    if (member_init(&G.m[k], &geoms[k]) != SPDKFAC_OK) return 0;
  Carve c(nullptr, 0);
  group_carve(&G, c);
  return c.used + 256;
}

int spdkfac_factor_group_create(spdkfac_factor_group** out, int n, const spdkfac_factor_geom* geoms,
                                float* const* packed_out, const float* scales, void* ws, size_t ws_bytes,
                                void* stream) {
  SPD_ARG(out && n >= 1 && geoms && packed_out && scales, SPDKFAC_ERR_ARG, "bad factor group arguments");
  auto* G = new spdkfac_factor_group();
  G->m.resize(n);
  int rc;
  for (int k = 0; k < n; ++k)
    if ((rc = member_init(&G->m[k], &geoms[k]))) {
      delete G;
      return rc;
    }
  Carve c(ws, ws_bytes);
  group_carve(G, c);
  if (!c.ok() || ws == nullptr) {
    delete G;
    set_error("factor group workspace too small: need %zu bytes, got %zu", c.used, ws_bytes);
    return SPDKFAC_ERR_ARG;
  }
  if ((rc = group_build(G, packed_out, scales, static_cast<cudaStream_t>(stream)))) {
    delete G;
    return rc;
  }
  *out = G;
  return SPDKFAC_OK;
}

int spdkfac_factor_group_stage(spdkfac_factor_group* G, int member, const float* x, void* stream) {
  SPD_ARG(G && x && member >= 0 && member < int(G->m.size()), SPDKFAC_ERR_ARG, "bad factor group stage arguments");
  return member_stage(G->m[member], x, static_cast<cudaStream_t>(stream));
}

int spdkfac_factor_group_compute(spdkfac_factor_group* G, float decay, float world_scale, void* stream) {
  SPD_ARG(G != nullptr, SPDKFAC_ERR_ARG, "null factor group");
  return group_compute(G, 1.f, decay, world_scale, nullptr, static_cast<cudaStream_t>(stream));
}

void spdkfac_factor_group_destroy(spdkfac_factor_group* G) { delete G; }

int spdkfac_factor_group_describe(const spdkfac_factor_group* G, int member, int64_t out[4]) {
  SPD_ARG(G && out && member >= 0 && member < int(G->m.size()), SPDKFAC_ERR_ARG, "bad describe arguments");
  const Member& mb = G->m[member];
  out[0] = mb.S ? 1 : (mb.f32 ? 2 : (mb.i2c ? 3 : 0)), out[1] = mb.splits, out[2] = mb.M, out[3] = mb.d;
  return SPDKFAC_OK;
}

}  // extern "C"
