// Kronecker-factor construction: X^T X over rows (linear), im2col patches (conv A)
// or spatial output-gradient rows (conv G), on tcgen05 with 3 x bf16 split operands.
//
// Pipeline per factor (one plan = one layer-side):
//   1. stage kernel  : gather rows of X into the K-major split operand Xt[2][d][Mpad] (bf16 hi/lo)
//                      -- the im2col / layout transform and the precision split in one HBM pass
//   2. tc3 GEMM      : upper-triangle 128x128 tiles (I <= J) x split-K slices, partial tiles to ws
//   3. reduce + pack : sum split-K partials in fixed order, apply 1/M, running average, 1/P,
//                      write the packed upper triangle (the all-reduce / fusion-buffer format)
#include <algorithm>

#include "runtime.cuh"

namespace spd {

// ------------------------------------------------------------------ staging kernels
// Xt[r][m] (r < d, m < Mpad) ; planes hi at 0, lo at d*Mpad.  Zero for m >= M.

__device__ __forceinline__ void store_split2(__nv_bfloat16* xt, int64_t plane, int64_t o, float v0, float v1);

// [M][d] rows (row stride ldx) -> K-major split planes Xt[2][d][Mpad].  64(m) x 32(r) tiles
// through shared memory: 128-B reads along r, bf16x2 (128-B per warp) writes along m.
__global__ void __launch_bounds__(256) stage_rows_kernel(const float* __restrict__ x, int64_t M, int64_t d,
                                                         int64_t ldx, __nv_bfloat16* __restrict__ xt, int64_t Mpad) {
  __shared__ float tile[64][33];
  const int64_t m0 = int64_t(blockIdx.x) * 64, r0 = int64_t(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
  for (int k = ty; k < 64; k += 8) {
    const int64_t m = m0 + k, r = r0 + tx;
    tile[k][tx] = (m < M && r < d) ? __ldg(x + m * ldx + r) : 0.f;
  }
  __syncthreads();
  const int64_t plane = d * Mpad;
#pragma unroll
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + k, m = m0 + 2 * tx;
    if (r < d && m < Mpad) store_split2(xt, plane, r * Mpad + m, tile[2 * tx][k], tile[2 * tx + 1][k]);
  }
}

struct ConvGeom {
  int B, C, H, W, Ho, Wo, kh, kw, sh, sw, ph, pw, dh, dw;
};

__device__ __forceinline__ void store_split2(__nv_bfloat16* xt, int64_t plane, int64_t o, float v0, float v1) {
  __nv_bfloat16 h0, l0, h1, l1;
  split_bf16(v0, h0, l0);
  split_bf16(v1, h1, l1);
  *reinterpret_cast<__nv_bfloat162*>(xt + o) = __halves2bfloat162(h0, h1);
  *reinterpret_cast<__nv_bfloat162*>(xt + plane + o) = __halves2bfloat162(l0, l1);
}

// One block per (patch row r = (c, ki, kj), image b): threads walk the output positions of
// image b two at a time (bf16x2 stores), 32-bit index math, one division per pair.
__global__ void __launch_bounds__(256) stage_im2col_kernel(const float* __restrict__ x, ConvGeom g, int64_t M,
                                                           int64_t d, __nv_bfloat16* __restrict__ xt, int64_t Mpad) {
  const int r = blockIdx.y;
  const int b = blockIdx.x;
  const int kj = r % g.kw, ki = (r / g.kw) % g.kh, c = r / (g.kw * g.kh);
  const int HWo = g.Ho * g.Wo;
  const int64_t plane = d * Mpad;
  const int64_t row = int64_t(r) * Mpad + int64_t(b) * HWo;  // m = b*HWo + hw
  const float* xc = x + (int64_t(b) * g.C + c) * g.H * g.W;
  const int hoff = ki * g.dh - g.ph, woff = kj * g.dw - g.pw;
  // HWo may be odd (7x7): pair (hw, hw+1) when both in range, row offsets are then even
  // only if b*HWo is even; fall back to scalar stores otherwise.
  const bool vec = ((int64_t(b) * HWo) & 1) == 0 && (Mpad & 1) == 0;
  if (vec) {
    for (int hw = 2 * threadIdx.x; hw < HWo; hw += 2 * blockDim.x) {
      float v[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int q = hw + u;
        v[u] = 0.f;
        if (q < HWo) {
          const int ho = q / g.Wo, wo = q - ho * g.Wo;
          const int hi = ho * g.sh + hoff, wi = wo * g.sw + woff;
          if (hi >= 0 && hi < g.H && wi >= 0 && wi < g.W) v[u] = __ldg(xc + hi * g.W + wi);
        }
      }
      if (hw + 1 < HWo) {
        store_split2(xt, plane, row + hw, v[0], v[1]);
      } else {
        __nv_bfloat16 h, l;
        split_bf16(v[0], h, l);
        xt[row + hw] = h;
        xt[plane + row + hw] = l;
      }
    }
  } else {
    for (int q = threadIdx.x; q < HWo; q += blockDim.x) {
      const int ho = q / g.Wo, wo = q - ho * g.Wo;
      const int hi = ho * g.sh + hoff, wi = wo * g.sw + woff;
      float v = 0.f;
      if (hi >= 0 && hi < g.H && wi >= 0 && wi < g.W) v = __ldg(xc + hi * g.W + wi);
      __nv_bfloat16 h, l;
      split_bf16(v, h, l);
      xt[row + q] = h;
      xt[plane + row + q] = l;
    }
  }
}

// channels-last input x[b][h][w][c]; patch rows ordered (ki, kj, c) -- the column order of a
// channels-last conv weight viewed as [cout][kh*kw*cin].  32(m) x 32(c) tiles through shared
// memory: reads coalesced along c, bf16x2 hi/lo writes coalesced along m.
__global__ void __launch_bounds__(256) stage_im2col_nhwc_kernel(const float* __restrict__ x, ConvGeom g, int64_t M,
                                                                int64_t d, __nv_bfloat16* __restrict__ xt,
                                                                int64_t Mpad) {
  __shared__ float tile[64][33];
  __shared__ int rowoff[64];  // element offset of (b, hi, wi, 0) for the block's 64 rows, -1 = padding
  const int kk = blockIdx.z, ki = kk / g.kw, kj = kk - ki * g.kw;
  const uint32_t m0 = blockIdx.x * 64u;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  if (threadIdx.x < 64) {
    const uint32_t m = m0 + threadIdx.x;
    int off = -1;
    if (m < uint32_t(M)) {
      const uint32_t HWo = uint32_t(g.Ho) * g.Wo;
      const uint32_t b = m / HWo, q = m - b * HWo;
      const uint32_t ho = q / uint32_t(g.Wo), wo = q - ho * g.Wo;
      const int hi = int(ho) * g.sh - g.ph + ki * g.dh, wi = int(wo) * g.sw - g.pw + kj * g.dw;
      if (hi >= 0 && hi < g.H && wi >= 0 && wi < g.W) off = ((int(b) * g.H + hi) * g.W + wi) * g.C;
    }
    rowoff[threadIdx.x] = off;
  }
  __syncthreads();
  const int c = c0 + tx;
#pragma unroll
  for (int r = ty; r < 64; r += 8) {
    const int off = rowoff[r];
    tile[r][tx] = (off >= 0 && c < g.C) ? __ldg(x + off + c) : 0.f;
  }
  __syncthreads();
  const int64_t plane = d * Mpad;
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int cc = c0 + r;
    const int64_t m = int64_t(m0) + 2 * tx;
    if (cc < g.C && m < Mpad)
      store_split2(xt, plane, (int64_t(kk) * g.C + cc) * Mpad + m, tile[2 * tx][r], tile[2 * tx + 1][r]);
  }
}

// channels-last im2col for few input channels (the stem conv: C = 3): one thread per pair of
// output positions walks all (ki, kj, c) patch rows; bf16x2 stores stay coalesced along m and
// the overlapping patch reads are served by L1.
__global__ void __launch_bounds__(256) stage_im2col_nhwc_smallc_kernel(const float* __restrict__ x, ConvGeom g,
                                                                       int64_t M, int64_t d,
                                                                       __nv_bfloat16* __restrict__ xt, int64_t Mpad) {
  const int64_t m = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
  if (m >= Mpad) return;
  const uint32_t HWo = uint32_t(g.Ho) * g.Wo;
  int hb[2], wb[2], bo[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const uint32_t mm = uint32_t(m) + u;
    if (mm < uint32_t(M)) {
      const uint32_t b = mm / HWo, q = mm - b * HWo;
      const uint32_t ho = q / uint32_t(g.Wo), wo = q - ho * g.Wo;
      bo[u] = int(b) * g.H;
      hb[u] = int(ho) * g.sh - g.ph;
      wb[u] = int(wo) * g.sw - g.pw;
    } else {
      bo[u] = -1, hb[u] = 0, wb[u] = 0;
    }
  }
  const int64_t plane = d * Mpad;
  for (int ki = 0; ki < g.kh; ++ki)
    for (int kj = 0; kj < g.kw; ++kj) {
      int off[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int hi = hb[u] + ki * g.dh, wi = wb[u] + kj * g.dw;
        off[u] = (bo[u] >= 0 && hi >= 0 && hi < g.H && wi >= 0 && wi < g.W) ? ((bo[u] + hi) * g.W + wi) * g.C : -1;
      }
      const int64_t row0 = int64_t(ki * g.kw + kj) * g.C;
      for (int c = 0; c < g.C; ++c) {
        const float v0 = off[0] >= 0 ? __ldg(x + off[0] + c) : 0.f;
        const float v1 = off[1] >= 0 ? __ldg(x + off[1] + c) : 0.f;
        store_split2(xt, plane, (row0 + c) * Mpad + m, v0, v1);
      }
    }
}

// rows m = (b, hw) of channel c: a contiguous copy of g[b][c][:] per image
__global__ void __launch_bounds__(256) stage_spatial_kernel(const float* __restrict__ g, int C, int HW,
                                                            __nv_bfloat16* __restrict__ xt, int64_t Mpad) {
  const int c = blockIdx.y, b = blockIdx.x;
  const int64_t plane = int64_t(C) * Mpad;
  const float* src = g + (int64_t(b) * C + c) * HW;
  const int64_t row = int64_t(c) * Mpad + int64_t(b) * HW;
  if (((int64_t(b) * HW) & 1) == 0 && (HW & 1) == 0) {
    for (int q = 2 * threadIdx.x; q < HW; q += 2 * blockDim.x) {
      const float2 v = *reinterpret_cast<const float2*>(src + q);
      store_split2(xt, plane, row + q, v.x, v.y);
    }
  } else {
    for (int q = threadIdx.x; q < HW; q += blockDim.x) {
      __nv_bfloat16 h, l;
      split_bf16(src[q], h, l);
      xt[row + q] = h;
      xt[plane + row + q] = l;
    }
  }
}

// zero the K padding columns [M, Mpad) of every row (once per plan; never written by staging)
__global__ void zero_pad_kernel(__nv_bfloat16* xt, int64_t d, int64_t M, int64_t Mpad) {
  const int64_t r = blockIdx.x;
  for (int64_t m = M + threadIdx.x; m < Mpad; m += blockDim.x) {
    xt[r * Mpad + m] = __float2bfloat16(0.f);
    xt[d * Mpad + r * Mpad + m] = __float2bfloat16(0.f);
  }
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
  int64_t M, d, Mpad;
  int T, splits, n_tiles;
  int Ho, Wo;
  __nv_bfloat16* xt;
  float* partial;
  float* chunks;
  int* counters;
};

struct spdkfac_factor_group {
  std::vector<Member> m;
  CUtensorMap* maps = nullptr;
  TcItem* items = nullptr;
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

// splits: fill ~148 SMs per factor (the group launch then has >= that many items), each
// K slice >= 16 blocks (1024 rows); splits == 1 stores straight into the packed buffer
int choose_splits(int64_t Mpad, int n_tiles) {
  const int64_t nkb = Mpad / 64;
  const int64_t want = cdiv(148, n_tiles);
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
  mb->Mpad = round_up(M, 64);
  mb->T = int(cdiv(d, 128));
  mb->n_tiles = mb->T * (mb->T + 1) / 2;
  mb->splits = choose_splits(mb->Mpad, mb->n_tiles);
  return SPDKFAC_OK;
}

// carve one group's workspace (c.base == nullptr: size only)
void group_carve(spdkfac_factor_group* G, Carve& c) {
  int items = 0, jobs = 0;
  for (Member& mb : G->m) {
    mb.xt = c.take<__nv_bfloat16>(size_t(2) * mb.d * mb.Mpad);
    if (mb.splits > 1) {
      mb.partial = c.take<float>(size_t(mb.n_tiles) * mb.splits * 16384);
      mb.chunks = c.take<float>(size_t(mb.n_tiles) * 16 * cdiv(mb.splits, kChunk) * 1024);
      mb.counters = c.take<int>(size_t(mb.n_tiles) * 16);
      jobs += mb.n_tiles;
    } else {
      mb.partial = nullptr, mb.chunks = nullptr, mb.counters = nullptr;
    }
    items += mb.n_tiles * mb.splits;
  }
  const size_t n = G->m.size();
  G->maps = c.take<CUtensorMap>(n, 128);
  G->items = c.take<TcItem>(size_t(std::max(items, 1)));
  G->epis = c.take<TcEpi>(n);
  G->jobs = c.take<RedJob>(size_t(std::max(jobs, 1)));
  G->rmem = c.take<RedMember>(n);
  G->n_items = items;
  G->n_jobs = jobs;
}

int group_build(spdkfac_factor_group* G, float* const* packed, const float* scales, cudaStream_t s) {
  const int n = int(G->m.size());
  std::vector<CUtensorMap> maps(n);
  std::vector<TcItem> items;
  std::vector<TcEpi> epis(n);
  std::vector<RedJob> jobs;
  std::vector<RedMember> rmem(n);
  G->max_chunks = 1;
  G->flops = 0;
  for (int k = 0; k < n; ++k) {
    Member& mb = G->m[k];
    int rc = make_operand_map(&maps[k], mb.xt, true, mb.Mpad, mb.d, mb.Mpad);
    if (rc) return rc;
    G->flops += double(mb.M) * mb.d * (mb.d + 1);
    const int64_t nkb = mb.Mpad / 64, per = cdiv(nkb, mb.splits);
    for (int I = 0; I < mb.T; ++I)
      for (int J = I; J < mb.T; ++J) {
        const int tile_idx = I * mb.T - I * (I - 1) / 2 + (J - I);
        if (mb.splits > 1) jobs.push_back(RedJob{k, tile_idx, I, J});
        for (int s2 = 0; s2 < mb.splits; ++s2) {
          TcItem it{};
          it.a_map = k;
          it.b_map = k;
          it.a_row = I * 128;
          it.b_row = J * 128;
          const int64_t kb0 = std::min<int64_t>(nkb, s2 * per), kb1 = std::min<int64_t>(nkb, (s2 + 1) * per);
          it.k0 = int(kb0 * 64);
          it.nk = int(kb1 - kb0);
          it.epi = k;
          it.flags = (I == J) ? kSameAB : 0;
          if (mb.splits > 1) {  // partial tile -> member workspace slot, reduced by reduce_pack_kernel
            it.out_r = 0;
            it.out_c = (tile_idx * mb.splits + s2) * 128;
          } else {              // direct packed-upper epilogue
            it.out_r = I * 128;
            it.out_c = J * 128;
          }
          it.m_valid = int(std::min<int64_t>(128, mb.d - int64_t(I) * 128));
          it.n_valid = int(std::min<int64_t>(128, mb.d - int64_t(J) * 128));
          if (it.nk > 0) items.push_back(it);
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
    if (mb.Mpad > mb.M) {
      zero_pad_kernel<<<unsigned(mb.d), 64, 0, s>>>(mb.xt, mb.d, mb.M, mb.Mpad);
      SPD_CHECK_LAUNCH();
    }
    if (mb.counters) SPD_CUDA(cudaMemsetAsync(mb.counters, 0, sizeof(int) * size_t(mb.n_tiles) * 16, s));
  }
  // persistent CTAs take items round-robin: longest K first balances the group
  std::stable_sort(items.begin(), items.end(), [](const TcItem& a, const TcItem& b) { return a.nk > b.nk; });
  G->n_items = int(items.size());
  int rc;
  if ((rc = upload(G->maps, maps, s)) || (rc = upload(G->items, items, s)) || (rc = upload(G->epis, epis, s)) ||
      (rc = upload(G->jobs, jobs, s)) || (rc = upload(G->rmem, rmem, s)))
    return rc;
  return SPDKFAC_OK;
}

int member_stage(const Member& mb, const float* x, cudaStream_t s) {
  const spdkfac_factor_geom& g = mb.g;
  stat_begin(kCatFactorStage, s);
  if (g.layout == SPDKFAC_ROWS || g.layout == SPDKFAC_SPATIAL_NHWC) {
    // channels-last output gradients are rows [b*h*w][C]: the same transpose
    const int64_t ld = g.layout == SPDKFAC_ROWS ? g.w : g.c;
    dim3 grid(unsigned(cdiv(mb.Mpad, 64)), unsigned(cdiv(mb.d, 32)));
    stage_rows_kernel<<<grid, 256, 0, s>>>(x, mb.M, mb.d, ld, mb.xt, mb.Mpad);
  } else if (g.layout == SPDKFAC_CONV_A_NHWC || g.layout == SPDKFAC_CONV_A) {
    ConvGeom cg{int(g.n), int(g.c), int(g.h), int(g.w), mb.Ho, mb.Wo, g.kh, g.kw, g.stride_h, g.stride_w,
                g.pad_h, g.pad_w, g.dil_h, g.dil_w};
    if (g.layout == SPDKFAC_CONV_A_NHWC) {
      if (g.c < 16) {
        stage_im2col_nhwc_smallc_kernel<<<unsigned(cdiv(mb.Mpad, 512)), 256, 0, s>>>(x, cg, mb.M, mb.d, mb.xt,
                                                                                     mb.Mpad);
      } else {
        dim3 grid(unsigned(cdiv(mb.Mpad, 64)), unsigned(cdiv(g.c, 32)), unsigned(g.kh * g.kw));
        stage_im2col_nhwc_kernel<<<grid, 256, 0, s>>>(x, cg, mb.M, mb.d, mb.xt, mb.Mpad);
      }
    } else {
      const int hwo = mb.Ho * mb.Wo;
      dim3 grid(unsigned(g.n), unsigned(mb.d));
      stage_im2col_kernel<<<grid, hwo >= 512 ? 256 : (hwo >= 128 ? 64 : 32), 0, s>>>(x, cg, mb.M, mb.d, mb.xt,
                                                                                      mb.Mpad);
    }
  } else {
    const int hw = int(g.h * g.w);
    dim3 grid(unsigned(g.n), unsigned(mb.d));
    stage_spatial_kernel<<<grid, hw >= 512 ? 256 : (hw >= 128 ? 64 : 32), 0, s>>>(x, int(g.c), hw, mb.xt, mb.Mpad);
  }
  SPD_CHECK_LAUNCH();
  stat_end(kCatFactorStage, s, 0, double(mb.M) * mb.d * 4 + 4.0 * mb.d * mb.Mpad);
  return SPDKFAC_OK;
}

int group_compute(spdkfac_factor_group* G, float scale, float decay, float world_scale, float* packed,
                  cudaStream_t s) {
  // algorithmic work: sum over members of M * d * (d + 1) flops
  stat_begin(kCatFactorSyrk, s);
  TcRun run{packed, G->m.empty() ? 0 : G->m[0].d, scale, decay, world_scale, 0};
  int rc = launch_tc3(Kind::BF16, G->maps, G->items, G->epis, G->n_items, s, run);
  if (rc) return rc;
  double bytes = 0;
  for (const Member& mb : G->m) bytes += 4.0 * mb.d * mb.Mpad;
  stat_end(kCatFactorSyrk, s, G->flops, bytes);
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

}  // extern "C"
