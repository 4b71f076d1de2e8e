// Preconditioning + update, batched over layers:
//   P_l = G_l^-1 grad_l A_l^-1,   W_l -= alpha P_l
// as two tcgen05 3 x tf32 GEMMs per layer with K-major operands only (both inverses are
// symmetric, so they serve as their own transposes).  The operands are tf32 hi/lo split planes
// (|x - hi - lo| <= 2^-22 |x|): grad A^-1 cancels heavily when grad lies in the span of a
// rank-deficient factor (ResNet-50's fc: 32 rows, d_in = 2048, kappa(A + gamma I) ~ 2e4), and
// 3 x bf16 operands (2^-17) left 7e-4 there against the north-star 1e-4
// (tests/test_gpu_config_parity.py); 3 x tf32 is fp32-class:
//   GEMM1  D1[m][n] = sum_k grad[m][k] A^-1[n][k]         = (grad A^-1)[m][n]     -> stored as T^T[n][m] (split)
//   GEMM2  D2[n][m] = sum_k T^T[n][k] G^-1[m][k]         = (G^-1 grad A^-1)[m][n] -> stored as P[m][n]
// The transposed epilogue store is the coalesced direction of the 32x32b TMEM layout.
//
// fp16 planes (opt-in, SPDKFAC_PRECOND_F16=1; see precond_f16): every operand ROW r is stored as fp16
// hi / lo planes of x * s[r], s[r] a power of two with |x s[r]| <= 2^13 -- from the row's exact
// absolute maximum (gradient rows, full inverses) or, for packed SPD inverses, from the bound
// sqrt(a_rr * max_i a_ii) >= |a_rj|.  The epilogues divide D[i][j] by s_A[i] s_B[j] (exact).  T = grad
// A^-1 is split with per-row scales from the bound |T[m][n]| <= max_m ||grad[m,:]||_1 * max_k |A^-1[n,k]|.
// kind::f16 runs at 2.25x the tf32 rate on half the operand bytes; hi + lo keep 22 bits of every
// entry above 2^-16 of its row bound.
#include <algorithm>

#include "runtime.cuh"

namespace spd {

constexpr int kBK = 32;     // tf32 K elements per 128-B swizzle row (one K block of the tile engine)
constexpr int kLdAlign = 64;  // operand rows padded to 64 elements: whole K blocks for tf32 (32) and fp16 (64)

// SPDKFAC_PRECOND_F16=1: fp16 row-scaled planes.  Off by default (measured): preconditioning 1.18 vs
// 1.63 ms/step live, but the bench step is not faster (16.8 vs 16.5 ms: the two-pass row splits) and
// Inception-v4's rank-4 fc update error rises from 9.3e-5 to 1.1e-4, past the 1e-4 contract.
bool precond_f16() {
  const char* e = getenv("SPDKFAC_PRECOND_F16");
  return e && e[0] == '1';
}

// One block per operand row: row r of matrix t -> fp16 hi / lo planes of x * s, s from the row's
// absolute maximum; scale[t][r] = s, amax[t][r] = max |x| (optional), and the row's L1 norm folded into
// *l1max[t] (optional; atomicMax on the non-negative float's bits).
struct SplitArgs16 {
  const float* src[kMaxPtrs];
  __half* dst[kMaxPtrs];
  float* scale[kMaxPtrs];
  float* amax[kMaxPtrs];
  float* l1max[kMaxPtrs];
  int32_t cols[kMaxPtrs], ldd[kMaxPtrs];
  int64_t plane[kMaxPtrs];
  int32_t row0[kMaxPtrs + 1];
  int n;
};

__device__ __forceinline__ float block_reduce(float v, bool is_max, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, w) : v + w;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : (is_max ? 0.f : 0.f);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float w = __shfl_xor_sync(0xffffffffu, x, o);
      x = is_max ? fmaxf(x, w) : x + w;
    }
    if (threadIdx.x == 0) red[0] = x;
  }
  __syncthreads();
  const float r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) split_rows_f16_kernel(const __grid_constant__ SplitArgs16 a) {
  __shared__ float red[8];
  const int row = blockIdx.x;
  int lo = 0, hi = a.n - 1;
  while (lo < hi) {  // last t with row0[t] <= row
    const int mid = (lo + hi + 1) >> 1;
    if (a.row0[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  const int t = lo;
  const int64_t r = row - a.row0[t];
  const int cols = a.cols[t];
  const float* src = a.src[t] + r * cols;
  float mx = 0.f, l1 = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float x = fabsf(__ldg(src + c));
    mx = fmaxf(mx, x);
    l1 += x;
  }
  mx = block_reduce(mx, true, red);
  if (a.l1max[t]) l1 = block_reduce(l1, false, red);
  const float sc = f16_scale(mx);
  __half* d = a.dst[t] + r * a.ldd[t];
  const int64_t pl = a.plane[t];
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    __half h, l;
    split_f16(__ldcs(src + c), sc, h, l);
    d[c] = h;
    d[c + pl] = l;
  }
  if (threadIdx.x == 0) {
    a.scale[t][r] = sc;
    if (a.amax[t]) a.amax[t][r] = mx;
    if (a.l1max[t]) atomicMax(reinterpret_cast<int*>(a.l1max[t]), __float_as_int(l1));
  }
}

// Packed SPD inverses (the broadcast path): per-row bound sqrt(a_rr * max_i a_ii) >= |a_rj| from the
// diagonal, its scale and bound; one block per matrix
struct DiagArgs {
  const float* src[kMaxPtrs];
  float* scale[kMaxPtrs];
  float* amax[kMaxPtrs];
  int32_t d[kMaxPtrs];
  int n;
};
__global__ void __launch_bounds__(256) packed_row_bounds_kernel(const __grid_constant__ DiagArgs a) {
  __shared__ float red[8];
  const int t = blockIdx.x;
  const int64_t d = a.d[t];
  const float* p = a.src[t];
  float mx = 0.f;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) mx = fmaxf(mx, fabsf(p[i * (2 * d - i + 1) / 2]));
  mx = block_reduce(mx, true, red);
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
    const float b = sqrtf(fabsf(p[i * (2 * d - i + 1) / 2]) * mx) * 1.0001f;  // (rounding slack)
    a.scale[t][i] = f16_scale(b);
    if (a.amax[t]) a.amax[t][i] = b;
  }
}

struct SplitArgs {
  const float* src[kMaxPtrs];
  float* dst[kMaxPtrs];
  int32_t cols[kMaxPtrs], ldd[kMaxPtrs];
  int64_t plane[kMaxPtrs];
  int32_t row0[kMaxPtrs + 1];
  int n;
};

// One block per operand row: row r of matrix t -> tf32 hi/lo planes (fp32 storage).  Rows whose
// length and source/destination alignment allow it move as float4 loads and stores.
__global__ void __launch_bounds__(256) split_rows_batched_kernel(const __grid_constant__ SplitArgs a) {
  const int row = blockIdx.x;
  int lo = 0, hi = a.n - 1;
  while (lo < hi) {  // last t with row0[t] <= row
    const int mid = (lo + hi + 1) >> 1;
    if (a.row0[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  const int t = lo;
  const int64_t r = row - a.row0[t];
  const int cols = a.cols[t];
  const float* s = a.src[t] + r * cols;
  float* d = a.dst[t] + r * a.ldd[t];
  const int64_t pl = a.plane[t];
  const bool vec = (cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(s) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(d) & 15) == 0) && (pl % 4 == 0);
  if (vec) {
    const int n4 = cols >> 2;
    for (int c = threadIdx.x; c < n4; c += blockDim.x) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(s) + c);
      float4 h, l;
      split_tf32(v.x, h.x, l.x);
      split_tf32(v.y, h.y, l.y);
      split_tf32(v.z, h.z, l.z);
      split_tf32(v.w, h.w, l.w);
      reinterpret_cast<float4*>(d)[c] = h;
      reinterpret_cast<float4*>(d + pl)[c] = l;
    }
    return;
  }
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    float h, l;
    split_tf32(s[c], h, l);
    d[c] = h;
    d[c + pl] = l;
  }
}

// Received packed inverse -> full fp32 matrix (optional) AND the preconditioner's tf32 hi/lo
// operand planes, one 64 x 64 upper tile (I <= J) per block, the mirrored tile through shared
// memory (the broadcast path: one pass instead of unpack + a re-read to split).
struct StagePackedArgs {
  const float* src[kMaxPtrs];     // packed upper, d(d+1)/2
  float* full[kMaxPtrs];          // d x d or nullptr
  float* dst[kMaxPtrs];           // planes [2][d][ld] (fp16 planes: the same storage as __half)
  const float* rscale[kMaxPtrs];  // fp16: per-row scales (packed_row_bounds_kernel)
  int32_t d[kMaxPtrs], ld[kMaxPtrs];
  int64_t plane[kMaxPtrs];
  int32_t tile0[kMaxPtrs + 1];
  int n;
};

template <bool kF16>
__global__ void __launch_bounds__(256) stage_packed_kernel(const __grid_constant__ StagePackedArgs a) {
  __shared__ float tile[64][65];
  const int blk = blockIdx.x;
  int t = 0;
  while (t + 1 < a.n && a.tile0[t + 1] <= blk) ++t;
  const int64_t d = a.d[t], ld = a.ld[t], pl = a.plane[t];
  const int T = int((d + 63) / 64);
  int k = blk - a.tile0[t], I = 0;
  while (k >= T - I) k -= T - I, ++I;
  const int J = I + k;
  const int64_t i0 = int64_t(I) * 64, j0 = int64_t(J) * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const float* src = a.src[t];
  float* full = a.full[t];
  float* dst = a.dst[t];
  float v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int64_t i = i0 + ty + 4 * u, j = j0 + tx;
    const int64_t r = i < j ? i : j, c = i < j ? j : i;
    v[u] = (i < d && j < d) ? src[r * (2 * d - r + 1) / 2 + (c - r)] : 0.f;
  }
  auto put = [&](int64_t i, int64_t j, float x) {
    if (i >= d || j >= d) return;
    if (full) full[i * d + j] = x;
    if constexpr (kF16) {
      __half h, l;
      split_f16(x, a.rscale[t][i], h, l);
      __half* d16 = reinterpret_cast<__half*>(dst);
      d16[i * ld + j] = h;
      d16[pl + i * ld + j] = l;
    } else {
      float h, l;
      split_tf32(x, h, l);
      dst[i * ld + j] = h;
      dst[pl + i * ld + j] = l;
    }
  };
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    put(i0 + ty + 4 * u, j0 + tx, v[u]);
    tile[ty + 4 * u][tx] = v[u];
  }
  if (I != J) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) put(j0 + ty + 4 * u, i0 + tx, tile[tx][ty + 4 * u]);
  }
}

struct ApplyArgs {
  const float* P[kMaxPtrs];
  float* W[kMaxPtrs];
  float* out[kMaxPtrs];
  int64_t n_el[kMaxPtrs];
  int n;
};

__global__ void apply_update_kernel(const __grid_constant__ ApplyArgs a, float alpha) {
  const int t = blockIdx.y;
  const int64_t n = a.n_el[t];
  const float* P = a.P[t];
  float* W = a.W[t];
  float* o = a.out[t];
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const float v = P[e];
    if (W) W[e] -= alpha * v;
    if (o) o[e] = v;
  }
}

}  // namespace spd

using namespace spd;

struct spdkfac_precond_plan {
  int n;
  bool f16 = true;  // fp16 row-scaled planes (kind::f16) or tf32 planes
  std::vector<int32_t> d_out, d_in;
  std::vector<int64_t> ldi, ldo;
  std::vector<float*> gW, aI, tT, gI;  // split planes [2][rows][ld] (tf32, or fp16 in the same storage)
  std::vector<float*> sg, sa, sT, sG;  // fp16: per-row plane scales of gW, aI, tT, gI
  std::vector<float*> amax_a;          // fp16: per-row bound of |A^-1| (the T bound)
  float* gl1 = nullptr;                // fp16: [n] max row L1 norm of the gradient
  std::vector<float*> P;
  CUtensorMap* maps;
  TcItem* items1;
  TcItem* items2;
  TcItem* items2u;  // GEMM2 items whose epilogue updates the weights in place (epis[2n + l])
  int n1, n2;
  TcEpi* epis;      // [2l] split T^T, [2l+1] P, [2n + l] W += alpha P (weights bound at first run)
  std::vector<float*> bound_w;
};

namespace {

void precond_carve(int n, const int32_t* d_out, const int32_t* d_in, Carve& c, spdkfac_precond_plan* p, int* n1,
                   int* n2) {
  *n1 = *n2 = 0;
  for (int l = 0; l < n; ++l) {
    const int64_t m = d_out[l], k = d_in[l];
    const int64_t ldi = round_up(k, kLdAlign), ldo = round_up(m, kLdAlign);
    auto* gW = c.take<float>(size_t(2) * m * ldi);
    auto* aI = c.take<float>(size_t(2) * k * ldi);
    auto* tT = c.take<float>(size_t(2) * k * ldo);
    auto* gI = c.take<float>(size_t(2) * m * ldo);
    auto* P = c.take<float>(size_t(m) * k);
    const int64_t mr = round_up(m, 128), kr = round_up(k, 128);  // scale rows of whole 128-tiles
    auto* sg = c.take<float>(size_t(mr));
    auto* sa = c.take<float>(size_t(kr));
    auto* sT = c.take<float>(size_t(kr));
    auto* sG = c.take<float>(size_t(mr));
    auto* am = c.take<float>(size_t(kr));
    if (p) {
      p->ldi.push_back(ldi);
      p->ldo.push_back(ldo);
      p->gW.push_back(gW);
      p->aI.push_back(aI);
      p->tT.push_back(tT);
      p->gI.push_back(gI);
      p->P.push_back(P);
      p->sg.push_back(sg);
      p->sa.push_back(sa);
      p->sT.push_back(sT);
      p->sG.push_back(sG);
      p->amax_a.push_back(am);
    }
    *n1 += int(cdiv(m, 128) * cdiv(k, 128));
    *n2 += int(cdiv(m, 128) * cdiv(k, 128));
  }
  auto* gl1 = c.take<float>(size_t(n));
  if (p) p->gl1 = gl1;
}

// Split operand rows of the selected layers (sel == nullptr: layers 0..n-1; src indexed like sel) into
// fp16 row-scaled planes: scales (and optional row bounds / L1 maxima) per layer.
int run_split16(int n, const int32_t* sel, const float* const* src, const std::vector<float*>& dst,
                const std::vector<int32_t>& rows, const std::vector<int32_t>& cols, const std::vector<int64_t>& ldd,
                const std::vector<float*>& scale, const std::vector<float*>* amax, float* l1max, cudaStream_t s) {
  for (int off = 0; off < n; off += kMaxPtrs) {
    SplitArgs16 a{};
    a.n = std::min(kMaxPtrs, n - off);
    int r = 0;
    for (int t = 0; t < a.n; ++t) {
      const int i = off + t, l = sel ? sel[i] : i;
      SPD_ARG(l >= 0 && l < int(dst.size()), SPDKFAC_ERR_ARG, "layer index %d out of range", l);
      SPD_ARG(src[i] != nullptr, SPDKFAC_ERR_ARG, "null operand pointer for layer %d", l);
      a.src[t] = src[i];
      a.dst[t] = reinterpret_cast<__half*>(dst[l]);
      a.scale[t] = scale[l];
      a.amax[t] = amax ? (*amax)[l] : nullptr;
      a.l1max[t] = l1max ? l1max + l : nullptr;
      a.cols[t] = cols[l];
      a.ldd[t] = int32_t(ldd[l]);
      a.plane[t] = int64_t(rows[l]) * ldd[l];
      a.row0[t] = r;
      r += rows[l];
    }
    a.row0[a.n] = r;
    stat_begin(kCatPrecSplit, s);
    split_rows_f16_kernel<<<r, 256, 0, s>>>(a);
    SPD_CHECK_LAUNCH();
    stat_end(kCatPrecSplit, s, 0, 0);
  }
  return SPDKFAC_OK;
}

// Split operand rows of the selected layers (sel == nullptr: layers 0..n-1; src indexed like sel).
int run_split(int n, const int32_t* sel, const float* const* src, const std::vector<float*>& dst,
              const std::vector<int32_t>& rows, const std::vector<int32_t>& cols, const std::vector<int64_t>& ldd,
              cudaStream_t s) {
  for (int off = 0; off < n; off += kMaxPtrs) {
    SplitArgs a{};
    a.n = std::min(kMaxPtrs, n - off);
    int r = 0;
    for (int t = 0; t < a.n; ++t) {
      const int i = off + t, l = sel ? sel[i] : i;
      SPD_ARG(l >= 0 && l < int(dst.size()), SPDKFAC_ERR_ARG, "layer index %d out of range", l);
      SPD_ARG(src[i] != nullptr, SPDKFAC_ERR_ARG, "null operand pointer for layer %d", l);
      a.src[t] = src[i];
      a.dst[t] = dst[l];
      a.cols[t] = cols[l];
      a.ldd[t] = int32_t(ldd[l]);
      a.plane[t] = int64_t(rows[l]) * ldd[l];
      a.row0[t] = r;
      r += rows[l];
    }
    a.row0[a.n] = r;
    stat_begin(kCatPrecSplit, s);
    split_rows_batched_kernel<<<r, 256, 0, s>>>(a);
    SPD_CHECK_LAUNCH();
    stat_end(kCatPrecSplit, s, 0, 0);
  }
  return SPDKFAC_OK;
}

}  // namespace

extern "C" {

size_t spdkfac_precond_workspace_size(int n, const int32_t* d_out, const int32_t* d_in) {
  if (n < 1 || !d_out || !d_in) return 0;
  Carve c(nullptr, 0);
  int n1, n2;
  precond_carve(n, d_out, d_in, c, nullptr, &n1, &n2);
  c.take<CUtensorMap>(size_t(4) * n, 128);
  c.take<TcItem>(size_t(n1));
  c.take<TcItem>(size_t(n2));
  c.take<TcItem>(size_t(n2));
  c.take<TcEpi>(size_t(3) * n);
  return c.used + 256;
}

int spdkfac_precond_plan_create(spdkfac_precond_plan** out, int n, const int32_t* d_out, const int32_t* d_in,
                                void* ws, size_t ws_bytes, void* stream) {
  SPD_ARG(out && n >= 1 && d_out && d_in, SPDKFAC_ERR_ARG, "bad precondition plan arguments");
  for (int l = 0; l < n; ++l) SPD_ARG(d_out[l] >= 1 && d_in[l] >= 1, SPDKFAC_ERR_ARG, "dimension must be >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* p = new spdkfac_precond_plan();
  p->n = n;
  p->d_out.assign(d_out, d_out + n);
  p->d_in.assign(d_in, d_in + n);
  p->f16 = precond_f16();
  const int bk = p->f16 ? 64 : kBK;  // K elements per 128-byte operand row
  Carve c(ws, ws_bytes);
  precond_carve(n, d_out, d_in, c, p, &p->n1, &p->n2);
  const size_t operand_bytes = c.used;
  p->maps = c.take<CUtensorMap>(size_t(4) * n, 128);
  p->items1 = c.take<TcItem>(size_t(p->n1));
  p->items2 = c.take<TcItem>(size_t(p->n2));
  p->items2u = c.take<TcItem>(size_t(p->n2));
  p->epis = c.take<TcEpi>(size_t(3) * n);
  if (!c.ok() || !ws) {
    delete p;
    set_error("precondition workspace too small: need %zu bytes, got %zu", c.used, ws_bytes);
    return SPDKFAC_ERR_ARG;
  }
  // zero the split operands once: K padding must read as 0 in every GEMM
  SPD_CUDA(cudaMemsetAsync(ws, 0, operand_bytes, s));
  std::vector<CUtensorMap> maps(size_t(4) * n);
  std::vector<TcItem> it1, it2;
  std::vector<TcEpi> epis(size_t(2) * n);
  int rc;
  for (int l = 0; l < n; ++l) {
    const int64_t m = d_out[l], k = d_in[l], ldi = p->ldi[l], ldo = p->ldo[l];
    if (p->f16 ? ((rc = make_operand_map_f16(&maps[4 * l + 0], p->gW[l], ldi, m, ldi)) ||
                  (rc = make_operand_map_f16(&maps[4 * l + 1], p->aI[l], ldi, k, ldi)) ||
                  (rc = make_operand_map_f16(&maps[4 * l + 2], p->tT[l], ldo, k, ldo)) ||
                  (rc = make_operand_map_f16(&maps[4 * l + 3], p->gI[l], ldo, m, ldo)))
               : ((rc = make_operand_map(&maps[4 * l + 0], p->gW[l], false, ldi, m, ldi)) ||
                  (rc = make_operand_map(&maps[4 * l + 1], p->aI[l], false, ldi, k, ldi)) ||
                  (rc = make_operand_map(&maps[4 * l + 2], p->tT[l], false, ldo, k, ldo)) ||
                  (rc = make_operand_map(&maps[4 * l + 3], p->gI[l], false, ldo, m, ldo)))) {
      delete p;
      return rc;
    }
    if (p->f16) {
      TcEpi e1{}, e2{};
      e1.out = p->tT[l], e1.ld = ldo, e1.plane_stride = k * ldo, e1.alpha = 1.f, e1.mode = kSplitF16;
      e1.rs_a = p->sg[l], e1.rs_b = p->sa[l], e1.gmax = p->gl1 + l, e1.amax_b = p->amax_a[l], e1.rs_out = p->sT[l];
      e2.out = p->P[l], e2.ld = k, e2.alpha = 1.f, e2.mode = kAxpby, e2.rs_a = p->sT[l], e2.rs_b = p->sG[l];
      epis[2 * l] = e1;
      epis[2 * l + 1] = e2;
    } else {
      epis[2 * l] = TcEpi{p->tT[l], ldo, k * ldo, 1.f, 0.f, kSplitTf32, 0, nullptr, 0, 0};
      epis[2 * l + 1] = TcEpi{p->P[l], k, 0, 1.f, 0.f, kAxpby, 0, nullptr, 0, 0};
    }
    for (int mb = 0; mb < cdiv(m, 128); ++mb)
      for (int nb = 0; nb < cdiv(k, 128); ++nb) {
        TcItem a{};
        a.a_map = 4 * l + 0;
        a.b_map = 4 * l + 1;
        a.a_row = mb * 128;
        a.b_row = nb * 128;
        a.k0 = 0;
        a.nk = int(ldi / bk);
        a.epi = 2 * l;
        a.out_r = mb * 128;
        a.out_c = nb * 128;
        a.m_valid = int(std::min<int64_t>(128, m - mb * 128));
        a.n_valid = int(std::min<int64_t>(128, k - nb * 128));
        it1.push_back(a);
        TcItem b{};
        b.a_map = 4 * l + 2;
        b.b_map = 4 * l + 3;
        b.a_row = nb * 128;
        b.b_row = mb * 128;
        b.k0 = 0;
        b.nk = int(ldo / bk);
        b.epi = 2 * l + 1;
        b.out_r = nb * 128;
        b.out_c = mb * 128;
        b.m_valid = int(std::min<int64_t>(128, k - nb * 128));
        b.n_valid = int(std::min<int64_t>(128, m - mb * 128));
        it2.push_back(b);
      }
  }
  std::vector<TcItem> it2u(it2);
  for (TcItem& b : it2u) b.epi = 2 * n + (b.epi - 1) / 2;
  if ((rc = upload(p->maps, maps, s)) || (rc = upload(p->items1, it1, s)) || (rc = upload(p->items2, it2, s)) ||
      (rc = upload(p->items2u, it2u, s)) || (rc = upload(p->epis, epis, s))) {
    delete p;
    return rc;
  }
  *out = p;
  return SPDKFAC_OK;
}

int spdkfac_precond_plan_run(spdkfac_precond_plan* p, const float* const* g_inv, const float* const* grad,
                             const float* const* a_inv, float* const* weight, float alpha, float* const* precond_out,
                             void* stream) {
  SPD_ARG(p && grad, SPDKFAC_ERR_ARG, "null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = p->n;
  std::vector<int64_t> ldi(p->ldi), ldo(p->ldo);
  int rc;
  const Kind kind = p->f16 ? Kind::F16 : Kind::TF32;
  if (p->f16) {
    SPD_CUDA(cudaMemsetAsync(p->gl1, 0, sizeof(float) * size_t(n), s));  // max row L1 of the gradient, per layer
    if ((rc = run_split16(n, nullptr, grad, p->gW, p->d_out, p->d_in, ldi, p->sg, nullptr, p->gl1, s))) return rc;
    if (a_inv && (rc = run_split16(n, nullptr, a_inv, p->aI, p->d_in, p->d_in, ldi, p->sa, &p->amax_a, nullptr, s)))
      return rc;
    if (g_inv && (rc = run_split16(n, nullptr, g_inv, p->gI, p->d_out, p->d_out, ldo, p->sG, nullptr, nullptr, s)))
      return rc;
  } else {
    if ((rc = run_split(n, nullptr, grad, p->gW, p->d_out, p->d_in, ldi, s))) return rc;
    if (a_inv && (rc = run_split(n, nullptr, a_inv, p->aI, p->d_in, p->d_in, ldi, s))) return rc;
    if (g_inv && (rc = run_split(n, nullptr, g_inv, p->gI, p->d_out, p->d_out, ldo, s))) return rc;
  }
  // algorithmic work: 2 g a (a + g) per layer, split over the two GEMMs
  double f1 = 0, f2 = 0;
  for (int l = 0; l < n; ++l) {
    f1 += 2.0 * p->d_out[l] * p->d_in[l] * p->d_in[l];
    f2 += 2.0 * p->d_out[l] * p->d_out[l] * p->d_in[l];
  }
  // persistent-grid cap (SPDKFAC_PRECOND_CTAS): SMs left to a concurrent latency-bound inversion chain
  static const int prec_ctas = getenv("SPDKFAC_PRECOND_CTAS") ? atoi(getenv("SPDKFAC_PRECOND_CTAS")) : 0;
  TcRun run1{};
  run1.probe = stat_begin(kCatPrecGemm, s);
  if ((rc = launch_tc3_acc(p->maps, p->items1, p->epis, p->n1, s, run1, kind, prec_ctas))) return rc;
  stat_end(kCatPrecGemm, s, f1, 0);
  // weight update fused into GEMM2's epilogue (W += (-alpha) P, no P round trip) once the weight
  // pointers are bound: bound on the first run outside stream capture (weights do not move)
  bool fused = false;
  if (weight && !precond_out) {
    fused = p->bound_w.size() == size_t(n) && std::equal(p->bound_w.begin(), p->bound_w.end(), weight);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SPD_CUDA(cudaStreamIsCapturing(s, &cs));
    if (!fused && cs == cudaStreamCaptureStatusNone) {
      std::vector<TcEpi> ew(static_cast<size_t>(n));
      for (int l = 0; l < n; ++l) {
        SPD_ARG(weight[l] != nullptr, SPDKFAC_ERR_ARG, "null weight pointer for layer %d", l);
        ew[l] = TcEpi{weight[l], p->d_in[l], 0, 0.f, 1.f, kUpdate, 0, nullptr, 0, 0};
        if (p->f16) ew[l].rs_a = p->sT[l], ew[l].rs_b = p->sG[l];
      }
      SPD_CUDA(cudaMemcpyAsync(p->epis + 2 * n, ew.data(), ew.size() * sizeof(TcEpi), cudaMemcpyHostToDevice, s));
      p->bound_w.assign(weight, weight + n);
      fused = true;
    }
  }
  Probe* pr2 = stat_begin(kCatPrecGemm, s);
  if ((rc = launch_tc3_acc(p->maps, fused ? p->items2u : p->items2, p->epis, p->n2, s,
                           TcRun{nullptr, 0, -alpha, 0.f, 1.f, 0, pr2}, kind, prec_ctas)))
    return rc;
  stat_end(kCatPrecGemm, s, f2, 0);
  if (fused || (!weight && !precond_out)) return SPDKFAC_OK;
  for (int off = 0; off < n; off += kMaxPtrs) {
    ApplyArgs a{};
    a.n = std::min(kMaxPtrs, n - off);
    for (int t = 0; t < a.n; ++t) {
      const int l = off + t;
      a.P[t] = p->P[l];
      a.W[t] = weight ? weight[l] : nullptr;
      a.out[t] = precond_out ? precond_out[l] : nullptr;
      a.n_el[t] = int64_t(p->d_out[l]) * p->d_in[l];
    }
    stat_begin(kCatPrecApply, s);
    apply_update_kernel<<<dim3(64, a.n), 256, 0, s>>>(a, alpha);
    SPD_CHECK_LAUNCH();
    stat_end(kCatPrecApply, s, 0, 0);
  }
  return SPDKFAC_OK;
}

int spdkfac_precond_plan_stage_inverses(spdkfac_precond_plan* p, int which, int n_sel, const int32_t* layers,
                                        const float* const* inv, void* stream) {
  SPD_ARG(p && (which == 0 || which == 1) && n_sel >= 0 && (n_sel == 0 || (layers && inv)), SPDKFAC_ERR_ARG,
          "bad stage_inverses arguments");
  if (n_sel == 0) return SPDKFAC_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int64_t> ld(which == 0 ? p->ldi : p->ldo);
  const auto& dims = which == 0 ? p->d_in : p->d_out;
  if (p->f16)
    return run_split16(n_sel, layers, inv, which == 0 ? p->aI : p->gI, dims, dims, ld, which == 0 ? p->sa : p->sG,
                       which == 0 ? &p->amax_a : nullptr, nullptr, s);
  return run_split(n_sel, layers, inv, which == 0 ? p->aI : p->gI, dims, dims, ld, s);
}

int spdkfac_precond_plan_stage_packed(spdkfac_precond_plan* p, int which, int n_sel, const int32_t* layers,
                                      const float* const* packed, float* const* full_out, void* stream) {
  SPD_ARG(p && (which == 0 || which == 1) && n_sel >= 0 && (n_sel == 0 || (layers && packed)), SPDKFAC_ERR_ARG,
          "bad stage_packed arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const auto& dims = which == 0 ? p->d_in : p->d_out;
  const auto& lds = which == 0 ? p->ldi : p->ldo;
  const auto& planes = which == 0 ? p->aI : p->gI;
  for (int off = 0; off < n_sel; off += kMaxPtrs) {
    StagePackedArgs a{};
    DiagArgs da{};
    a.n = da.n = std::min(kMaxPtrs, n_sel - off);
    int tiles = 0;
    for (int t = 0; t < a.n; ++t) {
      const int i = off + t, l = layers[i];
      SPD_ARG(l >= 0 && l < p->n, SPDKFAC_ERR_ARG, "layer index %d out of range", l);
      SPD_ARG(packed[i] != nullptr, SPDKFAC_ERR_ARG, "null packed inverse for layer %d", l);
      a.src[t] = packed[i];
      a.full[t] = full_out ? full_out[i] : nullptr;
      a.dst[t] = planes[l];
      a.rscale[t] = which == 0 ? p->sa[l] : p->sG[l];
      da.src[t] = packed[i];
      da.scale[t] = which == 0 ? p->sa[l] : p->sG[l];
      da.amax[t] = which == 0 ? p->amax_a[l] : nullptr;
      da.d[t] = dims[l];
      a.d[t] = dims[l];
      a.ld[t] = int32_t(lds[l]);
      a.plane[t] = int64_t(dims[l]) * lds[l];
      a.tile0[t] = tiles;
      const int T = (dims[l] + 63) / 64;
      tiles += T * (T + 1) / 2;
    }
    a.tile0[a.n] = tiles;
    stat_begin(kCatPrecSplit, s);
    if (p->f16) {
      packed_row_bounds_kernel<<<da.n, 256, 0, s>>>(da);
      SPD_CHECK_LAUNCH();
      stage_packed_kernel<true><<<tiles, 256, 0, s>>>(a);
    } else {
      stage_packed_kernel<false><<<tiles, 256, 0, s>>>(a);
    }
    SPD_CHECK_LAUNCH();
    stat_end(kCatPrecSplit, s, 0, 0);
  }
  return SPDKFAC_OK;
}

void spdkfac_precond_plan_destroy(spdkfac_precond_plan* p) { delete p; }

}  // extern "C"
