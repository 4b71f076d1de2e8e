// Batched damped inverse of symmetric positive-definite Kronecker factors.
//
// Algorithm: Gauss-Jordan "sweep" (the symmetric sweep operator).  Sweeping pivot k
// of a symmetric matrix maps
//     a_kk -> -1/a_kk,  a_ik -> a_ik/a_kk,  a_kj -> a_kj/a_kk,  a_ij -> a_ij - a_ik a_kj / a_kk,
// and sweeping every pivot leaves -A^{-1}.  Its pivots are the Schur-complement
// diagonals, i.e. the squared Cholesky diagonals, so the first non-positive pivot is
// exactly LAPACK dpotrf's failing index (damped_inverse, linalg.py:141-145).
//
//   d <= 128 : one CTA per matrix, whole matrix in shared memory, scalar sweep.
//   d  > 128 : blocked sweep on the matrix padded to a multiple of 128 with an identity
//              block, one 128-pivot block per step k, batched over all matrices:
//                pivot  : P = W[K,K] swept in shared memory  -> P^-1, W[K,K] = -P^-1
//                panel  : C_R = W[R,K] P^-1 (row blocks R != K), W[R,K] = C_R, W[K,R] = C_R^T,
//                         old panel and C staged as tf32 hi/lo planes
//                update : W[I,J] -= Wold[I,K] C_J^T for I <= J (I,J != K) on tcgen05
//                         (3 x tf32, rank-128), mirrored to W[J,I]
//              finalize: out = -(W + W^T)/2 cropped to d x d (the reference's symmetrisation).
#include "runtime.cuh"

namespace spd {

constexpr int kB = 128;          // pivot block = tile edge
constexpr int kSmemLd = kB + 1;  // padded row stride of the shared-memory block

struct InvMat {
  float* W;          // padded working matrix [dp][dp] (blocked path)
  float* pinv;       // [128][128] scratch for the current pivot inverse
  const float* in;   // packed upper input
  float* out;        // full d x d output (ld = d)
  int32_t* info;     // 0 or failing pivot + 1
  int32_t d, dp;
  int32_t panel_row0;  // first row of this matrix's panels in the shared panel planes
  int32_t pad_;
};

// Register-resident scalar sweep of one 128 x 128 block by 512 threads: thread t owns
// row i = t >> 2, columns [32q, 32q + 32), q = t & 3, in registers.  Per pivot k the four
// owners of row k publish it to shared memory (double-buffered by k parity, rows skewed by
// 4 floats per 32 so the four column quarters hit distinct banks); every thread then
// applies  a_ij -= (a_ik / p) a_kj,  a_ik <- a_ik / p,  a_kj <- a_kj / p,  a_kk <- -1/p,
// using a_ik = a_ki (the swept block stays symmetric to rounding).  Rows/columns >= n are
// identity padding and are never pivots.  Returns -1, or the failing pivot (uniform).
constexpr int kRowSkew = 36;  // skewed row buffer: element j at (j >> 5) * 36 + (j & 31)

__device__ __forceinline__ int sweep128(float (&a)[32], int n, float* rbuf /* 2 x 4*36 */) {
  const int t = threadIdx.x, i = t >> 2, q = t & 3;
  for (int k = 0; k < n; ++k) {
    float* rk = rbuf + (k & 1) * (4 * kRowSkew);
    if (i == k) {
#pragma unroll
      for (int jj = 0; jj < 32; jj += 4)
        *reinterpret_cast<float4*>(rk + q * kRowSkew + jj) = make_float4(a[jj], a[jj + 1], a[jj + 2], a[jj + 3]);
    }
    __syncthreads();
    const float p = rk[(k >> 5) * kRowSkew + (k & 31)];
    if (!(p > 0.f)) return k;  // dpotrf's "ajj <= 0 or NaN" test, on the same Schur pivots
    const float pinv = 1.0f / p;
    const float ci = rk[(i >> 5) * kRowSkew + (i & 31)] * pinv;  // a_ik / p
    const int kq = k >> 5, kj = k & 31;
    if (i == k) {
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) a[jj] = (q == kq && jj == kj) ? -pinv : a[jj] * pinv;
    } else {
#pragma unroll
      for (int jj = 0; jj < 32; jj += 4) {
        const float4 r = *reinterpret_cast<const float4*>(rk + q * kRowSkew + jj);
        a[jj + 0] = fmaf(-ci, r.x, a[jj + 0]);
        a[jj + 1] = fmaf(-ci, r.y, a[jj + 1]);
        a[jj + 2] = fmaf(-ci, r.z, a[jj + 2]);
        a[jj + 3] = fmaf(-ci, r.w, a[jj + 3]);
      }
      if (q == kq) {  // column k: a_ik <- a_ik / p
#pragma unroll
        for (int jj = 0; jj < 32; ++jj)
          if (jj == kj) a[jj] = ci;
      }
    }
  }
  return -1;
}

__device__ __forceinline__ float packed_at(const float* p, int64_t d, int64_t i, int64_t j) {
  const int64_t r = i < j ? i : j, c = i < j ? j : i;
  return p[r * (2 * d - r + 1) / 2 + (c - r)];
}

// ---------------------------------------------------------------- d <= 128
__global__ void __launch_bounds__(512) small_inverse_kernel(const InvMat* __restrict__ mats,
                                                            const int32_t* __restrict__ ids, float gamma) {
  __shared__ __align__(16) float rbuf[2 * 4 * kRowSkew];
  const InvMat m = mats[ids[blockIdx.x]];
  const int n = m.d;
  const int i = threadIdx.x >> 2, q = threadIdx.x & 3;
  float a[32];
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) {
    const int j = q * 32 + jj;
    a[jj] = (i < n && j < n) ? packed_at(m.in, n, i, j) + (i == j ? gamma : 0.f) : (i == j ? 1.f : 0.f);
  }
  const int f = sweep128(a, n, rbuf);
  if (f >= 0) {
    if (threadIdx.x == 0) *m.info = f + 1;
    return;
  }
  if (threadIdx.x == 0) *m.info = 0;
  // out = -(S + S^T)/2 through shared memory (uniform control flow)
  extern __shared__ float sm[];
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) sm[i * kSmemLd + q * 32 + jj] = -a[jj];
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e - r * n;
    m.out[e] = 0.5f * (sm[r * kSmemLd + c] + sm[c * kSmemLd + r]);
  }
}

// ---------------------------------------------------------------- blocked path
__global__ void damp_unpack_kernel(const InvMat* __restrict__ mats, const int32_t* __restrict__ ids, float gamma) {
  const InvMat m = mats[ids[blockIdx.y]];
  const int64_t dp = m.dp, d = m.d;
  if (blockIdx.x == 0 && threadIdx.x == 0) *m.info = 0;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < dp * dp; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / dp, j = e - i * dp;
    float v;
    if (i < d && j < d) v = packed_at(m.in, d, i, j) + (i == j ? gamma : 0.f);
    else v = (i == j) ? 1.f : 0.f;  // identity padding: never fails, decouples
    m.W[e] = v;
  }
}

__global__ void __launch_bounds__(512) pivot_kernel(const InvMat* __restrict__ mats,
                                                    const int32_t* __restrict__ ids, int k) {
  __shared__ __align__(16) float rbuf[2 * 4 * kRowSkew];
  const InvMat m = mats[ids[blockIdx.x]];
  if (*m.info != 0) return;
  const int64_t dp = m.dp, K0 = int64_t(k) * kB;
  const int i = threadIdx.x >> 2, q = threadIdx.x & 3;
  float a[32];
  const float* src = m.W + (K0 + i) * dp + K0 + q * 32;
#pragma unroll
  for (int jj = 0; jj < 32; jj += 4) {
    const float4 v = *reinterpret_cast<const float4*>(src + jj);
    a[jj] = v.x, a[jj + 1] = v.y, a[jj + 2] = v.z, a[jj + 3] = v.w;
  }
  const int f = sweep128(a, kB, rbuf);
  if (f >= 0) {
    if (threadIdx.x == 0) *m.info = int(K0) + f + 1;
    return;
  }
  float* dst = m.W + (K0 + i) * dp + K0 + q * 32;  // W[K,K] <- -P^-1
  float* pv = m.pinv + i * kB + q * 32;             // P^-1
#pragma unroll
  for (int jj = 0; jj < 32; jj += 4) {
    *reinterpret_cast<float4*>(dst + jj) = make_float4(a[jj], a[jj + 1], a[jj + 2], a[jj + 3]);
    *reinterpret_cast<float4*>(pv + jj) = make_float4(-a[jj], -a[jj + 1], -a[jj + 2], -a[jj + 3]);
  }
}

struct PanelJob {
  int32_t mat, rb;  // matrix id, row block R (!= K)
};

// C_R = W[R,K] P^-1 (fp32 FFMA, 8x8 register tile per thread), stage split planes.
__global__ void __launch_bounds__(256) panel_kernel(const InvMat* __restrict__ mats,
                                                    const PanelJob* __restrict__ jobs, int k,
                                                    float* __restrict__ panA, float* __restrict__ panC,
                                                    int64_t plane_rows) {
  extern __shared__ float sm[];
  float* a = sm;                  // [128][129] old panel W[R,K]
  float* p = sm + kB * kSmemLd;   // [128][129] P^-1
  const PanelJob job = jobs[blockIdx.x];
  const InvMat m = mats[job.mat];
  if (*m.info != 0) return;
  const int64_t dp = m.dp, K0 = int64_t(k) * kB, R0 = int64_t(job.rb) * kB;
  const int64_t prow = int64_t(m.panel_row0) + R0;  // panel plane row of local row 0
  const int64_t plane = plane_rows * kB;
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    const int i = e / kB, j = e % kB;
    const float v = m.W[(R0 + i) * dp + K0 + j];
    a[i * kSmemLd + j] = v;
    p[i * kSmemLd + j] = m.pinv[e];
    float h, l;
    split_tf32(v, h, l);
    panA[(prow + i) * kB + j] = h;
    panA[plane + (prow + i) * kB + j] = l;
  }
  __syncthreads();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // rows ty*8.., cols tx + 16*c
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
  for (int kk = 0; kk < kB; ++kk) {
    float av[8], pv[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) av[r] = a[(ty * 8 + r) * kSmemLd + kk];
#pragma unroll
    for (int c = 0; c < 8; ++c) pv[c] = p[kk * kSmemLd + tx + 16 * c];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(av[r], pv[c], acc[r][c]);
  }
  __syncthreads();  // all reads of `a` done: reuse it to stage C for the transposed store
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = ty * 8 + r, j = tx + 16 * c;
      const float v = acc[r][c];
      m.W[(R0 + i) * dp + K0 + j] = v;  // A_ik <- A_ik P^-1
      a[j * kSmemLd + i] = v;           // staged transposed
      float h, l;
      split_tf32(v, h, l);
      panC[(prow + i) * kB + j] = h;
      panC[plane + (prow + i) * kB + j] = l;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {  // A_ki <- P^-1 A_ki, coalesced along i
    const int j = e / kB, i = e % kB;
    m.W[(K0 + j) * dp + R0 + i] = a[j * kSmemLd + i];
  }
}

__global__ void finalize_kernel(const InvMat* __restrict__ mats, const int32_t* __restrict__ ids) {
  const InvMat m = mats[ids[blockIdx.y]];
  if (*m.info != 0) return;
  const int64_t d = m.d, dp = m.dp;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < d * d; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / d, j = e - i * d;
    m.out[e] = -0.5f * (m.W[i * dp + j] + m.W[j * dp + i]);
  }
}

}  // namespace spd

using namespace spd;

struct spdkfac_inverse_plan {
  int n;
  std::vector<int32_t> dims;
  double small_flops = 0;       // sum d^3 of the shared-memory path (algorithmic potrf+potri)
  double algo_flops = 0;        // sum d^3 over all matrices
  InvMat* mats;                 // device
  int32_t* small_ids;           // device
  int n_small;
  int32_t* blocked_ids;         // device
  int n_blocked;
  int steps;
  std::vector<int> piv_off, piv_cnt, pan_off, pan_cnt, upd_off, upd_cnt;
  int32_t* piv_ids;             // device, concatenated per step
  PanelJob* pan_jobs;           // device
  CUtensorMap* maps;            // [0] = panel A planes, [1] = panel C planes
  TcItem* items;
  TcEpi* epis;
  float* panA;
  float* panC;
  int64_t plane_rows;
};

namespace {

struct InvLayout {
  size_t bytes;
};

size_t inverse_carve(int n, const int32_t* dims, Carve& c, spdkfac_inverse_plan* p, std::vector<InvMat>* mats,
                     std::vector<int32_t>* small, std::vector<int32_t>* blocked, int64_t* plane_rows,
                     int64_t* total_items, int64_t* total_piv, int64_t* total_pan, int* steps) {
  int64_t rows = 0, items = 0, piv = 0, pan = 0;
  int st = 0;
  for (int t = 0; t < n; ++t) {
    const int d = dims[t];
    InvMat m{};
    m.d = d;
    if (d <= kB) {
      m.dp = d;
      if (small) small->push_back(t);
    } else {
      const int dp = int(round_up(d, kB));
      const int T = dp / kB;
      m.dp = dp;
      m.W = c.take<float>(size_t(dp) * dp);
      m.pinv = c.take<float>(size_t(kB) * kB);
      m.panel_row0 = int(rows);
      rows += dp;
      if (blocked) blocked->push_back(t);
      st = std::max(st, T);
      piv += T;
      pan += int64_t(T) * (T - 1);
      items += int64_t(T) * (int64_t(T - 1) * T / 2);  // per step: (T-1)T/2 upper pairs excluding K
    }
    if (mats) mats->push_back(m);
  }
  *plane_rows = rows;
  *total_items = items;
  *total_piv = piv;
  *total_pan = pan;
  *steps = st;
  return c.used;
}

}  // namespace

extern "C" {

size_t spdkfac_inverse_workspace_size(int n, const int32_t* dims) {
  if (n < 0 || (n > 0 && !dims)) return 0;
  Carve c(nullptr, 0);
  int64_t rows, items, piv, pan;
  int steps;
  inverse_carve(n, dims, c, nullptr, nullptr, nullptr, nullptr, &rows, &items, &piv, &pan, &steps);
  c.take<float>(size_t(2) * rows * kB);  // panA
  c.take<float>(size_t(2) * rows * kB);  // panC
  c.take<InvMat>(size_t(n));
  c.take<int32_t>(size_t(n));
  c.take<int32_t>(size_t(n));
  c.take<int32_t>(size_t(piv));
  c.take<PanelJob>(size_t(pan));
  c.take<CUtensorMap>(2, 128);
  c.take<TcItem>(size_t(items));
  c.take<TcEpi>(size_t(n));
  return c.used + 256;
}

int spdkfac_inverse_plan_create(spdkfac_inverse_plan** out, int n, const int32_t* dims, const float* const* packed_in,
                                float* const* out_full, int32_t* info_dev, void* ws, size_t ws_bytes, void* stream) {
  SPD_ARG(out && n >= 1 && dims && packed_in && out_full && info_dev, SPDKFAC_ERR_ARG, "bad inverse plan arguments");
  for (int t = 0; t < n; ++t) SPD_ARG(dims[t] >= 1, SPDKFAC_ERR_ARG, "dimension must be >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* p = new spdkfac_inverse_plan();
  p->n = n;
  p->dims.assign(dims, dims + n);
  Carve c(ws, ws_bytes);
  std::vector<InvMat> mats;
  std::vector<int32_t> small, blocked;
  int64_t items_total, piv_total, pan_total;
  inverse_carve(n, dims, c, p, &mats, &small, &blocked, &p->plane_rows, &items_total, &piv_total, &pan_total,
                &p->steps);
  p->panA = c.take<float>(size_t(2) * p->plane_rows * kB);
  p->panC = c.take<float>(size_t(2) * p->plane_rows * kB);
  p->mats = c.take<InvMat>(size_t(n));
  p->small_ids = c.take<int32_t>(size_t(n));
  p->blocked_ids = c.take<int32_t>(size_t(n));
  p->piv_ids = c.take<int32_t>(size_t(piv_total));
  p->pan_jobs = c.take<PanelJob>(size_t(pan_total));
  p->maps = c.take<CUtensorMap>(2, 128);
  p->items = c.take<TcItem>(size_t(items_total));
  p->epis = c.take<TcEpi>(size_t(n));
  if (!c.ok() || !ws) {
    delete p;
    set_error("inverse workspace too small: need %zu bytes, got %zu", c.used, ws_bytes);
    return SPDKFAC_ERR_ARG;
  }
  for (int t = 0; t < n; ++t) {
    mats[t].in = packed_in[t];
    mats[t].out = out_full[t];
    mats[t].info = info_dev + t;
  }
  p->n_small = int(small.size());
  for (int t = 0; t < n; ++t) {
    const double d3 = double(dims[t]) * dims[t] * dims[t];
    p->algo_flops += d3;
    if (dims[t] <= kB) p->small_flops += d3;
  }
  p->n_blocked = int(blocked.size());
  // per-step schedules
  std::vector<int32_t> piv_ids;
  std::vector<PanelJob> pan;
  std::vector<TcItem> items;
  std::vector<TcEpi> epis(n);
  for (int t = 0; t < n; ++t)
    epis[t] = TcEpi{mats[t].W, mats[t].dp, 0, -1.f, 1.f, kAxpby, 0};
  for (int k = 0; k < p->steps; ++k) {
    p->piv_off.push_back(int(piv_ids.size()));
    p->pan_off.push_back(int(pan.size()));
    p->upd_off.push_back(int(items.size()));
    for (int t : blocked) {
      const int T = mats[t].dp / kB;
      if (k >= T) continue;
      piv_ids.push_back(t);
      for (int r = 0; r < T; ++r)
        if (r != k) pan.push_back(PanelJob{t, r});
      for (int I = 0; I < T; ++I)
        for (int J = I; J < T; ++J) {
          if (I == k || J == k) continue;
          TcItem it{};
          it.a_map = 0;
          it.b_map = 1;
          it.a_row = mats[t].panel_row0 + I * kB;
          it.b_row = mats[t].panel_row0 + J * kB;
          it.k0 = 0;
          it.nk = kB / 32;
          it.epi = t;
          it.flags = (I == J) ? 0 : kMirror;
          it.out_r = I * kB;
          it.out_c = J * kB;
          it.m_valid = kB;
          it.n_valid = kB;
          items.push_back(it);
        }
    }
    p->piv_cnt.push_back(int(piv_ids.size()) - p->piv_off.back());
    p->pan_cnt.push_back(int(pan.size()) - p->pan_off.back());
    p->upd_cnt.push_back(int(items.size()) - p->upd_off.back());
  }
  std::vector<CUtensorMap> maps(2);
  int rc = SPDKFAC_OK;
  if (p->plane_rows > 0) {
    if ((rc = make_operand_map(&maps[0], p->panA, false, kB, p->plane_rows, kB)) ||
        (rc = make_operand_map(&maps[1], p->panC, false, kB, p->plane_rows, kB))) {
      delete p;
      return rc;
    }
  }
  if ((rc = upload(p->mats, mats, s)) || (rc = upload(p->small_ids, small, s)) ||
      (rc = upload(p->blocked_ids, blocked, s)) || (rc = upload(p->piv_ids, piv_ids, s)) ||
      (rc = upload(p->pan_jobs, pan, s)) || (p->plane_rows > 0 && (rc = upload(p->maps, maps, s))) ||
      (rc = upload(p->items, items, s)) || (rc = upload(p->epis, epis, s))) {
    delete p;
    return rc;
  }
  static bool attrs = false;
  if (!attrs) {
    SPD_CUDA(cudaFuncSetAttribute(small_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kB * kSmemLd * 4));
    SPD_CUDA(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kB * kSmemLd * 4));
    attrs = true;
  }
  *out = p;
  return SPDKFAC_OK;
}

int spdkfac_inverse_plan_run(spdkfac_inverse_plan* p, float gamma, void* stream) {
  SPD_ARG(p != nullptr, SPDKFAC_ERR_ARG, "null plan");
  SPD_ARG(gamma >= 0.f, SPDKFAC_ERR_ARG, "damping must be nonnegative, got %g", double(gamma));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->n_small > 0) {
    stat_begin(kCatInvSmall, s);
    small_inverse_kernel<<<p->n_small, 512, kB * kSmemLd * 4, s>>>(p->mats, p->small_ids, gamma);
    SPD_CHECK_LAUNCH();
    stat_end(kCatInvSmall, s, p->small_flops, 0);
  }
  if (p->n_blocked > 0) {
    stat_begin(kCatInvUnpackFinal, s);
    damp_unpack_kernel<<<dim3(64, p->n_blocked), 256, 0, s>>>(p->mats, p->blocked_ids, gamma);
    SPD_CHECK_LAUNCH();
    stat_end(kCatInvUnpackFinal, s, 0, 0);
    for (int k = 0; k < p->steps; ++k) {
      if (p->piv_cnt[k] > 0) {
        stat_begin(kCatInvPivot, s);
        pivot_kernel<<<p->piv_cnt[k], 512, 0, s>>>(p->mats, p->piv_ids + p->piv_off[k], k);
        SPD_CHECK_LAUNCH();
        stat_end(kCatInvPivot, s, 2.0 * kB * kB * kB * p->piv_cnt[k], 0);
      }
      if (p->pan_cnt[k] > 0) {
        stat_begin(kCatInvPanel, s);
        panel_kernel<<<p->pan_cnt[k], 256, 2 * kB * kSmemLd * 4, s>>>(p->mats, p->pan_jobs + p->pan_off[k], k,
                                                                        p->panA, p->panC, p->plane_rows);
        SPD_CHECK_LAUNCH();
        stat_end(kCatInvPanel, s, 2.0 * kB * kB * kB * p->pan_cnt[k], 0);
      }
      stat_begin(kCatInvUpdate, s);
      int rc = launch_tc3(Kind::TF32, p->maps, p->items + p->upd_off[k], p->epis, p->upd_cnt[k], s);
      if (rc) return rc;
      stat_end(kCatInvUpdate, s, 2.0 * kB * kB * kB * p->upd_cnt[k], 0);
    }
    stat_begin(kCatInvUnpackFinal, s);
    finalize_kernel<<<dim3(64, p->n_blocked), 256, 0, s>>>(p->mats, p->blocked_ids);
    SPD_CHECK_LAUNCH();
    stat_end(kCatInvUnpackFinal, s, 0, 0);
  }
  return SPDKFAC_OK;
}

void spdkfac_inverse_plan_destroy(spdkfac_inverse_plan* p) { delete p; }

}  // extern "C"
