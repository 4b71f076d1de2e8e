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
//                pivot  : P = W[K,K] swept in registers -> W[K,K] = -P^-1, P^-1 as tf32 planes
//                stage  : old column panel W[:,K] -> tf32 hi/lo planes
//                panel  : C = Wold[:,K] P^-1 on tcgen05 (3 x tf32); epilogue writes W[R,K] = C_R,
//                         W[K,R] = C_R^T and C as tf32 planes
//                update : W[I,J] -= Wold[I,K] C_J^T for I <= J (I,J != K) on tcgen05
//                         (3 x tf32, rank-128), mirrored to W[J,I]
//              finalize: out = -(W + W^T)/2 cropped to d x d (the reference's symmetrisation).
#include <algorithm>
#include <cstdint>
#include <map>
#include <tuple>
#include <type_traits>

#include "runtime.cuh"

namespace spd {

constexpr int kB = 128;          // pivot block = tile edge
constexpr int kSmemLd = kB + 1;  // padded row stride of the shared-memory block
// Panel planes panA / panC: [2 planes][rows][kPanCols]; step k uses the 128 columns of slot
// k % kPanSlots, so the panels of a fused step group are adjacent columns (one K = 128 x steps
// update reads them all) and the look-ahead step never overwrites a slot still being read.
constexpr int kFuse = 8;                // trailing-update steps fused per W pass (see the update plan)
constexpr int kPanSlots = 2 * kFuse;    // a group's slots + the next group's look-ahead never alias
constexpr int kPanCols = kPanSlots * kB;
// fp16 operand classes of the panel / P^-1 planes (InvMat::scale index; see inv_scale_kernel)
constexpr int kScInv = 0, kScReg = 1, kScSchur = 2;
// Accuracy model of the fp16 planes: an entry of class bound B is held to 2^-38 B absolute, so the
// inverse keeps a normwise error ~ (sigma / gamma) 2^-38 -- fp32-class (<= 2^-22) while max_i (F_ii +
// gamma) / gamma <= 2^16 (the BASELINE configs: <= 2^10).  Runs with gamma < kF16MinGamma use tf32
// planes (exponent range of fp32, 2^-22 relative per entry); SPDKFAC_INV_TF32=1 forces them.
constexpr float kF16MinGamma = 1e-4f;

struct InvMat {
  float* W;          // padded working matrix [dp][dp] (blocked path)
  const float* in;   // packed upper input
  float* out;        // full d x d output (ld = d)
  int32_t* info;     // 0 or failing pivot + 1
  int32_t d, dp;
  int32_t panel_row0;  // first row of this matrix's panels in the shared panel planes
  int32_t slot;        // index among blocked matrices (row slot*128 of the P^-1 planes)
  float* scale;        // [4] fp16 operand-class scales (inv_scale_kernel, kScInv / kScReg / kScSchur)
};

struct TileJob {  // one 64 x 64 tile (I <= J) of a blocked matrix, for unpack/finalize
  int32_t mat, ti, tj, pad_;
};

// Register-resident sweep of one 128 x 128 block by 512 threads: thread t owns row
// i = t & 127, columns [32q, 32q + 32), q = t >> 7 (warp-uniform), in registers.
// 8-pivot block sweep used by the kernels: thread t owns rows 2r, 2r+1
// (r = t & 63) x columns [16q, 16q + 16) (q = t >> 6, warp-uniform), so every pivot-row
// vector R[j] read from shared memory serves two rows.  Warp 0 sweeps the 8x8 pivot block
// (shuffles) once; warps 0-3 then form the row weights w_i once per row (not once per column
// quarter) and publish them, so the update costs 2 x LDS.128 + 8 FFMA per element pair.
struct B8v2Shared {
  float4 R[2][128][2];  // pivot rows K0..K0+7 of column j (double-buffered)
  float4 W[2][128][2];  // row weights w_i
  float S[8][8];
  int fail[2];
};

// reciprocal: MUFU approximation + one Newton step (<= 1 ulp); __frcp_rn's IEEE path measured ~1.2k
// cycles per call inside the 8x8 pivot sweep, the serial core of every pivot block
__device__ __forceinline__ float rcp_nr1(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r * fmaf(-x, r, 2.f);
}
#ifdef SPD_PIVOT_TIMING
#define B8_MARK(i) \
  do {             \
    const long long c_ = clock64(); ph[i] += c_ - last; last = c_; \
  } while (0)  // every thread (no divergence); thread 0 prints
#else
#define B8_MARK(i) \
  do {             \
  } while (0)
#endif
__device__ __forceinline__ int sweep128_b8v2(float (&a)[2][16], int n, B8v2Shared& sh) {
  const int t = threadIdx.x, r = t & 63, q = t >> 6;
  const int lane = t & 31, warp = t >> 5;
  const int nb = (n + 7) >> 3;
#ifdef SPD_PIVOT_TIMING
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, last = clock64();
#endif
  for (int kb = 0; kb < nb; ++kb) {
    const int buf = kb & 1;
    float* Rf = reinterpret_cast<float*>(sh.R[buf]);
    const int K0 = kb * 8;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int s0 = 2 * r + u - K0;
      if (s0 >= 0 && s0 < 8) {
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) Rf[(q * 16 + jj) * 8 + s0] = a[u][jj];
      }
    }
    B8_MARK(0);
    __syncthreads();
    B8_MARK(1);
    if (warp < 4) {
      if (warp == 0) {  // lane holds S[rr][c] and S[rr][c + 4]
        const int rr = lane >> 2, c = lane & 3;
        float v0 = Rf[(K0 + c) * 8 + rr], v1 = Rf[(K0 + c + 4) * 8 + rr];
        int fail = -1;
#pragma unroll
        for (int p = 0; p < 8; ++p) {  // branch-free: a `break` here made every shuffle of the sweep
          // take the compiler's divergent-collective path (WARPSYNC loops), ~9k cycles per 8x8 sweep
          const float pv = __shfl_sync(0xffffffffu, (p < 4) ? v0 : v1, (p << 2) | (p & 3));
          if (fail < 0 && !(pv > 0.f)) fail = p;  // warp-uniform; later pivots compute garbage, unused
          const float pinv = rcp_nr1(pv);
          const float rp0 = __shfl_sync(0xffffffffu, v0, (p << 2) | c);
          const float rp1 = __shfl_sync(0xffffffffu, v1, (p << 2) | c);
          const float cp = __shfl_sync(0xffffffffu, (p < 4) ? v0 : v1, (rr << 2) | (p & 3));
          float n0, n1;
          if (rr == p) {
            n0 = (c == p) ? -pinv : rp0 * pinv;
            n1 = (c + 4 == p) ? -pinv : rp1 * pinv;
          } else {
            n0 = (c == p) ? cp * pinv : fmaf(-cp * pinv, rp0, v0);
            n1 = (c + 4 == p) ? cp * pinv : fmaf(-cp * pinv, rp1, v1);
          }
          v0 = n0, v1 = n1;
        }
        sh.S[rr][c] = v0;
        sh.S[rr][c + 4] = v1;
        if (lane == 0) sh.fail[buf] = fail;
      }
      B8_MARK(2);
      named_bar_sync(1, 128);
      B8_MARK(3);
      const int i = t;  // row weights for row i = t (128 threads)
      const int s0 = i - K0;
      float w[8];
      if (s0 >= 0 && s0 < 8) {
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) w[cc] = sh.S[s0][cc];
      } else {
        const float4 ra = sh.R[buf][i][0], rb = sh.R[buf][i][1];
        const float rv[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          float acc = 0.f;
#pragma unroll
          for (int ss = 0; ss < 8; ++ss) acc = fmaf(rv[ss], sh.S[ss][cc], acc);
          w[cc] = -acc;
        }
      }
      sh.W[buf][i][0] = make_float4(w[0], w[1], w[2], w[3]);
      sh.W[buf][i][1] = make_float4(w[4], w[5], w[6], w[7]);
    }
    B8_MARK(4);
    __syncthreads();
    B8_MARK(5);
    const int f = sh.fail[buf];
    if (f >= 0) return K0 + f;
    float w[2][8];
    bool pk[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = 2 * r + u;
      const float4 wa = sh.W[buf][i][0], wb = sh.W[buf][i][1];
      w[u][0] = wa.x, w[u][1] = wa.y, w[u][2] = wa.z, w[u][3] = wa.w;
      w[u][4] = wb.x, w[u][5] = wb.y, w[u][6] = wb.z, w[u][7] = wb.w;
      pk[u] = (i >= K0 && i < K0 + 8);
    }
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const float4 ra = sh.R[buf][q * 16 + jj][0], rb = sh.R[buf][q * 16 + jj][1];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        float v = pk[u] ? 0.f : a[u][jj];
        v = fmaf(-w[u][0], ra.x, v);
        v = fmaf(-w[u][1], ra.y, v);
        v = fmaf(-w[u][2], ra.z, v);
        v = fmaf(-w[u][3], ra.w, v);
        v = fmaf(-w[u][4], rb.x, v);
        v = fmaf(-w[u][5], rb.y, v);
        v = fmaf(-w[u][6], rb.z, v);
        v = fmaf(-w[u][7], rb.w, v);
        a[u][jj] = v;
      }
    }
    if (q == (K0 >> 4)) {  // warp-uniform: the eight pivot columns of this column group
      if ((K0 & 15) == 0) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) a[u][cc] = w[u][cc];
      } else {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) a[u][8 + cc] = w[u][cc];
      }
    }
    B8_MARK(6);
  }
#ifdef SPD_PIVOT_TIMING
  if (t == 0 && blockIdx.x == 0)
    printf("b8 sweep phases (cycles over %d steps): write-R %lld sync1 %lld sweep8x8 %lld nbar %lld weights %lld sync2 %lld update %lld\n",
           nb, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6]);
#endif
  return -1;
}

// ---- v3: the 8-pivot sweep with the serial part off the bulk update's path.
// Same arithmetic as sweep128_b8v2 (8x8 block sweep S = -B^-1, row weights w_i = -W[i,K] S,
// rank-8 update W[i,j] -= w_i W[K,j] with the pivot rows' base zeroed, pivot columns <- w), but
// R_g is taken from the pivot COLUMNS (W[i, K_g], symmetric) so the two warps that hold group
// g+1's columns produce everything group g+1 needs while the other 14 warps apply group g's bulk
// update: they update those 8 columns first, publish them (R_{g+1}), sweep the 8x8 block, form
// the 128 row weights from their own registers, then finish their other 8 columns.  One block
// barrier per group instead of three, and the 8x8 sweep (~70 cycles per pivot of shuffle /
// MUFU latency) overlaps the bulk FFMA work.
struct B8v3Shared {
  float Rt[2][8][128];  // R_g^T: Rt[s][i] = W[i][K_g + s]   (buffer g & 1; column pairs feed FFMA2)
  float4 W[2][128][2];  // row weights of group g
  float S[8][8];
  int fail[2];
};

// 8x8 block B (lane: rr = lane >> 2, c = lane & 3 holds v0 = B[rr][c], v1 = B[rr][c + 4]) -> S =
// -B^-1 into S; returns the first non-positive pivot (warp-uniform) or -1.  (A variant in which every
// lane sweeps its own register copy of B, without shuffles, measured slower: 61 vs 48 us per block.)
__device__ __forceinline__ int sweep8x8(float v0, float v1, int lane, float (&S)[8][8]) {
  const int rr = lane >> 2, c = lane & 3;
  int fail = -1;
#pragma unroll
  for (int p = 0; p < 8; ++p) {  // branch-free (a `break` makes every shuffle take the divergent path)
    const float pv = __shfl_sync(0xffffffffu, (p < 4) ? v0 : v1, (p << 2) | (p & 3));
    if (fail < 0 && !(pv > 0.f)) fail = p;
    const float pinv = rcp_nr1(pv);
    const float rp0 = __shfl_sync(0xffffffffu, v0, (p << 2) | c);
    const float rp1 = __shfl_sync(0xffffffffu, v1, (p << 2) | c);
    const float cp = __shfl_sync(0xffffffffu, (p < 4) ? v0 : v1, (rr << 2) | (p & 3));
    float n0, n1;
    if (rr == p) {
      n0 = (c == p) ? -pinv : rp0 * pinv;
      n1 = (c + 4 == p) ? -pinv : rp1 * pinv;
    } else {
      n0 = (c == p) ? cp * pinv : fmaf(-cp * pinv, rp0, v0);
      n1 = (c + 4 == p) ? cp * pinv : fmaf(-cp * pinv, rp1, v1);
    }
    v0 = n0, v1 = n1;
  }
  S[rr][c] = v0;
  S[rr][c + 4] = v1;
  return fail;
}

// d = a * b + c on two fp32 lanes (FFMA2: one issue slot for two FMAs, each rounded as fmaf)
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b, c;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%0, %1};\n\t"
      "fma.rn.f32x2 c, a, b, c;\n\tmov.b64 {%0, %1}, c;\n\t}"
      : "+f"(d0), "+f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// group g's rank-8 update of this thread's columns [8H, 8H + 8) of its 16: W[i,j] = base - sum_c
// w_i[c] R[j][c] in the order c = 0..7 (base = 0 on the pivot rows), two adjacent columns per FFMA2
template <int H>
__device__ __forceinline__ void b8v3_update_half(float (&a)[2][16], const float (&wn)[2][8], const bool (&pk)[2],
                                                 const float (*Rt)[128], int q) {
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int jj = 8 * H; jj < 8 * H + 8; ++jj) a[u][jj] = pk[u] ? 0.f : a[u][jj];
#pragma unroll
  for (int jq = 0; jq < 2; ++jq) {  // 4 columns 16 q + 8 H + 4 jq .. + 3
    const int j0 = 8 * H + 4 * jq;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 r = *reinterpret_cast<const float4*>(&Rt[c][q * 16 + j0]);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        ffma2(a[u][j0], a[u][j0 + 1], wn[u][c], wn[u][c], r.x, r.y);
        ffma2(a[u][j0 + 2], a[u][j0 + 3], wn[u][c], wn[u][c], r.z, r.w);
      }
    }
  }
}

// group Kn's serial part, run by the two warps holding its columns (half H of their 16):
// publish R, sweep the 8x8 block (the warp holding rows Kn..Kn+7), form and publish the weights
template <int H>
__device__ __forceinline__ void b8v3_pivot_work(const float (&a)[2][16], int Kn, int nb, B8v3Shared& sh, int r,
                                                int lane, int warp, int qn) {
  float(*Rt)[128] = sh.Rt[nb];
#pragma unroll
  for (int ss = 0; ss < 8; ++ss)  // rows 2r, 2r + 1 are adjacent columns of R^T
    *reinterpret_cast<float2*>(&Rt[ss][2 * r]) = make_float2(a[0][8 * H + ss], a[1][8 * H + ss]);
  named_bar_sync(1, 64);
  if (warp == 2 * qn + (Kn >= 64 ? 1 : 0)) {  // rows Kn..Kn+7 live in this warp
    const int rr = lane >> 2, c = lane & 3;
    const int f = sweep8x8(Rt[c][Kn + rr], Rt[c + 4][Kn + rr], lane, sh.S);
    if (lane == 0) sh.fail[nb] = f;
  }
  named_bar_sync(1, 64);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = 2 * r + u, s0 = i - Kn;
    float wn[8];
    if (s0 >= 0 && s0 < 8) {
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) wn[cc] = sh.S[s0][cc];
    } else {
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        float acc = 0.f;
#pragma unroll
        for (int ss = 0; ss < 8; ++ss) acc = fmaf(a[u][8 * H + ss], sh.S[ss][cc], acc);
        wn[cc] = -acc;
      }
    }
    sh.W[nb][i][0] = make_float4(wn[0], wn[1], wn[2], wn[3]);
    sh.W[nb][i][1] = make_float4(wn[4], wn[5], wn[6], wn[7]);
  }
}

// one group g (P = g & 1); returns the failing pivot of group g+1 or -1
template <int P>
__device__ __forceinline__ int b8v3_step(float (&a)[2][16], int g, int ng, B8v3Shared& sh, int r, int q, int lane,
                                         int warp) {
  constexpr int H1 = P ^ 1;  // half of the column block holding group g+1
  const int buf = g & 1, nb = buf ^ 1, K0 = 8 * g, qg = g >> 1, q1 = (g + 1) >> 1;
  float wn[2][8];  // -w (the FFMA2 operand); the pivot columns get w = -wn back exactly
  bool pk[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = 2 * r + u;
    const float4 wa = sh.W[buf][i][0], wb = sh.W[buf][i][1];
    wn[u][0] = -wa.x, wn[u][1] = -wa.y, wn[u][2] = -wa.z, wn[u][3] = -wa.w;
    wn[u][4] = -wb.x, wn[u][5] = -wb.y, wn[u][6] = -wb.z, wn[u][7] = -wb.w;
    pk[u] = (i >= K0 && i < K0 + 8);
  }
  const float(*Rt)[128] = sh.Rt[buf];
  b8v3_update_half<H1>(a, wn, pk, Rt, q);
  const bool next = g + 1 < ng;
  if (next && q == q1) b8v3_pivot_work<H1>(a, K0 + 8, nb, sh, r, lane, warp, q1);
  b8v3_update_half<P>(a, wn, pk, Rt, q);
  if (q == qg) {  // group g's pivot columns (half P of column block qg) <- w
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) a[u][8 * P + cc] = -wn[u][cc];
  }
  __syncthreads();
  if (next) {
    const int f = sh.fail[nb];
    if (f >= 0) return K0 + 8 + f;
  }
  return -1;
}

// -> W[K,K] = -P^-1 in a (the same contract as sweep128_b8v2)
__device__ __forceinline__ int sweep128_b8v3(float (&a)[2][16], int n, B8v3Shared& sh) {
  const int t = threadIdx.x, r = t & 63, q = t >> 6, lane = t & 31, warp = t >> 5;
  const int ng = (n + 7) >> 3;
  if (q == 0) b8v3_pivot_work<0>(a, 0, 0, sh, r, lane, warp, 0);
  __syncthreads();
  if (sh.fail[0] >= 0) return sh.fail[0];
#pragma unroll 1
  for (int g = 0; g < ng; g += 2) {
    int f = b8v3_step<0>(a, g, ng, sh, r, q, lane, warp);
    if (f >= 0) return f;
    if (g + 1 < ng) {
      f = b8v3_step<1>(a, g + 1, ng, sh, r, q, lane, warp);
      if (f >= 0) return f;
    }
  }
  return -1;
}

__device__ __forceinline__ float packed_at(const float* p, int64_t d, int64_t i, int64_t j) {
  const int64_t r = i < j ? i : j, c = i < j ? j : i;
  return p[r * (2 * d - r + 1) / 2 + (c - r)];
}

// ---------------------------------------------------------------- 128-pivot block on tcgen05
// One CTA (256 threads = 8 warps) sweeps one 128 x 128 pivot block P.  Thread (row i, half h)
// keeps D[i][64 h, 64 h + 64) in registers (warp w: TMEM lanes / rows [32 (w % 4), +32),
// h = w / 4).  Four 32-pivot steps s (K = columns [32 s, 32 s + 32), held by half s / 2):
//   1. D[:,K] -> shared memory as the A operand; warp s + 4 (s / 2) (rows K) sweeps the 32 x 32
//      pivot block in registers in fp32 (8-pivot groups: an 8 x 8 shuffle sweep, then a rank-8
//      update) -> S_K = -P_K^-1.  The pivots are the Schur complements in order, so the first
//      non-positive one is LAPACK dpotrf's failing index;
//   2. panel C = D[:,K] P_K^-1 on the tensor cores (M = 128, N = 32);
//   3. U = A B^T, A = D[:,K], B = -C (M = N = 128) on the tensor cores; every thread adds its
//      row of U to its registers;
//   4. fix-up in registers: D[i,K] = C[i] (i not in K), D[K,j] = C[j]^T, D[K,K] = S_K.
// After the four steps D = -P^-1.
// Precision: the Schur updates inside a pivot block cancel heavily (the result is much smaller
// than |A||C|), so the products must be fp32-exact relative to |A||C|.  The operands are split
// three ways into tf32 (x = hi + mid + lo, |x - hi - mid - lo| <= 2^-33 |x|) and the six
// products above 2^-33 are issued into TWO accumulators: hi*hi alone (4 accumulating MMAs: the
// tcgen05 accumulation truncates, ~2^-24 per MMA, so it stays at the fp32 FFMA level) and the five
// cross terms (magnitude <= 2^-11 of it) in the other; the two are summed in registers with
// round-to-nearest adds.  (A 2-way split into one accumulator measured 10-35x larger inverse
// errors on rank-deficient factors than fp32 FFMA and failed pivots inside the bench step.)
#ifdef SPD_PIVOT_TIMING  // per-phase clock64 marks of thread 0, printed by block 0 (diagnostic build)
#define PVT_MARK(slot) \
  do {                 \
    if (threadIdx.x == 0) clk[slot] = clock64(); \
  } while (0)
#else
#define PVT_MARK(slot) \
  do {                 \
  } while (0)
#endif
namespace pvt {
constexpr int kThreads = 256;
constexpr int kLd = 33;                   // C fp32 [128][kLd]: conflict-free columns
constexpr int kFLd = 132;                 // 128 x 128 fp32 staging rows (float4-aligned)
constexpr int kGLd = 36;                  // 8 published rows of the 32 x 32 sweep
constexpr uint32_t kOpBytes = 128 * 128;  // one 128 x 32 fp32 operand plane (128-B rows, SWIZZLE_128B)
constexpr uint32_t kPBytes = 32 * 128;    // one 32 x 32 fp32 operand plane
// smem: [opA hi, mid, lo | opB hi, mid, lo | opP hi, mid, lo | C fp32 | sweep rows | barrier];
// the 128 x 132 fp32 staging of the global load / store overlays the front
constexpr uint32_t kOffB = 3 * kOpBytes, kOffP = 6 * kOpBytes, kOffC = kOffP + 3 * kPBytes;
constexpr uint32_t kOffG = kOffC + 128 * kLd * 4, kOffBar = kOffG + 8 * kGLd * 4;
constexpr size_t kSmem = 1024 + size_t(kOffBar) + 64;
static_assert(128 * kFLd * 4 <= kOffBar, "staging overlay fits");
// TMEM columns: U hi*hi [0, 128), U cross terms [128, 256), C hi*hi [256, 288), C cross [288, 320)
constexpr uint32_t kTU1 = 0, kTU2 = 128, kTC1 = 256, kTC2 = 288;
// byte offset of 16-B chunk `chunk` of row i in a K-major x 32 fp32 plane with the 128-B swizzle
__device__ __forceinline__ uint32_t sw128(int i, int chunk) { return uint32_t(i) * 128u + (uint32_t(chunk ^ (i & 7)) << 4); }
__device__ __forceinline__ void split3(float x, float& h, float& m, float& l) {
  h = tf32_rna(x);
  const float r = x - h;
  m = tf32_rna(r);
  l = tf32_rna(r - m);
}
// three tf32 planes (hi, mid, lo) of one 16-B chunk
__device__ __forceinline__ void put_split3(uint8_t* plane0, uint32_t plane_bytes, uint32_t off, float4 x) {
  float4 h, m, l;
  split3(x.x, h.x, m.x, l.x);
  split3(x.y, h.y, m.y, l.y);
  split3(x.z, h.z, m.z, l.z);
  split3(x.w, h.w, m.w, l.w);
  *reinterpret_cast<float4*>(plane0 + off) = h;
  *reinterpret_cast<float4*>(plane0 + plane_bytes + off) = m;
  *reinterpret_cast<float4*>(plane0 + 2 * plane_bytes + off) = l;
}
// the six split products of one 128 x N tile over K = 32: hi*hi into acc1, the cross terms into acc2
template <int N>
__device__ __forceinline__ void mma_split3(uint32_t acc1, uint32_t acc2, const uint8_t* a, uint32_t a_plane,
                                           const uint8_t* b, uint32_t b_plane) {
  constexpr uint32_t idesc = make_idesc<Kind::TF32>(128, N);
  const uint64_t ah = make_sdesc_sw128(a), am = make_sdesc_sw128(a + a_plane), al = make_sdesc_sw128(a + 2 * a_plane);
  const uint64_t bh = make_sdesc_sw128(b), bm = make_sdesc_sw128(b + b_plane), bl = make_sdesc_sw128(b + 2 * b_plane);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {  // 4 x 32 B of K per 128-B swizzle row
    const uint64_t off = uint64_t(kk * 2);
    umma<Kind::TF32>(acc1, ah + off, bh + off, idesc, kk != 0);
    umma<Kind::TF32>(acc2, ah + off, bm + off, idesc, kk != 0);
    umma<Kind::TF32>(acc2, am + off, bh + off, idesc, 1u);
    umma<Kind::TF32>(acc2, ah + off, bl + off, idesc, 1u);
    umma<Kind::TF32>(acc2, am + off, bm + off, idesc, 1u);
    umma<Kind::TF32>(acc2, al + off, bh + off, idesc, 1u);
  }
}
__device__ __forceinline__ float rcp_nr(float x) {  // reciprocal: MUFU approximation + one Newton step
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r * fmaf(-x, r, 2.f);
}
// Sweep the 32 x 32 block held by one warp (lane r = row r, w[t] = D[r][t]) -> -D^-1; returns the
// first non-positive pivot (warp-uniform) or -1.  Groups g of 8 pivots: the row is kept rotated
// by 8 g so that the group's columns sit in w[0..8).  buf: [8][kGLd] shared scratch of this warp.
__device__ __forceinline__ int sweep32(float (&w)[32], int lane, float* buf) {
  int fail = -1;
#pragma unroll 1
  for (int g = 0; g < 4; ++g) {
    // (1) 8 x 8 diagonal block B = W[G,G] (rows in lanes 8g..8g+7) -> S = -B^-1 (shuffles)
    float b[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) b[c] = w[c];
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // branch-free: the row shuffles issue together with the pivot's
      const int p = 8 * g + u;
      float rp[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) rp[c] = __shfl_sync(0xffffffffu, b[c], p);
      const float piv = rp[u];
      if (fail < 0 && !(piv > 0.f)) fail = p;  // warp-uniform (broadcast value); NaN fails too
      const float rinv = rcp_nr(piv);
      const bool me = lane == p;
      const float fct = b[u] * rinv;
      const float mult = me ? rinv : -fct;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c != u) b[c] = fmaf(mult, rp[c], me ? 0.f : b[c]);
      b[u] = me ? -rinv : fct;
    }
    if (fail >= 0) break;
    // (2) rows G publish [S_r | W[G_r, 8..32)]
    const bool inG = (lane >> 3) == g;
    if (inG) {
      float* row = buf + (lane & 7) * kGLd;
      *reinterpret_cast<float4*>(row) = make_float4(b[0], b[1], b[2], b[3]);
      *reinterpret_cast<float4*>(row + 4) = make_float4(b[4], b[5], b[6], b[7]);
#pragma unroll
      for (int t = 0; t < 6; ++t)
        *reinterpret_cast<float4*>(row + 8 + 4 * t) = make_float4(w[8 + 4 * t], w[9 + 4 * t], w[10 + 4 * t], w[11 + 4 * t]);
    }
    __syncwarp();
    // (3) rank-8 update.  Row i not in G: y = W[i,G] B^-1 = -W[i,G] S, W[i,j] -= y W[G,j], W[i,G] = y.
    //     Row r in G: W[G_r,j] = B^-1 W[G,j] = -S_r W[G,j], W[G_r,G] = S_r.  One code path:
    //     coef = inG ? S_r : y, base = inG ? 0 : W[i,j], W[i,j] = base - coef W[G,j].
    float y[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float4 s0 = *reinterpret_cast<const float4*>(buf + m * kGLd);
      const float4 s1 = *reinterpret_cast<const float4*>(buf + m * kGLd + 4);
      const float wm = w[m];
      y[0] = fmaf(-wm, s0.x, y[0]), y[1] = fmaf(-wm, s0.y, y[1]), y[2] = fmaf(-wm, s0.z, y[2]);
      y[3] = fmaf(-wm, s0.w, y[3]), y[4] = fmaf(-wm, s1.x, y[4]), y[5] = fmaf(-wm, s1.y, y[5]);
      y[6] = fmaf(-wm, s1.z, y[6]), y[7] = fmaf(-wm, s1.w, y[7]);
    }
    float coef[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) coef[c] = inG ? b[c] : y[c];
#pragma unroll
    for (int t = 8; t < 32; ++t) w[t] = inG ? 0.f : w[t];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const float4 g4 = *reinterpret_cast<const float4*>(buf + m * kGLd + 8 + 4 * t);
        w[8 + 4 * t] = fmaf(-coef[m], g4.x, w[8 + 4 * t]);
        w[9 + 4 * t] = fmaf(-coef[m], g4.y, w[9 + 4 * t]);
        w[10 + 4 * t] = fmaf(-coef[m], g4.z, w[10 + 4 * t]);
        w[11 + 4 * t] = fmaf(-coef[m], g4.w, w[11 + 4 * t]);
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) w[c] = coef[c];
    __syncwarp();  // buf is rewritten by the next group
    float tmp[8];  // rotate left by 8: the next group's columns move to w[0..8)
#pragma unroll
    for (int t = 0; t < 8; ++t) tmp[t] = w[t];
#pragma unroll
    for (int t = 0; t < 24; ++t) w[t] = w[t + 8];
#pragma unroll
    for (int t = 0; t < 8; ++t) w[24 + t] = tmp[t];
  }
  return fail;
}
}  // namespace pvt

// kSmall: the whole matrix (d <= 128, packed input + gamma I, identity padding) -> out =
// -(D + D^T)/2 cropped to d x d.  Otherwise: pivot block k of a blocked matrix (W[K,K]) ->
// W[K,K] = -P^-1 and P^-1 as tf32 hi/lo planes for the panel GEMM.
template <bool kSmall>
__global__ void __launch_bounds__(pvt::kThreads, 1)
    pivot_tc_kernel(const InvMat* __restrict__ mats, const int32_t* __restrict__ ids, int k,
                    void* __restrict__ pinv_planes, int64_t pinv_plane, int f16, float gamma, Probe* probe) {
  using namespace pvt;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_align1024(smem_raw);
  uint8_t* opA = sm;          // A = D[:,K]: hi, mid, lo planes
  uint8_t* opB = sm + kOffB;  // B = -C
  uint8_t* opP = sm + kOffP;  // P_K^-1 (32 rows)
  float* Cs = reinterpret_cast<float*>(sm + kOffC);
  float* gbuf = reinterpret_cast<float*>(sm + kOffG);
  float* F = reinterpret_cast<float*>(sm);  // 128 x kFLd staging overlay (load / store)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kOffBar);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  int* sfail = reinterpret_cast<int*>(tslot + 1);
#ifdef SPD_PIVOT_TIMING
  long long clk[32];
#endif
  PVT_MARK(0);
  probe_start(probe);

  const InvMat m = mats[ids[blockIdx.x]];
  if constexpr (!kSmall) {
    if (*m.info != 0) {  // an earlier pivot block failed (uniform)
      probe_stop(probe);
      return;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, h = warp >> 2, i = 32 * q + lane;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tslot);
  const int n = kSmall ? m.d : kB;
  const int64_t dp = m.dp, K0 = int64_t(k) * kB;

  float d[64];  // D[i][64 h + t]
  if constexpr (kSmall) {
#pragma unroll
    for (int t = 0; t < 64; ++t) {
      const int j = 64 * h + t;
      d[t] = (i < n && j < n) ? packed_at(m.in, n, i, j) + (i == j ? gamma : 0.f) : (i == j ? 1.f : 0.f);
    }
  } else {  // coalesced: warp w loads rows 16 w .. 16 w + 15, one 512-B row per instruction
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int row = 16 * warp + r;
      const float4 x = __ldcg(reinterpret_cast<const float4*>(m.W + (K0 + row) * dp + K0) + lane);
      *reinterpret_cast<float4*>(F + row * kFLd + 4 * lane) = x;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const float4 x = *reinterpret_cast<const float4*>(F + i * kFLd + 64 * h + 4 * t);
      d[4 * t] = x.x, d[4 * t + 1] = x.y, d[4 * t + 2] = x.z, d[4 * t + 3] = x.w;
    }
  }
  tc_fence_before();
  __syncthreads();  // (the staging overlay is free again; TMEM allocated)
  tc_fence_after();
  PVT_MARK(1);
  const uint32_t tbase = *tslot;
  const uint32_t tq = tbase + (uint32_t(32 * q) << 16);  // this warp's lane quarter

  const int nsteps = (n + 31) >> 5;
  int fail = -1;
  uint32_t phase = 0;
#pragma unroll 1
  for (int s = 0; s < nsteps; ++s) {
    const int hs = s >> 1;
    const bool odd = s & 1;
    // ---- 1. A = D[:,K] -> shared memory; the pivot warp sweeps P_K -> S_K, publishes P_K^-1
    float a[32];
    if (h == hs) {
#pragma unroll
      for (int t = 0; t < 32; ++t) a[t] = odd ? d[32 + t] : d[t];
#pragma unroll
      for (int t = 0; t < 8; ++t)
        put_split3(opA, kOpBytes, sw128(i, t), make_float4(a[4 * t], a[4 * t + 1], a[4 * t + 2], a[4 * t + 3]));
      if (q == s) {
        const int f = sweep32(a, lane, gbuf);
#pragma unroll
        for (int t = 0; t < 8; ++t)  // P_K^-1 = -S_K, row `lane`
          put_split3(opP, kPBytes, sw128(lane, t), make_float4(-a[4 * t], -a[4 * t + 1], -a[4 * t + 2], -a[4 * t + 3]));
        if (lane == 0) *sfail = f;
      }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    PVT_MARK(2 + 4 * s);
    const int f = *sfail;
    if (f >= 0) {  // uniform
      fail = 32 * s + f;
      break;
    }
    // ---- 2. C = A P_K^-1 on the tensor cores
    if (threadIdx.x == 0) {
      tc_fence_after();
      mma_split3<32>(tbase + kTC1, tbase + kTC2, opA, kOpBytes, opP, kPBytes);
      tc_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    tc_fence_after();
    float c[32];  // C[i][0..32)
    {
      uint32_t c1[32], c2[32];
      tmem_ld_32x32b_x32_nowait(tq + kTC1, c1);
      tmem_ld_32x32b_x32_nowait(tq + kTC2, c2);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 32; ++t) c[t] = __uint_as_float(c1[t]) + __uint_as_float(c2[t]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {  // this thread's 16 columns of -C -> the B operand, C -> Cs
      const float4 lo4 = make_float4(-c[4 * t], -c[4 * t + 1], -c[4 * t + 2], -c[4 * t + 3]);
      const float4 hi4 = make_float4(-c[16 + 4 * t], -c[17 + 4 * t], -c[18 + 4 * t], -c[19 + 4 * t]);
      put_split3(opB, kOpBytes, sw128(i, 4 * h + t), h ? hi4 : lo4);
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) Cs[i * kLd + 16 * h + t] = h ? c[16 + t] : c[t];
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    PVT_MARK(3 + 4 * s);
    // ---- 3. U = A B^T on the tensor cores, D += U in registers
    if (threadIdx.x == 0) {
      tc_fence_after();
      mma_split3<128>(tbase + kTU1, tbase + kTU2, opA, kOpBytes, opB, kOpBytes);
      tc_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    tc_fence_after();
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t u1[32], u2[32];
      tmem_ld_32x32b_x32_nowait(tq + kTU1 + 64 * h + 32 * half, u1);
      tmem_ld_32x32b_x32_nowait(tq + kTU2 + 64 * h + 32 * half, u2);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 32; ++t) d[32 * half + t] += __uint_as_float(u1[t]) + __uint_as_float(u2[t]);
    }
    PVT_MARK(4 + 4 * s);
    // ---- 4. fix-up of row / column block K
    if (q != s) {
      if (h == hs) {  // D[i,K] = C[i]
        if (odd) {
#pragma unroll
          for (int t = 0; t < 32; ++t) d[32 + t] = c[t];
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) d[t] = c[t];
        }
      }
    } else {  // rows K: D[K,j] = C[j]^T (j not in K), D[K,K] = S_K (the sweeping warp's registers)
      if (h == hs) {
        if (odd) {
#pragma unroll
          for (int t = 0; t < 32; ++t) d[t] = Cs[(64 * h + t) * kLd + lane], d[32 + t] = a[t];
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) d[t] = a[t], d[32 + t] = Cs[(64 * h + 32 + t) * kLd + lane];
        }
      } else {
#pragma unroll
        for (int t = 0; t < 64; ++t) d[t] = Cs[(64 * h + t) * kLd + lane];
      }
    }
    tc_fence_before();
    __syncthreads();  // shared staging and the TMEM accumulators are reused by the next step
    tc_fence_after();
    PVT_MARK(5 + 4 * s);
  }
  PVT_MARK(26);

  if (fail >= 0) {
    if (threadIdx.x == 0) *m.info = int(kSmall ? 0 : K0) + fail + 1;
  } else {
#pragma unroll
    for (int t = 0; t < 16; ++t)
      *reinterpret_cast<float4*>(F + i * kFLd + 64 * h + 4 * t) = make_float4(d[4 * t], d[4 * t + 1], d[4 * t + 2], d[4 * t + 3]);
    __syncthreads();
    if constexpr (!kSmall) {  // W[K,K] <- -P^-1 and P^-1 hi / lo planes, whole rows per warp instruction
      const int64_t pbase = int64_t(m.slot) * kB * kB;
      const float sc = f16 ? m.scale[kScInv] : 1.f;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int row = 16 * warp + r;
        const float4 x = *reinterpret_cast<const float4*>(F + row * kFLd + 4 * lane);
        reinterpret_cast<float4*>(m.W + (K0 + row) * dp + K0)[lane] = x;
        if (f16) {  // fp16 planes of P^-1 * s
          __half* ph = static_cast<__half*>(pinv_planes) + pbase + row * kB + 4 * lane;
          __half h0, l0, h1, l1, h2, l2, h3, l3;
          split_f16(-x.x, sc, h0, l0);
          split_f16(-x.y, sc, h1, l1);
          split_f16(-x.z, sc, h2, l2);
          split_f16(-x.w, sc, h3, l3);
          *reinterpret_cast<uint2*>(ph) =
              make_uint2(uint32_t(__half_as_ushort(h0)) | (uint32_t(__half_as_ushort(h1)) << 16),
                         uint32_t(__half_as_ushort(h2)) | (uint32_t(__half_as_ushort(h3)) << 16));
          *reinterpret_cast<uint2*>(ph + pinv_plane) =
              make_uint2(uint32_t(__half_as_ushort(l0)) | (uint32_t(__half_as_ushort(l1)) << 16),
                         uint32_t(__half_as_ushort(l2)) | (uint32_t(__half_as_ushort(l3)) << 16));
          continue;
        }
        float* ph = static_cast<float*>(pinv_planes) + pbase;
        float4 hi, lo;
        split_tf32(-x.x, hi.x, lo.x);
        split_tf32(-x.y, hi.y, lo.y);
        split_tf32(-x.z, hi.z, lo.z);
        split_tf32(-x.w, hi.w, lo.w);
        reinterpret_cast<float4*>(ph + row * kB)[lane] = hi;
        reinterpret_cast<float4*>(ph + pinv_plane + row * kB)[lane] = lo;
      }
    } else {  // out = -(D + D^T)/2 cropped
      for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int r = e / n, cc = e - r * n;
        m.out[e] = -0.5f * (F[r * kFLd + cc] + F[cc * kFLd + r]);
      }
      if (threadIdx.x == 0) *m.info = 0;
    }
  }
  PVT_MARK(27);
#ifdef SPD_PIVOT_TIMING
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    printf("pivot k=%d load %lld |", k, clk[1] - clk[0]);
    for (int s2 = 0; s2 < 4; ++s2)
      printf(" s%d: sweep %lld panel %lld update %lld fix %lld |", s2, clk[2 + 4 * s2] - clk[s2 ? 1 + 4 * s2 : 1],
             clk[3 + 4 * s2] - clk[2 + 4 * s2], clk[4 + 4 * s2] - clk[3 + 4 * s2], clk[5 + 4 * s2] - clk[4 + 4 * s2]);
    printf(" out %lld total %lld\n", clk[27] - clk[26], clk[27] - clk[0]);
  }
#endif
  tc_fence_before();
  __syncthreads();
  probe_stop(probe);
  if (warp == 0) tmem_free<512>(tbase);
}

// ---------------------------------------------------------------- d <= 128
template <bool kV3>
__global__ void __launch_bounds__(512) small_inverse_kernel(const InvMat* __restrict__ mats,
                                                            const int32_t* __restrict__ ids, float gamma,
                                                            Probe* probe) {
  __shared__ std::conditional_t<kV3, B8v3Shared, B8v2Shared> sh;
  probe_start(probe);
  const InvMat m = mats[ids[blockIdx.x]];
  const int n = m.d;
  const int r = threadIdx.x & 63, q = threadIdx.x >> 6;
  float a[2][16];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = 2 * r + u;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = q * 16 + jj;
      a[u][jj] = (i < n && j < n) ? packed_at(m.in, n, i, j) + (i == j ? gamma : 0.f) : (i == j ? 1.f : 0.f);
    }
  }
  int f;
  if constexpr (kV3) f = sweep128_b8v3(a, n, sh);
  else f = sweep128_b8v2(a, n, sh);
  if (f >= 0) {
    if (threadIdx.x == 0) *m.info = f + 1;
    probe_stop(probe);
    return;
  }
  if (threadIdx.x == 0) *m.info = 0;
  // out = -(S + S^T)/2 through shared memory (uniform control flow)
  extern __shared__ float sm[];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) sm[(2 * r + u) * kSmemLd + q * 16 + jj] = -a[u][jj];
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int rr = e / n, c = e - rr * n;
    m.out[e] = 0.5f * (sm[rr * kSmemLd + c] + sm[c * kSmemLd + rr]);
  }
  __syncthreads();
  probe_stop(probe);
}

// ---------------------------------------------------------------- blocked path
// W = unpack(packed) + gamma I, identity padding; one 64x64 tile (I <= J) per block, 256
// threads x 16 elements, every load issued before the first store.  Only the upper block
// triangle of W is ever read (pivot: diagonal 128-blocks; panel, update, finalize: blocks
// (I, J) with I <= J), so the mirrored (J, I) tile is written only inside a diagonal
// 128-block.
constexpr int kT = 64;  // unpack / finalize tile edge
__global__ void __launch_bounds__(256) damp_unpack_kernel(const InvMat* __restrict__ mats,
                                                          const TileJob* __restrict__ jobs, float gamma, float pad) {
  __shared__ float tile[kT][kT + 1];
  const TileJob jb = jobs[blockIdx.x];
  const InvMat m = mats[jb.mat];
  const int64_t d = m.d, dp = m.dp;
  if (jb.ti == 0 && jb.tj == 0 && threadIdx.x == 0) *m.info = 0;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  const int64_t i0 = int64_t(jb.ti) * kT, j0 = int64_t(jb.tj) * kT;
  const bool diag = jb.ti == jb.tj;
  const bool mirror = !diag && (jb.ti >> 1) == (jb.tj >> 1);  // both halves of a diagonal 128-block
  float v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int64_t i = i0 + ty + 4 * u, j = j0 + tx;
    const int64_t r = i < j ? i : j, c = i < j ? j : i;  // diagonal tile: the lower half reads (j, i)
    v[u] = (c < d) ? __ldcs(m.in + r * (2 * d - r + 1) / 2 + (c - r)) : 0.f;
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int64_t i = i0 + ty + 4 * u, j = j0 + tx;
    if (i == j) v[u] = (i < d) ? v[u] + gamma : pad;  // padding: decoupled unit (tf32) or gamma (fp16) pivots
    m.W[i * dp + j] = v[u];
    if (mirror) tile[ty + 4 * u][tx] = v[u];
  }
  if (mirror) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) m.W[(j0 + ty + 4 * u) * dp + i0 + tx] = tile[tx][ty + 4 * u];  // (J, I)
  }
}

// Operand classes of the fp16 planes and their bounds over the whole sweep (F + gamma I with
// sigma = max(max_i (F_ii + gamma), 1), the 1 covering the identity padding):
//   kScInv   entries of inverses of principal submatrices (P^-1, panel rows already swept):
//            |(A_PP^-1)_ij| <= 1 / lambda_min(A_PP) <= 1 / gamma
//   kScReg   regression blocks A_PP^-1 A_PQ (old panel rows already swept, new panel rows not yet
//            swept): |.| <= sqrt((A_PP^-1)_ii A_jj) <= sqrt(sigma / gamma)
//   kScSchur Schur complements (old panel rows not yet swept): |S_ij| <= sqrt(S_ii S_jj) <= sigma
// Each class gets s = 2^(13 - ceil(log2 bound)), so |x s| <= 2^13 (fp16 max 65504: 8x headroom for
// rounding) and the split hi + lo keeps every entry to 2^-22 relative or 2^-38 x bound absolute.
__device__ __forceinline__ float class_scale(float bound) {
  int e = 0;
  if (isfinite(bound)) frexpf(bound, &e);  // bound <= 2^e (NaN / inf diagonals: the sweep reports them)
  e = max(min(e, 76), -100);               // the epilogue's 1 / (s_A s_B) stays finite
  return ldexpf(1.f, 13 - e);
}
__global__ void __launch_bounds__(256) inv_scale_kernel(const InvMat* __restrict__ mats,
                                                        const int32_t* __restrict__ ids, float gamma) {
  __shared__ float red[8];
  const InvMat m = mats[ids[blockIdx.x]];
  const int64_t d = m.d;
  float mx = gamma;  // the padding pivots are gamma
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) mx = fmaxf(mx, m.in[i * (2 * d - i + 1) / 2] + gamma);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float sig = red[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) sig = fmaxf(sig, red[w]);
    m.scale[kScInv] = class_scale(1.f / gamma);
    m.scale[kScReg] = class_scale(sqrtf(sig / gamma));
    m.scale[kScSchur] = class_scale(sig);
    m.scale[3] = sig / gamma;  // the accuracy model's range (diagnostics)
  }
}

template <bool kV3>
__global__ void __launch_bounds__(512) pivot_kernel(const InvMat* __restrict__ mats,
                                                    const int32_t* __restrict__ ids, int k,
                                                    void* __restrict__ pinv_planes, int64_t pinv_plane, int f16,
                                                    Probe* probe) {
  __shared__ std::conditional_t<kV3, B8v3Shared, B8v2Shared> sh;
  probe_start(probe);
  const InvMat m = mats[ids[blockIdx.x]];
  if (*m.info != 0) {
    probe_stop(probe);
    return;
  }
  const int64_t dp = m.dp, K0 = int64_t(k) * kB;
  const int r = threadIdx.x & 63, q = threadIdx.x >> 6;
  float a[2][16];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const float* src = m.W + (K0 + 2 * r + u) * dp + K0 + q * 16;
#pragma unroll
    for (int jj = 0; jj < 16; jj += 4) {
      const float4 v = *reinterpret_cast<const float4*>(src + jj);
      a[u][jj] = v.x, a[u][jj + 1] = v.y, a[u][jj + 2] = v.z, a[u][jj + 3] = v.w;
    }
  }
  int f;
  if constexpr (kV3) f = sweep128_b8v3(a, kB, sh);
  else f = sweep128_b8v2(a, kB, sh);
  if (f >= 0) {
    if (threadIdx.x == 0) *m.info = int(K0) + f + 1;
    probe_stop(probe);
    return;
  }
  const float sc = f16 ? m.scale[kScInv] : 1.f;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = 2 * r + u;
    float* dst = m.W + (K0 + i) * dp + K0 + q * 16;                           // W[K,K] <- -P^-1
    const int64_t po = (int64_t(m.slot) * kB + i) * kB + q * 16;             // P^-1 hi plane
#pragma unroll
    for (int jj = 0; jj < 16; jj += 4)
      *reinterpret_cast<float4*>(dst + jj) = make_float4(a[u][jj], a[u][jj + 1], a[u][jj + 2], a[u][jj + 3]);
    if (f16) {  // fp16 planes of P^-1 * s (uniform branch)
      __half* ph = static_cast<__half*>(pinv_planes) + po;
#pragma unroll
      for (int jj = 0; jj < 16; jj += 8) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          __half h0, l0, h1, l1;
          split_f16(-a[u][jj + 2 * v], sc, h0, l0);
          split_f16(-a[u][jj + 2 * v + 1], sc, h1, l1);
          hw[v] = uint32_t(__half_as_ushort(h0)) | (uint32_t(__half_as_ushort(h1)) << 16);
          lw[v] = uint32_t(__half_as_ushort(l0)) | (uint32_t(__half_as_ushort(l1)) << 16);
        }
        *reinterpret_cast<uint4*>(ph + jj) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(ph + pinv_plane + jj) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    } else {
      float* ph = static_cast<float*>(pinv_planes) + po;
#pragma unroll
      for (int jj = 0; jj < 16; jj += 4) {
        float h[4], l[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) split_tf32(-a[u][jj + v], h[v], l[v]);
        *reinterpret_cast<float4*>(ph + jj) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(ph + pinv_plane + jj) = make_float4(l[0], l[1], l[2], l[3]);
      }
    }
  }
  __syncthreads();
  probe_stop(probe);
}

struct PanelJob {
  int32_t mat, rb;  // matrix, row block R != K
};

// Old column panel Wold[R, K] -> tf32 hi/lo planes panA[prow(R) + i][j].  Only the upper
// block triangle of W is maintained, so blocks below the pivot (R > K) are read as
// W[K, R]^T through a shared-memory transpose.  Block (job, quarter q) writes panel rows
// [32q, 32q + 32); every thread issues all of its loads before its first store.
template <bool kF16>  // fp16 planes of x * s (InvMat::scale) instead of tf32 planes
__global__ void __launch_bounds__(256) stage_panel_kernel(const InvMat* __restrict__ mats,
                                                          const PanelJob* __restrict__ jobs, int k,
                                                          void* __restrict__ panA_, int64_t plane) {
  using PT = std::conditional_t<kF16, __half, float>;
  PT* panA = static_cast<PT*>(panA_);
  __shared__ float tile[128][33];
  const PanelJob jb = jobs[blockIdx.x];
  const InvMat m = mats[jb.mat];
  if (*m.info != 0) return;
  const int q = blockIdx.y;
  const int64_t dp = m.dp, K0 = int64_t(k) * kB, R0 = int64_t(jb.rb) * kB;
  PT* dst = panA + (int64_t(m.panel_row0) + R0 + 32 * q) * kPanCols;  // panA: slot base
  const float sc = kF16 ? m.scale[jb.rb < k ? kScReg : kScSchur] : 1.f;  // swept rows: A_PP^-1 A_PK
  const float* __restrict__ W = m.W;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  if (jb.rb < k) {  // rows R0 + 32q + i, columns K0 + c: 32 x 128 floats, 4 float4 per thread
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + 256 * u, i = e >> 5, c = (e & 31) * 4;
      v[u] = __ldcg(reinterpret_cast<const float4*>(W + (R0 + 32 * q + i) * dp + K0 + c));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + 256 * u, i = e >> 5, c = (e & 31) * 4;
      if constexpr (kF16) {
        __half h0, l0, h1, l1, h2, l2, h3, l3;
        split_f16(v[u].x, sc, h0, l0);
        split_f16(v[u].y, sc, h1, l1);
        split_f16(v[u].z, sc, h2, l2);
        split_f16(v[u].w, sc, h3, l3);
        *reinterpret_cast<uint2*>(dst + i * kPanCols + c) =
            make_uint2(uint32_t(__half_as_ushort(h0)) | (uint32_t(__half_as_ushort(h1)) << 16),
                       uint32_t(__half_as_ushort(h2)) | (uint32_t(__half_as_ushort(h3)) << 16));
        *reinterpret_cast<uint2*>(dst + plane + i * kPanCols + c) =
            make_uint2(uint32_t(__half_as_ushort(l0)) | (uint32_t(__half_as_ushort(l1)) << 16),
                       uint32_t(__half_as_ushort(l2)) | (uint32_t(__half_as_ushort(l3)) << 16));
      } else {
        float h[4], l[4];
        split_tf32(v[u].x, h[0], l[0]);
        split_tf32(v[u].y, h[1], l[1]);
        split_tf32(v[u].z, h[2], l[2]);
        split_tf32(v[u].w, h[3], l[3]);
        *reinterpret_cast<float4*>(dst + i * kPanCols + c) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(dst + plane + i * kPanCols + c) = make_float4(l[0], l[1], l[2], l[3]);
      }
    }
  } else {  // panel row 32q + r, column j = W[K0 + j][R0 + 32q + r]
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldcg(W + (K0 + ty + 8 * u) * dp + R0 + 32 * q + tx);
#pragma unroll
    for (int u = 0; u < 16; ++u) tile[ty + 8 * u][tx] = v[u];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {  // output row r = ty + 8 (u & 3), column j = tx + 32 (u >> 2)
      const int r = ty + 8 * (u & 3), j = tx + 32 * (u >> 2);
      if constexpr (kF16) {
        __half h, l;
        split_f16(tile[j][r], sc, h, l);
        dst[r * kPanCols + j] = h;
        dst[plane + r * kPanCols + j] = l;
      } else {
        float h, l;
        split_tf32(tile[j][r], h, l);
        dst[r * kPanCols + j] = h;
        dst[plane + r * kPanCols + j] = l;
      }
    }
  }
}

// out = -(W + W^T)/2 cropped to d x d, one 64x64 tile pair (I <= J) per block.  Inside a
// diagonal 128-block both triangles are valid and are averaged; elsewhere only the upper
// block triangle is valid and is mirrored.
__global__ void __launch_bounds__(256) finalize_kernel(const InvMat* __restrict__ mats,
                                                       const TileJob* __restrict__ jobs) {
  __shared__ float tile[kT][kT + 1];
  const TileJob jb = jobs[blockIdx.x];
  const InvMat m = mats[jb.mat];
  if (*m.info != 0) return;
  const int64_t d = m.d, dp = m.dp;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  const int64_t i0 = int64_t(jb.ti) * kT, j0 = int64_t(jb.tj) * kT;
  if (i0 >= d || j0 >= d) return;
  const bool same_block = (jb.ti >> 1) == (jb.tj >> 1);
  float v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) v[u] = __ldcs(m.W + (i0 + ty + 4 * u) * dp + j0 + tx);
  if (same_block) {  // W[J, I] rows, coalesced, transposed through shared memory
    float w[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) w[u] = __ldcs(m.W + (j0 + ty + 4 * u) * dp + i0 + tx);
#pragma unroll
    for (int u = 0; u < 16; ++u) tile[ty + 4 * u][tx] = w[u];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = -0.5f * (v[u] + tile[tx][ty + 4 * u]);
    __syncthreads();
  } else {
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = -v[u];
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int64_t i = i0 + ty + 4 * u, j = j0 + tx;
    if (i < d && j < d) m.out[i * d + j] = v[u];
    tile[ty + 4 * u][tx] = v[u];
  }
  if (jb.ti != jb.tj) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {  // out[j0 + r][i0 + tx] = v(i0 + tx, j0 + r)
      const int64_t j = j0 + ty + 4 * u, i = i0 + tx;
      if (i < d && j < d) m.out[j * d + i] = tile[tx][ty + 4 * u];
    }
  }
}

}  // namespace spd

using namespace spd;

struct spdkfac_inverse_plan {
  int n;
  std::vector<int32_t> dims;
  double small_flops = 0;       // sum d^3 of the register path (algorithmic potrf+potri)
  double algo_flops = 0;        // sum d^3 over all matrices
  InvMat* mats;                 // device
  int32_t* small_ids;           // device
  int n_small;
  int32_t* blocked_ids;         // device
  int n_blocked;
  int steps;
  std::vector<int> act_off, act_cnt, pan_off, pan_cnt, upd_off, upd_cnt, pj_off, u1_cnt;
  std::vector<int> u1d_cnt;     // per step: U1 items of the diagonal tile (k+1, k+1), first in U1
  bool diag_first = true;       // pivot(k+1) starts after U1's diagonal tiles (SPDKFAC_DIAG_FIRST=0: after all of U1)
  cudaEvent_t ev_diag = nullptr;
  std::vector<double> upd_flops, u2_flops;  // per step: U1 / U2 tensor work (algorithmic, per launch)
  cudaStream_t side = nullptr;  // look-ahead stream: pivot/stage/panel of step k+1
  bool lookahead = true;        // SPDKFAC_NO_LOOKAHEAD=1 serialises (diagnostics)
  bool legacy_pivot = true;     // fp32 FFMA pivot sweep; SPDKFAC_PIVOT=tc: the tcgen05 pivot kernel
  bool pivot_v3 = true;         // the pipelined 8-pivot sweep; SPDKFAC_PIVOT=b8: round-2 v2 sweep (A/B)
  // panel / update operands as scaled fp16 planes (kind::f16) for runs with gamma >= kF16MinGamma;
  // SPDKFAC_INV_TF32=1 (or the CTA-pair update engine) keeps every run on tf32 planes
  bool f16 = true;
  int panel_ctas = 0;           // grid cap of the panel GEMM (SPDKFAC_PANEL_CTAS; 0 = all SMs: the chain latency wins)
  cudaEvent_t ev_u1 = nullptr, ev_panel = nullptr;
  int32_t* act_ids;             // device, active blocked matrices per step (concatenated)
  PanelJob* pan_jobs;           // device, (matrix, R != K) per step, same order as the panel items
  TileJob* tiles;               // device, 32x32 tile pairs of all blocked matrices
  int n_tiles;
  CUtensorMap* maps;            // [0] panA, [1] panC, [2] P^-1, [3], [4] unused, [5 + slot] W_slot tiles
  TcItem* items;                // per step: panel GEMM items then update items
  CUtensorMap* maps16;          // the same over fp16 planes
  TcItem* items16;              // the same with K blocks of 64 (fp16)
  TcEpi* epis16;
  TcPairCItem* pitems;          // per step: CTA-pair super tiles of the bulk update (U2)
  TcPairCItem* pitems16;        // the same with K blocks of 64 (fp16)
  std::vector<int> pu_off, pu_cnt;
  std::vector<double> pu_flops;
  TcEpi* epis;                  // [0, n): update, [n + q n, n + (q + 1) n): panel writing panC slot q
  float* panA;                  // [2 planes][rows][kPanCols] (slot q = columns [128 q, 128 q + 128))
  float* panC;
  float* pinvS;
  int64_t plane_rows;
  int max_rows;                 // largest dp (stage grid)
};

namespace {

// SPDKFAC_UPDATE_PAIRS=1: 2 x 2 blocks of update tiles with one K range go to the CTA-pair engine
// (tc3_pair_ctile_kernel, 70 % tensor-pipe under ncu vs 47 % for the single-CTA engine).  Off by
// default: the aligned-pair cover takes ~57 % of the ResNet-50 update work and the leftover single
// tiles run less efficiently, so the batched inverse and the bench step are unchanged.
bool update_pairs() {
  const char* e = getenv("SPDKFAC_UPDATE_PAIRS");
  return e && e[0] == '1';
}

bool eager_rows_schedule() {  // SPDKFAC_EAGER_ROWS=1: the round-2 update schedule (A/B)
  const char* e = getenv("SPDKFAC_EAGER_ROWS");
  return e && e[0] == '1';
}

bool update_order_by_matrix() {  // SPDKFAC_UPDATE_ORDER=nk: the round-1 order (longest K first across matrices)
  const char* e = getenv("SPDKFAC_UPDATE_ORDER");
  return !(e && std::string(e) == "nk");
}

void inverse_sizes(int n, const int32_t* dims, int64_t* rows, int64_t* items, int64_t* act, int64_t* tiles,
                   int* steps, int* nblk) {
  *rows = *items = *act = *tiles = 0;
  *steps = *nblk = 0;
  for (int t = 0; t < n; ++t) {
    if (dims[t] <= kB) continue;
    const int64_t dp = round_up(dims[t], kB), T = dp / kB;
    *rows += dp;
    *steps = std::max<int>(*steps, int(T));
    *act += T;
    *items += T * (T - 1) + T * ((T - 1) * T / 2);  // panel items + update items over all steps
    *tiles += (dp / kT) * (dp / kT + 1) / 2;
    *nblk += 1;
  }
}

size_t inverse_carve(int n, const int32_t* dims, Carve& c, spdkfac_inverse_plan* p, std::vector<InvMat>* mats) {
  int64_t rows, items, act, tiles;
  int steps, nblk;
  inverse_sizes(n, dims, &rows, &items, &act, &tiles, &steps, &nblk);
  int64_t prow = 0;
  int slot = 0;
  for (int t = 0; t < n; ++t) {
    InvMat m{};
    m.d = dims[t];
    if (dims[t] <= kB) {
      m.dp = dims[t];
    } else {
      m.dp = int(round_up(dims[t], kB));
      m.W = c.take<float>(size_t(m.dp) * m.dp);
      m.panel_row0 = int(prow);
      m.slot = slot++;
      prow += m.dp;
    }
    if (mats) mats->push_back(m);
  }
  float* panA = c.take<float>(size_t(2) * std::max<int64_t>(rows, 1) * kPanCols);
  float* panC = c.take<float>(size_t(2) * std::max<int64_t>(rows, 1) * kPanCols);
  float* pinvS = c.take<float>(size_t(2) * std::max(nblk, 1) * kB * kB);
  float* scales = c.take<float>(size_t(4) * n);
  if (mats && c.ok())
    for (int t = 0; t < n; ++t) (*mats)[t].scale = scales + 4 * t;
  auto* dm = c.take<InvMat>(size_t(n));
  auto* sid = c.take<int32_t>(size_t(n));
  auto* bid = c.take<int32_t>(size_t(n));
  auto* aid = c.take<int32_t>(size_t(std::max<int64_t>(act, 1)));
  auto* tj = c.take<TileJob>(size_t(std::max<int64_t>(tiles, 1)));
  auto* pj = c.take<PanelJob>(size_t(std::max<int64_t>(items, 1)));
  auto* mp = c.take<CUtensorMap>(size_t(5 + nblk), 128);
  auto* mp16 = c.take<CUtensorMap>(size_t(5 + nblk), 128);
  auto* it = c.take<TcItem>(size_t(std::max<int64_t>(items, 1)));
  auto* it16 = c.take<TcItem>(size_t(std::max<int64_t>(items, 1)));
  auto* ep16 = c.take<TcEpi>(size_t(1 + kPanSlots) * n);
  auto* pit = c.take<TcPairCItem>(size_t(std::max<int64_t>(items / 4, 1)));
  auto* pit16 = c.take<TcPairCItem>(size_t(std::max<int64_t>(items / 4, 1)));
  auto* ep = c.take<TcEpi>(size_t(1 + kPanSlots) * n);
  if (p) {
    p->panA = panA, p->panC = panC, p->pinvS = pinvS, p->mats = dm, p->small_ids = sid, p->blocked_ids = bid;
    p->act_ids = aid, p->tiles = tj, p->pan_jobs = pj, p->maps = mp, p->items = it, p->epis = ep;
    p->maps16 = mp16, p->items16 = it16, p->epis16 = ep16;
    p->pitems = pit, p->pitems16 = pit16;
    p->plane_rows = rows, p->steps = steps, p->n_tiles = int(tiles);
  }
  return c.used;
}

}  // namespace

extern "C" {

size_t spdkfac_inverse_workspace_size(int n, const int32_t* dims) {
  if (n < 0 || (n > 0 && !dims)) return 0;
  Carve c(nullptr, 0);
  return inverse_carve(n, dims, c, nullptr, nullptr) + 256;
}

int spdkfac_inverse_plan_create(spdkfac_inverse_plan** out, int n, const int32_t* dims, const float* const* packed_in,
                                float* const* out_full, int32_t* info_dev, void* ws, size_t ws_bytes, void* stream) {
  SPD_ARG(out && n >= 1 && dims && packed_in && out_full && info_dev, SPDKFAC_ERR_ARG, "bad inverse plan arguments");
  for (int t = 0; t < n; ++t) SPD_ARG(dims[t] >= 1, SPDKFAC_ERR_ARG, "dimension must be >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* p = new spdkfac_inverse_plan();
  p->n = n;
  p->dims.assign(dims, dims + n);
  {
    const char* e = getenv("SPDKFAC_INV_TF32");
    p->f16 = !(e && e[0] == '1');
  }
  const int bk = 32;  // K elements per 128-byte tf32 operand row (the fp16 item copies hold half as many blocks)
  Carve c(ws, ws_bytes);
  std::vector<InvMat> mats;
  inverse_carve(n, dims, c, p, &mats);
  if (!c.ok() || !ws) {
    delete p;
    set_error("inverse workspace too small: need %zu bytes, got %zu", c.used, ws_bytes);
    return SPDKFAC_ERR_ARG;
  }
  std::vector<int32_t> small, blocked;
  p->max_rows = 0;
  for (int t = 0; t < n; ++t) {
    mats[t].in = packed_in[t];
    mats[t].out = out_full[t];
    mats[t].info = info_dev + t;
    const double d3 = double(dims[t]) * dims[t] * dims[t];
    p->algo_flops += d3;
    if (dims[t] <= kB) {
      small.push_back(t);
      p->small_flops += d3;
    } else {
      blocked.push_back(t);
      p->max_rows = std::max(p->max_rows, mats[t].dp);
    }
  }
  p->n_small = int(small.size());
  p->n_blocked = int(blocked.size());
  const int64_t plane = p->plane_rows * kPanCols;
  std::vector<TcEpi> epis(size_t(1 + kPanSlots) * n), epis16(epis.size());
  for (int t = 0; t < n; ++t) {
    const int cm = dims[t] > kB ? 5 + mats[t].slot : 0;
    epis[t] = TcEpi{mats[t].W, mats[t].dp, 0, -1.f, 1.f, kAxpby, 0, nullptr, 0, 0, cm, 0, nullptr};  // update
    epis16[t] = TcEpi{mats[t].W, mats[t].dp, 0, -1.f, 1.f, kAxpby, 0, nullptr, 0, 0, cm, 0, mats[t].scale};
    for (int q = 0; q < kPanSlots; ++q) {  // panel GEMM writing panC slot q
      epis[n + q * n + t] = TcEpi{mats[t].W, mats[t].dp, 0, 1.f, 0.f, kAxpby, 0, p->panC + q * kB, kPanCols, plane};
      epis16[n + q * n + t] = TcEpi{mats[t].W, mats[t].dp, 0, 1.f, 0.f, kAxpby, 1,
                                    reinterpret_cast<__half*>(p->panC) + q * kB, kPanCols, plane, 0, 0, mats[t].scale};
    }
  }
  std::vector<TileJob> tiles;
  for (int t : blocked) {
    const int T64 = mats[t].dp / kT;
    for (int I = 0; I < T64; ++I)
      for (int J = I; J < T64; ++J) tiles.push_back(TileJob{t, I, J, 0});
  }
  std::vector<int32_t> act;
  std::vector<TcItem> items;
  std::vector<TcPairCItem> pitems;
  std::vector<PanelJob> pan;
  for (int k = 0; k < p->steps; ++k) {
    p->act_off.push_back(int(act.size()));
    for (int t : blocked)
      if (k < mats[t].dp / kB) act.push_back(t);
    p->act_cnt.push_back(int(act.size()) - p->act_off.back());
    p->pan_off.push_back(int(items.size()));
    p->pj_off.push_back(int(pan.size()));
    for (int t : blocked) {  // panel GEMM: C_R = Wold[R,K] P^-1, stored into the upper block triangle
      const int T = mats[t].dp / kB;
      if (k >= T) continue;
      for (int R = 0; R < T; ++R) {
        if (R == k) continue;
        pan.push_back(PanelJob{t, R});
        const int prow = mats[t].panel_row0 + R * kB;
        const int q = k % kPanSlots;  // panel slot of step k
        TcItem it{};
        it.nk = kB / bk;
        it.epi = n + q * n + t;
        it.m_valid = kB;
        it.n_valid = kB;
        it.o2_row = prow;
        if (R < k) {  // D'[j][i] = (P^-1 Wold[R,K]^T)[j][i] = C_R[i][j] -> W[R0 + i][K0 + j], panC coalesced
          it.a_map = 2, it.a_row = mats[t].slot * kB, it.k0 = 0;
          it.b_map = 0, it.b_row = prow, it.b_koff = q * kB;
          it.out_r = k * kB, it.out_c = R * kB;
          it.flags = (kScInv << kScaleShiftA) | (kScReg << kScaleShiftB) | (kScInv << kScaleShiftO);
        } else {      // D[i][j] = C_R[i][j] -> W[K0 + j][R0 + i] (row panel), panC row-style
          it.a_map = 0, it.a_row = prow, it.k0 = q * kB;
          it.b_map = 2, it.b_row = mats[t].slot * kB, it.b_koff = -q * kB;
          it.out_r = R * kB, it.out_c = k * kB;
          it.flags = kOut2Rows | (kScSchur << kScaleShiftA) | (kScInv << kScaleShiftB) | (kScReg << kScaleShiftO);
        }
        items.push_back(it);
      }
    }
    p->pan_cnt.push_back(int(items.size()) - p->pan_off.back());
    p->upd_off.push_back(int(items.size()));
    // Update of step k, split into U1 (issued before step k+1's look-ahead front: it must
    // see these tiles) and U2 (runs under the front).  Steps are fused in groups of kFuse
    // (k0 = multiple of kFuse, last = min(k0 + kFuse - 1, T - 1)).  A non-last step s updates
    // only block row/column s+1 (U1: the next pivot block and panel read it), with all of that
    // tile's pending group steps in ONE contraction of K = (pending steps) x 128 (their panel
    // slots are adjacent); the last step also updates every other tile the same way (U2), so
    // W is read-modify-written about once per group instead of once per step.  A tile's pending
    // steps are those after the last group step that updated it (its row s+1) or had it in its
    // pivot row/column (the panel epilogue writes those).  SPDKFAC_EAGER_ROWS=1: the round-2
    // schedule (step s also updates rows s+2 .. last+1 eagerly, one step per contraction).
    int u1 = 0;
    std::vector<TcItem> u1v, u2v;
    const bool eager_rows = eager_rows_schedule();
    for (int t : blocked) {
      const int T = mats[t].dp / kB;
      if (k >= T) continue;
      const int k0 = k - k % kFuse, last = std::min(k0 + kFuse - 1, T - 1);
      const bool bulk = (k == last);
      auto touched = [&](int s, int I, int J) {  // group step s < k updated or owned tile (I, J)
        if (I == s || J == s) return true;  // pivot row/column: written by the panel epilogue
        if (!eager_rows) return I == s + 1 || J == s + 1;  // the next block row of step s
        return (I >= s + 1 && I <= last + 1) || (J >= s + 1 && J <= last + 1);  // eager rows of step s
      };
      for (int I = 0; I < T; ++I)
        for (int J = I; J < T; ++J) {
          if (I == k || J == k) continue;
          const bool row1 = (I == k + 1 || J == k + 1);
          const bool eager = eager_rows ? ((I >= k + 1 && I <= last + 1) || (J >= k + 1 && J <= last + 1)) : row1;
          int first = k;  // first pending step of this tile
          if (bulk || !eager_rows) {
            if (!bulk && !eager) continue;  // deferred to the group's last step
            first = k0;
            for (int s2 = k - 1; s2 >= k0; --s2)
              if (touched(s2, I, J)) {
                first = s2 + 1;
                break;
              }
          } else if (!eager) {
            continue;  // deferred to the group's last step
          }
          const bool in_u1 = row1;
          // D'[y][x] = sum_k Wold[J0+y][k] C[I0+x][k] = U[I0+x][J0+y] (U symmetric):
          // the coalesced transposed store lands on the upper block W[I, J]
          TcItem it{};
          it.a_map = 0;
          it.b_map = 1;
          it.a_row = mats[t].panel_row0 + J * kB;
          it.b_row = mats[t].panel_row0 + I * kB;
          it.k0 = (first % kPanSlots) * kB;
          it.nk = (k - first + 1) * (kB / bk);
          it.epi = t;
          // A = old panel rows J, B = new panel rows I; neither block is a pivot block of steps
          // first..k (those tiles were written by the panel epilogue), so both keep one class
          it.flags = ((J < first ? kScReg : kScSchur) << kScaleShiftA) | ((I < first ? kScInv : kScReg) << kScaleShiftB);
          it.out_r = J * kB;
          it.out_c = I * kB;
          it.m_valid = kB;
          it.n_valid = kB;
          (in_u1 ? u1v : u2v).push_back(it);
        }
    }
    // CTA-pair super tiles (2 x 2 target tiles sharing their K range) out of the U2 items; the
    // rest stay single-CTA items
    p->pu_off.push_back(int(pitems.size()));
    p->pu_flops.push_back(0.0);
    if (update_pairs()) {
      std::map<std::tuple<int, int, int>, size_t> at;  // (matrix, I, J) -> index in u2v
      for (size_t x = 0; x < u2v.size(); ++x)
        at[{u2v[x].epi, u2v[x].out_c / kB, u2v[x].out_r / kB}] = x;
      std::vector<bool> used(u2v.size(), false);
      for (int t : blocked) {
        const int T = mats[t].dp / kB;
        if (k >= T) continue;
        // greedy row-major cover of the upper block triangle by 2 x 2 super tiles (I0 .. I0+1) x
        // (J0 .. J0+1), J0 >= I0.  A diagonal super tile (J0 == I0) also computes the lower block
        // (I0+1, I0): the sweep maintains only the upper block triangle, which is all any kernel
        // reads, so that block's store is dead and harmless.
        for (int I0 = 0; I0 + 1 < T; ++I0)
          for (int J0 = I0; J0 + 1 < T; ++J0) {
            size_t ix[4];
            int n_up = 0;
            bool ok = true;
            for (int h = 0; h < 2 && ok; ++h)
              for (int r = 0; r < 2 && ok; ++r) {
                ix[2 * h + r] = SIZE_MAX;
                if (I0 + h > J0 + r) continue;  // the dead lower block of a diagonal super tile
                auto f = at.find({t, I0 + h, J0 + r});
                ok = f != at.end() && !used[f->second];
                if (ok) ix[2 * h + r] = f->second, ++n_up;
              }
            if (!ok || n_up < 3) continue;
            const TcItem& q0 = u2v[ix[0]];
            for (int e = 1; e < 4 && ok; ++e)
              if (ix[e] != SIZE_MAX) ok = u2v[ix[e]].k0 == q0.k0 && u2v[ix[e]].nk == q0.nk;
            if (!ok) continue;
            TcPairCItem pi{};
            pi.a_map = 0, pi.b_map = 1;
            pi.a_row = mats[t].panel_row0 + J0 * kB;
            pi.b_row = mats[t].panel_row0 + I0 * kB;
            pi.k0 = q0.k0, pi.nk = q0.nk, pi.epi = t;
            pi.out_r[0] = J0 * kB, pi.out_r[1] = (J0 + 1) * kB;
            pi.out_c[0] = I0 * kB, pi.out_c[1] = (I0 + 1) * kB;
            pi.flags = q0.flags & ((3 << kScaleShiftA) | (3 << kScaleShiftB));  // uniform over the super tile
            pitems.push_back(pi);
            p->pu_flops.back() += n_up * 2.0 * kB * kB * 32 * q0.nk;
            for (size_t e : ix)
              if (e != SIZE_MAX) used[e] = true;
          }
      }
      std::vector<TcItem> rest;
      for (size_t x = 0; x < u2v.size(); ++x)
        if (!used[x]) rest.push_back(u2v[x]);
      u2v.swap(rest);
      std::stable_sort(pitems.begin() + p->pu_off.back(), pitems.end(),
                       [&](const TcPairCItem& a, const TcPairCItem& b) {
                         const int da = mats[a.epi].dp, db = mats[b.epi].dp;
                         if (da != db) return da > db;
                         if (a.epi != b.epi) return a.epi < b.epi;
                         return a.nk > b.nk;
                       });
    }
    p->pu_cnt.push_back(int(pitems.size()) - p->pu_off.back());
    if (update_order_by_matrix()) {
      // matrix-major (largest first), longest K first inside a matrix: the persistent CTAs then work
      // on one matrix's panels at a time, a working set that stays in L2, instead of streaming every
      // batched matrix's panels at once
      std::stable_sort(u2v.begin(), u2v.end(), [&](const TcItem& a, const TcItem& b) {
        const int da = mats[a.epi].dp, db = mats[b.epi].dp;
        if (da != db) return da > db;
        if (a.epi != b.epi) return a.epi < b.epi;
        return a.nk > b.nk;
      });
    } else {
      std::stable_sort(u2v.begin(), u2v.end(), [](const TcItem& a, const TcItem& b) { return a.nk > b.nk; });
    }
    // the diagonal tiles (k+1, k+1) first: the look-ahead pivot only needs them
    std::stable_partition(u1v.begin(), u1v.end(), [&](const TcItem& it) {
      return it.out_r == (k + 1) * kB && it.out_c == (k + 1) * kB;
    });
    p->u1d_cnt.push_back(int(std::count_if(u1v.begin(), u1v.end(), [&](const TcItem& it) {
      return it.out_r == (k + 1) * kB && it.out_c == (k + 1) * kB;
    })));
    u1 = int(u1v.size());
    items.insert(items.end(), u1v.begin(), u1v.end());
    items.insert(items.end(), u2v.begin(), u2v.end());
    p->upd_flops.push_back(0.0);
    for (const TcItem& it : u1v) p->upd_flops.back() += 2.0 * kB * kB * bk * it.nk;
    p->u2_flops.push_back(0.0);
    for (const TcItem& it : u2v) p->u2_flops.back() += 2.0 * kB * kB * bk * it.nk;
    p->u1_cnt.push_back(u1);
    p->upd_cnt.push_back(int(items.size()) - p->upd_off.back());
  }
  std::vector<CUtensorMap> maps(size_t(5 + p->n_blocked)), maps16(maps.size());
  int rc = SPDKFAC_OK;
  if (p->n_blocked > 0) {
    if ((rc = make_operand_map_f16(&maps16[0], p->panA, kPanCols, p->plane_rows, kPanCols)) ||
        (rc = make_operand_map_f16(&maps16[1], p->panC, kPanCols, p->plane_rows, kPanCols)) ||
        (rc = make_operand_map_f16(&maps16[2], p->pinvS, kB, int64_t(p->n_blocked) * kB, kB)) ||
        (rc = make_operand_map(&maps[0], p->panA, false, kPanCols, p->plane_rows, kPanCols)) ||
        (rc = make_operand_map(&maps[1], p->panC, false, kPanCols, p->plane_rows, kPanCols)) ||
        (rc = make_operand_map(&maps[2], p->pinvS, false, kB, int64_t(p->n_blocked) * kB, kB))) {
      delete p;
      return rc;
    }
    maps[3] = maps[0], maps[4] = maps[1];
    maps16[3] = maps16[0], maps16[4] = maps16[1];
    for (int t : blocked)
      if ((rc = make_ctile_map(&maps[5 + mats[t].slot], mats[t].W, mats[t].dp, mats[t].dp, mats[t].dp))) {
        delete p;
        return rc;
      }
    for (int t : blocked) maps16[5 + mats[t].slot] = maps[5 + mats[t].slot];
  }
  std::vector<TcItem> items16(items);
  for (TcItem& it : items16) it.nk /= 2;  // K blocks of 64 fp16 elements (tf32: 32)
  std::vector<TcPairCItem> pitems16(pitems);
  for (TcPairCItem& it : pitems16) it.nk /= 2;
  if ((rc = upload(p->mats, mats, s)) || (rc = upload(p->small_ids, small, s)) ||
      (rc = upload(p->blocked_ids, blocked, s)) || (rc = upload(p->act_ids, act, s)) ||
      (rc = upload(p->tiles, tiles, s)) || (rc = upload(p->pan_jobs, pan, s)) || (p->n_blocked > 0 && (rc = upload(p->maps, maps, s))) ||
      (p->n_blocked > 0 && (rc = upload(p->maps16, maps16, s))) || (rc = upload(p->items16, items16, s)) ||
      (rc = upload(p->epis16, epis16, s)) ||
      (rc = upload(p->items, items, s)) || (rc = upload(p->pitems, pitems, s)) ||
      (rc = upload(p->pitems16, pitems16, s)) || (rc = upload(p->epis, epis, s))) {
    delete p;
    return rc;
  }
  {
    if (const char* pc = getenv("SPDKFAC_PANEL_CTAS")) p->panel_ctas = atoi(pc);
    const char* e = getenv("SPDKFAC_NO_LOOKAHEAD");
    p->lookahead = !(e && e[0] == '1');
    const char* df = getenv("SPDKFAC_DIAG_FIRST");
    p->diag_first = !(df && df[0] == '0');
    // the fp32 FFMA pivot sweep is the default: the tcgen05 pivot kernel (SPDKFAC_PIVOT=tc) is 1.6x
    // faster per block but its 32-wide blocked sweep loses accuracy on rank-deficient factors
    // (ResNet-50 fc A, kappa 2e4: inverse error 2.6e-2 vs 5e-3), see DESIGN.md
    const char* pv = getenv("SPDKFAC_PIVOT");
    p->legacy_pivot = !(pv && std::string(pv) == "tc");
    p->pivot_v3 = !(pv && std::string(pv) == "b8");
  }
  if (p->n_blocked > 0) {
    {
      const char* pe = getenv("SPDKFAC_INV_PRIORITY");
      SPD_CUDA(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, pe ? atoi(pe) : 0));
    }
    SPD_CUDA(cudaEventCreateWithFlags(&p->ev_u1, cudaEventDisableTiming));
    SPD_CUDA(cudaEventCreateWithFlags(&p->ev_diag, cudaEventDisableTiming));
    SPD_CUDA(cudaEventCreateWithFlags(&p->ev_panel, cudaEventDisableTiming));
  }
  static bool attrs = false;
  if (!attrs) {
    SPD_CUDA(cudaFuncSetAttribute(small_inverse_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kB * kSmemLd * 4));
    SPD_CUDA(cudaFuncSetAttribute(small_inverse_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kB * kSmemLd * 4));
    SPD_CUDA(cudaFuncSetAttribute(pivot_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pvt::kSmem)));
    SPD_CUDA(cudaFuncSetAttribute(pivot_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pvt::kSmem)));
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
    Probe* pr = stat_begin(kCatInvSmall, s);
    if (p->legacy_pivot && p->pivot_v3)
      small_inverse_kernel<true><<<p->n_small, 512, kB * kSmemLd * 4, s>>>(p->mats, p->small_ids, gamma, pr);
    else if (p->legacy_pivot)
      small_inverse_kernel<false><<<p->n_small, 512, kB * kSmemLd * 4, s>>>(p->mats, p->small_ids, gamma, pr);
    else
      pivot_tc_kernel<true><<<p->n_small, pvt::kThreads, pvt::kSmem, s>>>(p->mats, p->small_ids, 0, nullptr, 0, 0,
                                                                          gamma, pr);
    SPD_CHECK_LAUNCH();
    stat_end(kCatInvSmall, s, p->small_flops, 0);
  }
  if (p->n_blocked > 0) {
    const int64_t plane = p->plane_rows * kPanCols;
    // fp16 operand planes when the damping bounds the inverse (gamma >= kF16MinGamma)
    const bool f16 = p->f16 && gamma >= kF16MinGamma;
    const CUtensorMap* maps = f16 ? p->maps16 : p->maps;
    const TcItem* items = f16 ? p->items16 : p->items;
    const TcEpi* epis = f16 ? p->epis16 : p->epis;
    stat_begin(kCatInvUnpackFinal, s);
    damp_unpack_kernel<<<p->n_tiles, 256, 0, s>>>(p->mats, p->tiles, gamma, f16 ? gamma : 1.f);
    SPD_CHECK_LAUNCH();
    if (f16) {
      inv_scale_kernel<<<p->n_blocked, 256, 0, s>>>(p->mats, p->blocked_ids, gamma);
      SPD_CHECK_LAUNCH();
    }
    stat_end(kCatInvUnpackFinal, s, 0, 0);
    // step k's pivot -> stage -> panel GEMM on stream q (the critical chain)
    auto front_pivot = [&](int k, cudaStream_t q) -> int {
      const int na = p->act_cnt[k];
      Probe* pr = stat_begin(kCatInvPivot, q);
      if (p->legacy_pivot && p->pivot_v3)
        pivot_kernel<true><<<na, 512, 0, q>>>(p->mats, p->act_ids + p->act_off[k], k, p->pinvS,
                                              int64_t(p->n_blocked) * kB * kB, int(f16), pr);
      else if (p->legacy_pivot)
        pivot_kernel<false><<<na, 512, 0, q>>>(p->mats, p->act_ids + p->act_off[k], k, p->pinvS,
                                               int64_t(p->n_blocked) * kB * kB, int(f16), pr);
      else
        pivot_tc_kernel<false><<<na, pvt::kThreads, pvt::kSmem, q>>>(p->mats, p->act_ids + p->act_off[k], k, p->pinvS,
                                                                     int64_t(p->n_blocked) * kB * kB, int(f16), 0.f, pr);
      SPD_CHECK_LAUNCH();
      stat_end(kCatInvPivot, q, 2.0 * kB * kB * kB * na, 0);
      return SPDKFAC_OK;
    };
    auto front_panel = [&](int k, cudaStream_t q) -> int {
      void* pa = f16 ? static_cast<void*>(reinterpret_cast<__half*>(p->panA) + (k % kPanSlots) * kB)
                     : static_cast<void*>(p->panA + (k % kPanSlots) * kB);
      TcRun prun{};
      prun.probe = stat_begin(kCatInvPanel, q);  // the probe times the panel GEMM launch
      if (f16)
        stage_panel_kernel<true><<<dim3(p->pan_cnt[k], 4), 256, 0, q>>>(p->mats, p->pan_jobs + p->pj_off[k], k, pa,
                                                                         plane);
      else
        stage_panel_kernel<false><<<dim3(p->pan_cnt[k], 4), 256, 0, q>>>(p->mats, p->pan_jobs + p->pj_off[k], k, pa,
                                                                          plane);
      SPD_CHECK_LAUNCH();
      // the panel GEMM has few K blocks per tile: a full persistent grid would hold every SM for
      // ~20 us per step while doing little work; a capped grid leaves the SMs to the
      // concurrent convolutions at almost the same chain latency
      int rc = launch_tc3(f16 ? Kind::F16 : Kind::TF32, maps, items + p->pan_off[k], epis, p->pan_cnt[k], q, prun,
                          p->panel_ctas);
      if (rc) return rc;
      stat_end(kCatInvPanel, q, 2.0 * kB * kB * kB * p->pan_cnt[k], 0);
      return SPDKFAC_OK;
    };
    auto front = [&](int k, cudaStream_t q) -> int {
      const int rc = front_pivot(k, q);
      return rc ? rc : front_panel(k, q);
    };
    const Kind ukind = f16 ? Kind::F16 : Kind::TF32;
    int rc = front(0, s);
    if (rc) return rc;
    for (int k = 0; k < p->steps; ++k) {
      // U1(k): the tiles step k+1 reads; then step k+1's front runs on the side stream
      // while U2(k) (the rest of the trailing update) runs here (look-ahead)
      const int u1 = p->u1_cnt[k], u2 = p->upd_cnt[k] - u1;
      const bool ahead = k + 1 < p->steps;
      // U1's diagonal tiles first, so step k+1's pivot (which reads only them) runs beside the rest of U1
      const bool split = ahead && p->lookahead && p->diag_first && p->u1d_cnt[k] > 0 && p->u1d_cnt[k] < u1;
      const int u1a = split ? p->u1d_cnt[k] : u1;
      Probe* pu = nullptr;
      if (u1a > 0) {
        pu = stat_begin(kCatInvUpdate, s);
        rc = launch_tc3_ctile(maps, items + p->upd_off[k], epis, u1a, s, pu, ukind);
        if (rc) return rc;
        stat_end(kCatInvUpdate, s, split ? 0.0 : p->upd_flops[k], 0);
      }
      if (split) {
        SPD_CUDA(cudaEventRecord(p->ev_diag, s));
        SPD_CUDA(cudaStreamWaitEvent(p->side, p->ev_diag, 0));
        if ((rc = front_pivot(k + 1, p->side))) return rc;
        pu = stat_begin(kCatInvUpdate, s);
        rc = launch_tc3_ctile(maps, items + p->upd_off[k] + u1a, epis, u1 - u1a, s, pu, ukind);
        if (rc) return rc;
        stat_end(kCatInvUpdate, s, p->upd_flops[k], 0);
      }
      if (ahead && !p->lookahead) {  // serial order: rest of the update, then the next front
        if (p->pu_cnt[k]) {
          Probe* pp = stat_begin(kCatInvUpdate, s);
          if ((rc = launch_tc3_pair_ctile(maps, (f16 ? p->pitems16 : p->pitems) + p->pu_off[k], epis, p->pu_cnt[k], s, pp,
                                          ukind)))
            return rc;
          stat_end(kCatInvUpdate, s, p->pu_flops[k], 0);
        }
        if (u2 > 0) {  // (non-last steps of a fused group have no U2)
          Probe* pu2 = stat_begin(kCatInvUpdate, s);
          rc = launch_tc3_ctile(maps, items + p->upd_off[k] + u1, epis, u2, s, pu2, ukind);
          if (rc) return rc;
          stat_end(kCatInvUpdate, s, p->u2_flops[k], 0);
        }
        if ((rc = front(k + 1, s))) return rc;
        continue;
      }
      if (ahead) {
        SPD_CUDA(cudaEventRecord(p->ev_u1, s));
        SPD_CUDA(cudaStreamWaitEvent(p->side, p->ev_u1, 0));
        if ((rc = split ? front_panel(k + 1, p->side) : front(k + 1, p->side))) return rc;
        SPD_CUDA(cudaEventRecord(p->ev_panel, p->side));
      }
      if (p->pu_cnt[k]) {
        Probe* pp = stat_begin(kCatInvUpdate, s);
        if ((rc = launch_tc3_pair_ctile(maps, (f16 ? p->pitems16 : p->pitems) + p->pu_off[k], epis, p->pu_cnt[k], s, pp,
                                          ukind)))
            return rc;
        stat_end(kCatInvUpdate, s, p->pu_flops[k], 0);
      }
      if (u2 > 0) {
        pu = stat_begin(kCatInvUpdate, s);
        rc = launch_tc3_ctile(maps, items + p->upd_off[k] + u1, epis, u2, s, pu, ukind);
        if (rc) return rc;
        stat_end(kCatInvUpdate, s, p->u2_flops[k], 0);
      }
      if (ahead) SPD_CUDA(cudaStreamWaitEvent(s, p->ev_panel, 0));
    }
    stat_begin(kCatInvUnpackFinal, s);
    finalize_kernel<<<p->n_tiles, 256, 0, s>>>(p->mats, p->tiles);
    SPD_CHECK_LAUNCH();
    stat_end(kCatInvUnpackFinal, s, 0, 0);
  }
  return SPDKFAC_OK;
}

void spdkfac_inverse_plan_destroy(spdkfac_inverse_plan* p) {
  if (!p) return;
  if (p->ev_u1) cudaEventDestroy(p->ev_u1);
  if (p->ev_diag) cudaEventDestroy(p->ev_diag);
  if (p->ev_panel) cudaEventDestroy(p->ev_panel);
  if (p->side) cudaStreamDestroy(p->side);
  delete p;
}

}  // extern "C"
