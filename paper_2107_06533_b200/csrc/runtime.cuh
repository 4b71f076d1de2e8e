// Host-side runtime helpers: error state, tensor-map encoding, workspace carving,
// table upload, tcgen05 GEMM launch.
#pragma once
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "tc_gemm.cuh"
#include "../../include/spdkfac.h"

namespace spd {

void set_error(const char* fmt, ...);

#define SPD_CUDA(call)                                                                \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      ::spd::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return SPDKFAC_ERR_CUDA;                                                        \
    }                                                                                 \
  } while (0)

#define SPD_CHECK_LAUNCH()                                                            \
  do {                                                                                \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess) {                                                          \
      ::spd::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return SPDKFAC_ERR_CUDA;                                                        \
    }                                                                                 \
  } while (0)

#define SPD_ARG(cond, code, ...)            \
  do {                                      \
    if (!(cond)) {                          \
      ::spd::set_error(__VA_ARGS__);        \
      return code;                          \
    }                                       \
  } while (0)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t cdiv(int64_t x, int64_t m) { return (x + m - 1) / m; }

// Bump allocator over a caller-provided device workspace (256-B aligned slices).
struct Carve {
  uint8_t* base;
  size_t cap, used = 0;
  Carve(void* b, size_t c) : base(static_cast<uint8_t*>(b)), cap(c) {}
  template <class T>
  T* take(size_t count, size_t align = 256) {
    used = (used + align - 1) / align * align;
    T* p = reinterpret_cast<T*>(base ? base + used : nullptr);
    used += count * sizeof(T);
    return p;
  }
  bool ok() const { return used <= cap; }
};

// 3-D tensor map over a split-precision operand: planes [2][rows][ld] with K (= ld
// axis, extent k_extent) innermost; box = {128 B of K, 128 rows, 1 plane}, SWIZZLE_128B.
int make_operand_map(CUtensorMap* out, const void* base, bool bf16, int64_t k_extent, int64_t rows, int64_t ld);
// MN-major bf16 split planes [2][k_rows][ld] (box 64 x 64, SWIZZLE_128B; items flagged kMnMajor)
int make_operand_map_mn(CUtensorMap* out, const void* base, int64_t ld, int64_t k_rows);
// im2col-mode map of one staged bf16 NHWC activation plane: boxes of 64 output positions x 64 channels
int make_im2col_map_bf16(CUtensorMap* out, const void* base, int n, int h, int w, int c, int kh, int kw, int stride_h,
                         int stride_w, int pad_h, int pad_w, int dil_h, int dil_w);
// fp16 split planes [2][rows][ld], K-major, box 64 (K) x 128 rows, SWIZZLE_128B
int make_operand_map_f16(CUtensorMap* out, const void* base, int64_t k_extent, int64_t rows, int64_t ld);

// 2-D map over fp32 rows [rows][cols] (row stride ld), box 128 columns x kF32Bk rows, no swizzle
int make_rows_map_f32(CUtensorMap* out, const float* base, int64_t rows, int64_t cols, int64_t ld);

// Upload `n` POD objects into device memory `dst` on `stream` (pageable source: the
// copy consumes the host buffer before returning).
template <class T>
int upload(T* dst, const std::vector<T>& v, cudaStream_t s) {
  if (v.empty()) return SPDKFAC_OK;
  SPD_CUDA(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return SPDKFAC_OK;
}

// Pointer table passed by value (kernel parameter space).
constexpr int kMaxPtrs = 128;
constexpr int kMaxPeers = 8;  // ranks of one NVSwitch node (peer-memory factor aggregation)
struct PtrTable {
  const void* p[kMaxPtrs];
};

int launch_tc3(Kind kind, const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n_items,
               cudaStream_t s, const TcRun& run = TcRun{}, int max_ctas = 0);
// BF16 SYRK engine whose kF32Rows items read fp32 rows through the tensor maps in `fm` (converter warps)
int launch_tc3_f32(const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n_items, cudaStream_t s,
                   const TcRun& run, const F32Maps& fm);
// CTA-pair SYRK engine (cta_group::2, 256 x 256 super tiles; bf16 MN-major split planes)
int launch_tc3_pair(const CUtensorMap* maps, const TcPairItem* items, const TcEpi* epis, int n_items, cudaStream_t s,
                    const TcRun& run);
// TF32 / F16 engine with a TMA-staged fp32 C tile (read-modify-write targets, TcEpi::c_map)
int launch_tc3_ctile(const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n_items, cudaStream_t s,
                     Probe* probe = nullptr, Kind kind = Kind::TF32);
// CTA-pair TF32 engine with the C-slice ring (256 x 256 super tiles of the inverse trailing update)
int launch_tc3_pair_ctile(const CUtensorMap* maps, const TcPairCItem* items, const TcEpi* epis, int n_items,
                          cudaStream_t s, Probe* probe = nullptr, Kind kind = Kind::TF32);
// TF32 engine with chunked accumulation (kAccChunk K blocks of 32 per TMEM chunk, chunks summed in
// fp32 registers): the preconditioning GEMMs (see tc3_gemm_kernel's kAcc)
constexpr int kAccChunk = 2;  // 64 K elements = 24 accumulating MMAs per TMEM chunk
int launch_tc3_acc(const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n_items, cudaStream_t s,
                   const TcRun& run = TcRun{}, Kind kind = Kind::TF32, int max_ctas = 0);
// 2-D tensor map over a row-major fp32 matrix [rows][ld], box 128 x 128, no swizzle
int make_ctile_map(CUtensorMap* out, const float* base, int64_t rows, int64_t cols, int64_t ld);

// Launch accounting (include/spdkfac.h spdkfac_stats_*): every kernel launch of the
// library is counted; with timing enabled each launch is bracketed by CUDA events on
// its own stream and attributed to a category with its algorithmic flop count.
enum StatCat : int {
  kCatFactorStage = 0, kCatFactorSyrk, kCatFactorReduce, kCatInvSmall, kCatInvPivot, kCatInvPanel, kCatInvUpdate,
  kCatInvUnpackFinal, kCatPrecSplit, kCatPrecGemm, kCatPrecApply, kCatPack, kNumCats
};
// stat_begin returns the launch's probe when `cat` is probe-timed (spdkfac_stats_set_probes): the
// launch site passes it to its kernel (TcRun::probe or a kernel argument); else nullptr
Probe* stat_begin(int cat, cudaStream_t s);
void stat_end(int cat, cudaStream_t s, double flops, double bytes);

}  // namespace spd
