// Runtime: error reporting, driver entry point for tensor-map encoding, GEMM launch,
// packed <-> full symmetric layout kernels.
#include <atomic>
#include <cstdarg>
#include <mutex>

#include <string>

#include "runtime.cuh"

namespace spd {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ------------------------------------------------------------------ launch accounting
namespace {
struct StatRec {
  cudaEvent_t a = nullptr, b = nullptr;
  int cat = 0;
  double flops = 0, bytes = 0;
};
std::mutex g_stat_mu;
std::vector<StatRec> g_recs;
size_t g_rec_used = 0;
uint32_t g_timing = 0;  // bitmask of event-timed categories
uint32_t g_probing = 0;  // bitmask of probe-timed categories (in-kernel stamps)
Probe* g_probes = nullptr;  // device array of probe slots
size_t g_probe_cap = 0, g_probe_used = 0;
std::vector<int> g_probe_cat;  // category of each used slot
std::atomic<uint64_t> g_launches{0};
uint64_t g_cat_launches[kNumCats] = {};
double g_cat_flops[kNumCats] = {}, g_cat_bytes[kNumCats] = {};
thread_local long g_open = -1;

// inside stream capture, record as an external event node so the timestamps of every
// graph replay are readable (and timeable) from the host
void record_stat_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &st);
  if (st == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else cudaEventRecord(e, s);
}
}  // namespace

Probe* stat_begin(int cat, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_probing & (1u << cat)) {
    std::lock_guard<std::mutex> lk(g_stat_mu);
    if (g_probe_used >= g_probe_cap) return nullptr;  // out of reserved slots: untimed
    g_probe_cat.push_back(cat);
    return g_probes + g_probe_used++;
  }
  if (!(g_timing & (1u << cat))) return nullptr;
  std::lock_guard<std::mutex> lk(g_stat_mu);
  if (g_rec_used == g_recs.size()) {
    StatRec r;
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    g_recs.push_back(r);
  }
  g_open = long(g_rec_used++);
  g_recs[g_open].cat = cat;
  record_stat_event(g_recs[g_open].a, s);
  return nullptr;
}

void stat_end(int cat, cudaStream_t s, double flops, double bytes) {
  std::lock_guard<std::mutex> lk(g_stat_mu);
  g_cat_launches[cat] += 1;
  g_cat_flops[cat] += flops;
  g_cat_bytes[cat] += bytes;
  if ((g_timing & (1u << cat)) && g_open >= 0) {
    g_recs[g_open].flops = flops;
    g_recs[g_open].bytes = bytes;
    record_stat_event(g_recs[g_open].b, s);
    g_open = -1;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

static EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
}

int make_im2col_map_bf16(CUtensorMap* out, const void* base, int n, int h, int w, int c, int kh, int kw, int stride_h,
                         int stride_w, int pad_h, int pad_w, int dil_h, int dil_w) {
  EncodeIm2colFn fn = encode_im2col_fn();
  SPD_ARG(fn != nullptr, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  SPD_ARG(c % 64 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0, SPDKFAC_ERR_ARG, "im2col map: misaligned");
  cuuint64_t dims[4] = {cuuint64_t(c), cuuint64_t(w), cuuint64_t(h), cuuint64_t(n)};
  cuuint64_t strides[3] = {cuuint64_t(c) * 2, cuuint64_t(w) * c * 2, cuuint64_t(h) * w * c * 2};
  // bounding box of the receptive fields' top-left corners: from (-pad) to (last index + pad -
  // (k - 1) dil).  Innermost spatial dimension first ({W, H}, like the coordinates; measured: the
  // {H, W} order of the driver documentation traps on non-square kernels)
  int lower[2] = {-pad_w, -pad_h};
  int upper[2] = {pad_w - (kw - 1) * dil_w, pad_h - (kh - 1) * dil_h};
  cuuint32_t estr[4] = {1, cuuint32_t(stride_w), cuuint32_t(stride_h), 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, lower, upper, 64,
                  64, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPD_ARG(r == CUDA_SUCCESS, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeIm2col failed (%d)", int(r));
  return SPDKFAC_OK;
}

int make_operand_map(CUtensorMap* out, const void* base, bool bf16, int64_t k_extent, int64_t rows, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  SPD_ARG(fn != nullptr, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int64_t es = bf16 ? 2 : 4;
  SPD_ARG((ld * es) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0, SPDKFAC_ERR_ARG,
          "tensor map: misaligned operand");
  cuuint64_t dims[3] = {cuuint64_t(k_extent), cuuint64_t(rows), 2};
  cuuint64_t strides[2] = {cuuint64_t(ld * es), cuuint64_t(ld * es * rows)};
  cuuint32_t box[3] = {cuuint32_t(128 / es), 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPD_ARG(r == CUDA_SUCCESS, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return SPDKFAC_OK;
}

int make_operand_map_f16(CUtensorMap* out, const void* base, int64_t k_extent, int64_t rows, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  SPD_ARG(fn != nullptr, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  SPD_ARG((ld * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0, SPDKFAC_ERR_ARG,
          "tensor map: misaligned operand");
  cuuint64_t dims[3] = {cuuint64_t(k_extent), cuuint64_t(rows), 2};
  cuuint64_t strides[2] = {cuuint64_t(ld * 2), cuuint64_t(ld * 2 * rows)};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPD_ARG(r == CUDA_SUCCESS, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled (fp16) failed (%d)", int(r));
  return SPDKFAC_OK;
}

int make_operand_map_mn(CUtensorMap* out, const void* base, int64_t ld, int64_t k_rows) {
  EncodeTiledFn fn = encode_fn();
  SPD_ARG(fn != nullptr, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  SPD_ARG((ld * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0, SPDKFAC_ERR_ARG,
          "tensor map: misaligned operand");
  cuuint64_t dims[3] = {cuuint64_t(ld), cuuint64_t(k_rows), 2};
  cuuint64_t strides[2] = {cuuint64_t(ld * 2), cuuint64_t(ld * 2 * k_rows)};
  cuuint32_t box[3] = {64, 64, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPD_ARG(r == CUDA_SUCCESS, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return SPDKFAC_OK;
}

int make_rows_map_f32(CUtensorMap* out, const float* base, int64_t rows, int64_t cols, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  SPD_ARG(fn != nullptr, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  SPD_ARG((ld * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0, SPDKFAC_ERR_ARG,
          "tensor map: misaligned fp32 rows");
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * 4)};
  cuuint32_t box[2] = {128, kF32Bk};  // 128 MN columns x 32 K rows, unswizzled (the converters read it)
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPD_ARG(r == CUDA_SUCCESS, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled (fp32 rows) failed (%d)", int(r));
  return SPDKFAC_OK;
}

// Grid policy of the tile engines: persistent (<= one CTA per SM, static round robin over the
// work items) or one CTA per work item (SPDKFAC_GRID=tiles): CTAs then retire tile by tile,
// so kernels of concurrent streams (the forward/backward convolutions) get SMs as soon as a
// tile finishes instead of after the whole launch.
static bool tile_grid() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("SPDKFAC_GRID");
    mode = (e && std::string(e) == "tiles") ? 1 : 0;
  }
  return mode == 1;
}

template <Kind K, int kSt, bool kCTile, int kAcc = 0, bool kF32 = false>
static int launch_kind(const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n, cudaStream_t s,
                       const TcRun& run, int max_ctas = 0, const F32Param<kF32>* fm = nullptr) {
  constexpr size_t smem = tc_smem_bytes<kSt>(kCTile);
  static bool attr_set = false;
  if (!attr_set) {
    SPD_CUDA(cudaFuncSetAttribute(tc3_gemm_kernel<K, kSt, kCTile, kAcc, kF32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    attr_set = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    SPD_CUDA(cudaGetDevice(&dev));
    SPD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // optional cap on the persistent grid (leaves SMs to concurrent streams); diagnostics
    if (const char* e = getenv("SPDKFAC_MAX_CTAS")) {
      const int cap = atoi(e);
      if (cap > 0 && cap < sms) sms = cap;
    }
  }
  int cap = sms;
  if (max_ctas > 0 && max_ctas < cap) cap = max_ctas;
  const int grid = (tile_grid() || n < cap) ? n : cap;
  if constexpr (kF32)
    tc3_gemm_kernel<K, kSt, kCTile, kAcc, true><<<grid, 320, smem, s>>>(maps, items, epis, run, n, *fm);
  else
    tc3_gemm_kernel<K, kSt, kCTile, kAcc, false><<<grid, 192, smem, s>>>(maps, items, epis, run, n, NoF32Maps{});
  SPD_CHECK_LAUNCH();
  return SPDKFAC_OK;
}

int launch_tc3(Kind kind, const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n, cudaStream_t s,
               const TcRun& run, int max_ctas) {
  if (n <= 0) return SPDKFAC_OK;
  if (kind == Kind::BF16) return launch_kind<Kind::BF16, kStages, false>(maps, items, epis, n, s, run, max_ctas);
  if (kind == Kind::F16) return launch_kind<Kind::F16, kStages, false>(maps, items, epis, n, s, run, max_ctas);
  return launch_kind<Kind::TF32, kStages, false>(maps, items, epis, n, s, run, max_ctas);
}

int launch_tc3_f32(const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n, cudaStream_t s,
                   const TcRun& run, const F32Maps& fm) {
  if (n <= 0) return SPDKFAC_OK;
  return launch_kind<Kind::BF16, kStages, false, 0, true>(maps, items, epis, n, s, run, 0, &fm);
}

int launch_tc3_acc(const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n, cudaStream_t s,
                   const TcRun& run, Kind kind, int max_ctas) {
  if (n <= 0) return SPDKFAC_OK;
  // fp16: chunks of one 64-element K block, the same partial-sum length as tf32's two blocks of 32 (the
  // TMEM accumulation truncates ~2^-24 of the running sum per MMA: longer chunks measured 1.6e-4 vs 9e-5
  // on Inception-v4's rank-4 fc update)
  if (kind == Kind::F16) return launch_kind<Kind::F16, kStages, false, 1>(maps, items, epis, n, s, run, max_ctas);
  return launch_kind<Kind::TF32, kStages, false, kAccChunk>(maps, items, epis, n, s, run, max_ctas);
}

int launch_tc3_ctile(const CUtensorMap* maps, const TcItem* items, const TcEpi* epis, int n, cudaStream_t s,
                     Probe* probe, Kind kind) {
  if (n <= 0) return SPDKFAC_OK;
  TcRun run{};
  run.probe = probe;
  if (kind == Kind::F16) return launch_kind<Kind::F16, 3, true>(maps, items, epis, n, s, run);
  return launch_kind<Kind::TF32, 3, true>(maps, items, epis, n, s, run);
}

int launch_tc3_pair(const CUtensorMap* maps, const TcPairItem* items, const TcEpi* epis, int n, cudaStream_t s,
                    const TcRun& run) {
  if (n <= 0) return SPDKFAC_OK;
  static bool attr_set = false;
  if (!attr_set) {
    SPD_CUDA(cudaFuncSetAttribute(tc3_pair_kernel<kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPairSmemBytes)));
    attr_set = true;
  }
  static int pairs = 0;
  if (!pairs) {
    int dev = 0, sms = 0;
    SPD_CUDA(cudaGetDevice(&dev));
    SPD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (const char* e = getenv("SPDKFAC_MAX_CTAS")) {
      const int cap = atoi(e);
      if (cap > 0 && cap < sms) sms = cap;
    }
    pairs = sms / 2;
  }
  const int grid = 2 * ((tile_grid() || n < pairs) ? n : pairs);
  tc3_pair_kernel<kStages><<<grid, 192, kPairSmemBytes, s>>>(maps, items, epis, run, n);
  SPD_CHECK_LAUNCH();
  return SPDKFAC_OK;
}

int launch_tc3_pair_ctile(const CUtensorMap* maps, const TcPairCItem* items, const TcEpi* epis, int n, cudaStream_t s,
                          Probe* probe, Kind kind) {
  if (n <= 0) return SPDKFAC_OK;
  static bool attr_set = false;
  if (!attr_set) {
    SPD_CUDA(cudaFuncSetAttribute(tc3_pair_ctile_kernel<kStages, Kind::TF32>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPairCSmemBytes)));
    SPD_CUDA(cudaFuncSetAttribute(tc3_pair_ctile_kernel<kStages, Kind::F16>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPairCSmemBytes)));
    attr_set = true;
  }
  static int pairs = 0;
  if (!pairs) {
    int dev = 0, sms = 0;
    SPD_CUDA(cudaGetDevice(&dev));
    SPD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (const char* e = getenv("SPDKFAC_MAX_CTAS")) {
      const int cap = atoi(e);
      if (cap > 0 && cap < sms) sms = cap;
    }
    pairs = sms / 2;
  }
  TcRun run{};
  run.probe = probe;
  const int grid = 2 * (n < pairs ? n : pairs);
  if (kind == Kind::F16)
    tc3_pair_ctile_kernel<kStages, Kind::F16><<<grid, 192, kPairCSmemBytes, s>>>(maps, items, epis, run, n);
  else
    tc3_pair_ctile_kernel<kStages, Kind::TF32><<<grid, 192, kPairCSmemBytes, s>>>(maps, items, epis, run, n);
  SPD_CHECK_LAUNCH();
  return SPDKFAC_OK;
}

int make_ctile_map(CUtensorMap* out, const float* base, int64_t rows, int64_t cols, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  SPD_ARG(fn != nullptr, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  SPD_ARG((ld * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0, SPDKFAC_ERR_ARG,
          "tensor map: misaligned target");
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * 4)};
  cuuint32_t box[2] = {128, kCSliceRows};  // 32-row slices (kCTile ring)
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SPD_ARG(r == CUDA_SUCCESS, SPDKFAC_ERR_CUDA, "cuTensorMapEncodeTiled (C tile) failed (%d)", int(r));
  return SPDKFAC_OK;
}

// ------------------------------------------------------------------ pack / unpack
// packed element (i <= j) at i*(2d-i+1)/2 + (j-i)  (row-major upper incl. diagonal)
__global__ void pack_kernel(const float* __restrict__ full, int64_t d, int64_t ld, float* __restrict__ packed) {
  const int64_t i = blockIdx.y;
  const int64_t base = i * (2 * d - i + 1) / 2 - i;
  for (int64_t j = i + blockIdx.x * blockDim.x + threadIdx.x; j < d; j += int64_t(gridDim.x) * blockDim.x)
    packed[base + j] = full[i * ld + j];
}

__global__ void unpack_kernel(const float* __restrict__ packed, int64_t d, float* __restrict__ full, int64_t ld) {
  // row i of the full matrix: j >= i from packed row i, j < i from packed row j (column i)
  const int64_t i = blockIdx.y;
  for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < d; j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = j < i ? j : i, c = j < i ? i : j;
    full[i * ld + j] = packed[r * (2 * d - r + 1) / 2 + (c - r)];
  }
}

struct PackArgs {
  const float* src[kMaxPtrs];
  float* dst[kMaxPtrs];
  int32_t d[kMaxPtrs];
  int32_t row0[kMaxPtrs + 1];  // prefix sum of rows (grid.y mapping)
  int n;
};

__global__ void pack_batched_kernel(const __grid_constant__ PackArgs a, int unpack) {
  const int row = blockIdx.x;  // x: a batch's rows can exceed gridDim.y's 65535
  int t = 0;
  while (t + 1 < a.n && a.row0[t + 1] <= row) ++t;
  const int64_t d = a.d[t], i = row - a.row0[t];
  if (i >= d) return;
  if (!unpack) {
    const int64_t base = i * (2 * d - i + 1) / 2 - i;
    for (int64_t j = i + threadIdx.x; j < d; j += blockDim.x) a.dst[t][base + j] = a.src[t][i * d + j];
  } else {
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
      const int64_t r = j < i ? j : i, c = j < i ? i : j;
      a.dst[t][i * d + j] = a.src[t][r * (2 * d - r + 1) / 2 + (c - r)];
    }
  }
}

// packed upper -> full symmetric, one 64 x 64 upper tile (I <= J) per block: rows of the
// upper tile are contiguous in the packed rows, the mirrored (J, I) tile goes through shared
// memory (a per-row gather of the lower triangle reads one 32-B sector per element).
// PackArgs::row0 holds the tile prefix of each matrix.
__global__ void __launch_bounds__(256) unpack_tiles_kernel(const __grid_constant__ PackArgs a) {
  __shared__ float tile[64][65];
  const int blk = blockIdx.x;
  int t = 0;
  while (t + 1 < a.n && a.row0[t + 1] <= blk) ++t;
  const int64_t d = a.d[t];
  const int T = int((d + 63) / 64);
  int k = blk - a.row0[t], I = 0;
  while (k >= T - I) k -= T - I, ++I;
  const int J = I + k;
  const int64_t i0 = int64_t(I) * 64, j0 = int64_t(J) * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const float* src = a.src[t];
  float* dst = a.dst[t];
  float v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int64_t i = i0 + ty + 4 * u, j = j0 + tx;
    const int64_t r = i < j ? i : j, c = i < j ? j : i;
    v[u] = (i < d && j < d) ? src[r * (2 * d - r + 1) / 2 + (c - r)] : 0.f;
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int64_t i = i0 + ty + 4 * u, j = j0 + tx;
    if (i < d && j < d) dst[i * d + j] = v[u];
    tile[ty + 4 * u][tx] = v[u];
  }
  if (I != J) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int64_t j = j0 + ty + 4 * u, i = i0 + tx;
      if (i < d && j < d) dst[j * d + i] = tile[tx][ty + 4 * u];
    }
  }
}

static int pack_batched(int n, const int32_t* dims, const float* const* src, float* const* dst, int unpack,
                        cudaStream_t s) {
  SPD_ARG(n >= 0 && (n == 0 || (dims && src && dst)), SPDKFAC_ERR_ARG, "bad batched pack arguments");
  for (int off = 0; off < n; off += kMaxPtrs) {
    PackArgs a{};
    a.n = std::min(kMaxPtrs, n - off);
    int rows = 0;
    for (int t = 0; t < a.n; ++t) {
      SPD_ARG(dims[off + t] >= 1, SPDKFAC_ERR_ARG, "dimension must be >= 1");
      a.src[t] = src[off + t];
      a.dst[t] = dst[off + t];
      a.d[t] = dims[off + t];
      a.row0[t] = rows;
      const int T = (dims[off + t] + 63) / 64;
      rows += unpack ? T * (T + 1) / 2 : dims[off + t];  // unpack: upper 64-tiles; pack: rows
    }
    a.row0[a.n] = rows;
    stat_begin(kCatPack, s);
    if (unpack) unpack_tiles_kernel<<<rows, 256, 0, s>>>(a);
    else pack_batched_kernel<<<rows, 256, 0, s>>>(a, 0);
    SPD_CHECK_LAUNCH();
    stat_end(kCatPack, s, 0, 0);
  }
  return SPDKFAC_OK;
}

}  // namespace spd

using namespace spd;

extern "C" {

const char* spdkfac_last_error(void) { return g_err; }
int spdkfac_version(void) { return 100; }

void spdkfac_stats_reset(int timing_mask) {
  std::lock_guard<std::mutex> lk(g_stat_mu);
  g_rec_used = 0;
  g_probe_used = 0;
  g_probe_cat.clear();
  g_timing = uint32_t(timing_mask) & ~g_probing;
  g_launches.store(0);
  for (int c = 0; c < kNumCats; ++c) g_cat_launches[c] = 0, g_cat_flops[c] = 0, g_cat_bytes[c] = 0;
}

uint64_t spdkfac_stats_launches(void) { return g_launches.load(); }

int spdkfac_stats_reserve(int n) {
  std::lock_guard<std::mutex> lk(g_stat_mu);
  while (int(g_recs.size()) < n) {
    StatRec r;
    SPD_CUDA(cudaEventCreate(&r.a));
    SPD_CUDA(cudaEventCreate(&r.b));
    g_recs.push_back(r);
  }
  return SPDKFAC_OK;
}

int spdkfac_stats_set_probes(int probe_mask, int n_slots) {
  std::lock_guard<std::mutex> lk(g_stat_mu);
  if (n_slots > 0 && size_t(n_slots) > g_probe_cap) {
    if (g_probes) SPD_CUDA(cudaFree(g_probes));
    g_probes = nullptr;
    g_probe_cap = 0;
    SPD_CUDA(cudaMalloc(&g_probes, sizeof(Probe) * size_t(n_slots)));
    SPD_CUDA(cudaMemset(g_probes, 0, sizeof(Probe) * size_t(n_slots)));
    g_probe_cap = size_t(n_slots);
  }
  g_probing = uint32_t(probe_mask);
  g_timing &= ~g_probing;
  g_probe_used = 0;
  g_probe_cat.clear();
  return SPDKFAC_OK;
}

int spdkfac_stats_read(int cat, double* ms, int64_t* launches, double* flops, double* bytes) {
  SPD_ARG(cat >= 0 && cat < kNumCats, SPDKFAC_ERR_ARG, "bad stats category");
  std::lock_guard<std::mutex> lk(g_stat_mu);
  double t = 0;
  if ((g_probing & (1u << cat)) && g_probe_used > 0) {  // probe stamps of the last run of each launch
    std::vector<Probe> h(g_probe_used);
    SPD_CUDA(cudaDeviceSynchronize());
    SPD_CUDA(cudaMemcpy(h.data(), g_probes, sizeof(Probe) * g_probe_used, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < g_probe_used; ++i)
      if (g_probe_cat[i] == cat && h[i].t1 > h[i].t0) t += double(h[i].t1 - h[i].t0) * 1e-6;
  }
  for (size_t i = 0; i < g_rec_used; ++i) {
    if (g_recs[i].cat != cat) continue;
    float e = 0;
    SPD_CUDA(cudaEventSynchronize(g_recs[i].b));
    SPD_CUDA(cudaEventElapsedTime(&e, g_recs[i].a, g_recs[i].b));
    t += e;
  }
  if (ms) *ms = t;
  if (launches) *launches = int64_t(g_cat_launches[cat]);
  if (flops) *flops = g_cat_flops[cat];
  if (bytes) *bytes = g_cat_bytes[cat];
  return SPDKFAC_OK;
}

int spdkfac_device_supported(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}

int spdkfac_pack_upper_f32(const float* full, int64_t d, int64_t ld, float* packed, void* stream) {
  SPD_ARG(d >= 1, SPDKFAC_ERR_ARG, "dimension must be >= 1");
  SPD_ARG(ld >= d && full && packed, SPDKFAC_ERR_ARG, "bad pack arguments");
  dim3 grid(unsigned(std::min<int64_t>(cdiv(d, 256), 16)), unsigned(d));
  stat_begin(kCatPack, static_cast<cudaStream_t>(stream));
  pack_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(full, d, ld, packed);
  SPD_CHECK_LAUNCH();
  stat_end(kCatPack, static_cast<cudaStream_t>(stream), 0, 8.0 * d * (d + 1) / 2);
  return SPDKFAC_OK;
}

int spdkfac_unpack_upper_f32(const float* packed, int64_t d, float* full, int64_t ld, void* stream) {
  SPD_ARG(d >= 1, SPDKFAC_ERR_ARG, "dimension must be >= 1");
  SPD_ARG(ld >= d && full && packed, SPDKFAC_ERR_ARG, "bad unpack arguments");
  dim3 grid(unsigned(std::min<int64_t>(cdiv(d, 256), 16)), unsigned(d));
  stat_begin(kCatPack, static_cast<cudaStream_t>(stream));
  unpack_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(packed, d, full, ld);
  SPD_CHECK_LAUNCH();
  stat_end(kCatPack, static_cast<cudaStream_t>(stream), 0, 4.0 * d * d);
  return SPDKFAC_OK;
}

int spdkfac_pack_upper_batched_f32(int n, const int32_t* dims, const float* const* full, float* const* packed,
                                   void* stream) {
  return pack_batched(n, dims, full, packed, 0, static_cast<cudaStream_t>(stream));
}

int spdkfac_unpack_upper_batched_f32(int n, const int32_t* dims, const float* const* packed, float* const* full,
                                     void* stream) {
  return pack_batched(n, dims, packed, full, 1, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
