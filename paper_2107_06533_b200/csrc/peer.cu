// Factor aggregation over NVLink / NVSwitch peer memory (factor_comm = "peer").
//
// The reference sums every worker's factors (_mean_sym, emulator.py:199-200 / 236-241) and
// then only the owner of a CT tensor's inverse reads the aggregate (placement walk,
// emulator.py:247-262).  Here the SYRK epilogue of every rank stores its 1/P-scaled packed
// factor tile STRAIGHT into the owner's inbox (a CUDA-IPC mapping of the owner's memory, one
// slot per source rank), tile by tile while the SYRK runs, so the transfer overlaps the math and
// no NCCL reduce is left on the step's critical path.  Per fusion group:
//
//   source rank r : SYRK launch (remote members' epilogue -> inbox[owner][r]) ; signal kernel:
//                   flag[owner][group][r] = epoch (system-scope release, after the SYRK in stream order)
//   owner         : wait kernel (acquire-poll the P-1 flags of the group, bounded by a timeout that
//                   records an error instead of hanging) ; sum kernel: packed[seg] += sum_r inbox[r][seg]
//                   over the owner's CT segments of the group, ranks in ascending order
//
// `epoch` is a device counter advanced once per step on every rank (also inside CUDA graphs),
// so a replayed graph signals and waits on fresh values without host involvement.
#include "runtime.cuh"

namespace spd {

__global__ void epoch_advance_kernel(int* epoch) { epoch[0] += 1; }

struct PeerBases {
  int* flags[kMaxPeers];
};

__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// thread q != me: flags_q[slot * P + me] = epoch
__global__ void peer_signal_kernel(PeerBases b, int world, int me, int slot, const int* __restrict__ epoch) {
  const int q = threadIdx.x;
  if (q >= world || q == me) return;
  const int e = *reinterpret_cast<const volatile int*>(epoch);
  __threadfence_system();  // the SYRK's peer stores (previous kernel in this stream) before the flag
  st_release_sys(b.flags[q] + int64_t(slot) * world + me, e);
}

// thread q != me polls flags[slot * P + q] until it equals epoch; a timeout sets *err (slot + 1)
__global__ void peer_wait_kernel(const int* flags, int world, int me, int slot, const int* __restrict__ epoch, int* err,
                                 uint64_t timeout_ns) {
  const int q = threadIdx.x;
  if (q >= world || q == me) return;
  const int e = *reinterpret_cast<const volatile int*>(epoch);
  const int* f = flags + int64_t(slot) * world + q;
  const uint64_t t0 = global_ns();
  while (ld_acquire_sys(f) != e) {
    if (global_ns() - t0 > timeout_ns) {
      atomicExch(err, slot + 1);
      return;
    }
    __nanosleep(256);
  }
}

struct PeerDsts {
  float* p[kMaxPeers];
};

// src[0, n) -> every dst: SM-driven NVLink stores, 16-byte vectors when src and every dst share their
// address mod 16 (the callers' regions sit at equal offsets of 256-aligned rows), else scalar
__global__ void __launch_bounds__(512) peer_scatter_kernel(PeerDsts d, int n_dst, const float* __restrict__ src,
                                                           int64_t n, int vec) {
  if (!vec) {  // some destination not co-aligned with the source: scalar stores
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
      const float v = src[i];
      for (int k = 0; k < n_dst; ++k) d.p[k][i] = v;
    }
    return;
  }
  const int64_t mis = int64_t((16 - (reinterpret_cast<uintptr_t>(src) & 15)) & 15) / 4;
  const int64_t head = n < mis ? n : mis;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x, nth = int64_t(gridDim.x) * blockDim.x;
  if (tid < head) {
    const float v = src[tid];
    for (int k = 0; k < n_dst; ++k) d.p[k][tid] = v;
  }
  const int64_t nv = (n - head) / 4;
  const float4* s4 = reinterpret_cast<const float4*>(src + head);
  for (int64_t i = tid; i < nv; i += nth) {
    const float4 v = __ldcs(s4 + i);
    for (int k = 0; k < n_dst; ++k) reinterpret_cast<float4*>(d.p[k] + head)[i] = v;
  }
  const int64_t t0 = head + nv * 4;
  if (tid < n - t0) {
    const float v = src[t0 + tid];
    for (int k = 0; k < n_dst; ++k) d.p[k][t0 + tid] = v;
  }
}

struct PeerSeg {
  int64_t start, count;
};

// packed[s + i] += sum_{q != me, ascending} inbox[q * stride + s + i] over the segments (blockIdx.y)
__global__ void __launch_bounds__(256) peer_sum_kernel(float* __restrict__ packed, const float* __restrict__ inbox,
                                                       int64_t stride, int world, int me,
                                                       const PeerSeg* __restrict__ segs) {
  const PeerSeg sg = segs[blockIdx.y];
  float* dst = packed + sg.start;
  const float* src = inbox + sg.start;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < sg.count; i += int64_t(gridDim.x) * blockDim.x) {
    float v = dst[i];
    for (int q = 0; q < world; ++q)
      if (q != me) v += __ldcs(src + q * stride + i);
    dst[i] = v;
  }
}

}  // namespace spd

using namespace spd;

extern "C" {

int spdkfac_peer_alloc(size_t bytes, void** out) {
  SPD_ARG(out && bytes > 0, SPDKFAC_ERR_ARG, "bad peer allocation arguments");
  void* p = nullptr;
  SPD_CUDA(cudaMalloc(&p, bytes));  // a whole allocation: its IPC handle maps exactly this range
  SPD_CUDA(cudaMemset(p, 0, bytes));
  *out = p;
  return SPDKFAC_OK;
}

int spdkfac_peer_free(void* p) {
  if (p) SPD_CUDA(cudaFree(p));
  return SPDKFAC_OK;
}

int spdkfac_peer_handle(void* p, void* handle_out) {
  SPD_ARG(p && handle_out, SPDKFAC_ERR_ARG, "bad peer handle arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "unexpected IPC handle size");
  cudaIpcMemHandle_t h;
  SPD_CUDA(cudaIpcGetMemHandle(&h, p));
  memcpy(handle_out, &h, sizeof(h));
  return SPDKFAC_OK;
}

int spdkfac_peer_open(const void* handle, void** out) {
  SPD_ARG(handle && out, SPDKFAC_ERR_ARG, "bad peer open arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  SPD_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *out = p;
  return SPDKFAC_OK;
}

int spdkfac_peer_close(void* p) {
  if (p) SPD_CUDA(cudaIpcCloseMemHandle(p));
  return SPDKFAC_OK;
}

int spdkfac_peer_copy(void* dst, const void* src, size_t bytes, void* stream) {
  SPD_ARG((dst && src) || bytes == 0, SPDKFAC_ERR_ARG, "bad peer copy arguments");
  if (bytes == 0) return SPDKFAC_OK;
  // copy engine over NVLink: no SM time, contiguous packets (the SYRK epilogue's per-row stores
  // would reach the peer as 4-byte writes)
  SPD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return SPDKFAC_OK;
}

int spdkfac_peer_scatter_f32(float* const* dsts, int n_dst, const float* src, int64_t count, void* stream) {
  SPD_ARG(dsts && n_dst >= 0 && n_dst <= kMaxPeers && (src || count == 0) && count >= 0, SPDKFAC_ERR_ARG,
          "bad peer scatter arguments");
  if (count == 0 || n_dst == 0) return SPDKFAC_OK;
  PeerDsts d{};
  int vec = 1;
  for (int k = 0; k < n_dst; ++k) {
    SPD_ARG(dsts[k], SPDKFAC_ERR_ARG, "peer scatter: null destination %d", k);
    if ((reinterpret_cast<uintptr_t>(dsts[k]) ^ reinterpret_cast<uintptr_t>(src)) & 15) vec = 0;
    d.p[k] = dsts[k];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(cdiv(count / 4 + 1, 512 * 4), 64)));
  stat_begin(kCatFactorReduce, s);
  peer_scatter_kernel<<<grid, 512, 0, s>>>(d, n_dst, src, count, vec);
  SPD_CHECK_LAUNCH();
  stat_end(kCatFactorReduce, s, 0, double(count) * 4 * (1 + n_dst));
  return SPDKFAC_OK;
}

int spdkfac_peer_epoch_advance(int* epoch, void* stream) {
  SPD_ARG(epoch, SPDKFAC_ERR_ARG, "null epoch");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  stat_begin(kCatFactorReduce, s);
  epoch_advance_kernel<<<1, 1, 0, s>>>(epoch);
  SPD_CHECK_LAUNCH();
  stat_end(kCatFactorReduce, s, 0, 0);
  return SPDKFAC_OK;
}

int spdkfac_peer_signal(int* const* flags, int world, int rank, int slot, const int* epoch, void* stream) {
  SPD_ARG(flags && epoch && world >= 1 && world <= kMaxPeers && rank >= 0 && rank < world && slot >= 0,
          SPDKFAC_ERR_ARG, "bad peer signal arguments");
  PeerBases b{};
  for (int q = 0; q < world; ++q) {
    SPD_ARG(q == rank || flags[q], SPDKFAC_ERR_ARG, "missing peer flag base %d", q);
    b.flags[q] = flags[q];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  stat_begin(kCatFactorReduce, s);
  peer_signal_kernel<<<1, 32, 0, s>>>(b, world, rank, slot, epoch);
  SPD_CHECK_LAUNCH();
  stat_end(kCatFactorReduce, s, 0, 0);
  return SPDKFAC_OK;
}

int spdkfac_peer_wait_sum(const int* flags, int world, int rank, int slot, const int* epoch, int* err,
                          double timeout_s, float* packed, const float* inbox, int64_t stride, int n_segs,
                          const int64_t* segs_dev, int64_t max_count, void* stream) {
  SPD_ARG(flags && epoch && err && world >= 1 && world <= kMaxPeers && rank >= 0 && rank < world && slot >= 0,
          SPDKFAC_ERR_ARG, "bad peer wait arguments");
  SPD_ARG(n_segs == 0 || (packed && inbox && segs_dev && stride > 0), SPDKFAC_ERR_ARG, "bad peer sum arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  stat_begin(kCatFactorReduce, s);
  peer_wait_kernel<<<1, 32, 0, s>>>(flags, world, rank, slot, epoch, err, uint64_t(timeout_s * 1e9));
  SPD_CHECK_LAUNCH();
  stat_end(kCatFactorReduce, s, 0, 0);
  if (n_segs > 0 && max_count > 0) {
    const unsigned gx = unsigned(std::min<int64_t>(cdiv(max_count, 256 * 4), 296));
    stat_begin(kCatFactorReduce, s);
    peer_sum_kernel<<<dim3(gx, unsigned(n_segs)), 256, 0, s>>>(packed, inbox, stride, world, rank,
                                                                reinterpret_cast<const PeerSeg*>(segs_dev));
    SPD_CHECK_LAUNCH();
    stat_end(kCatFactorReduce, s, 0, 0);
  }
  return SPDKFAC_OK;
}

}  // extern "C"
