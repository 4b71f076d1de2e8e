/*
 * spdkfac.h -- C ABI of the B200-native SPD-KFAC optimizer-step library
 * (libspdkfac.so, sm_100a).  Drop-in boundary for the reference package
 * `kfacsched` (pkg/src/kfacsched), whose public operator API is re-exported at
 * pkg/src/kfacsched/__init__.py:5-69.  Each entry point below names the
 * reference function it replaces (file:line relative to /root/reference).
 *
 * Conventions
 *  - All tensor pointers are caller-owned DEVICE memory; `stream` is a
 *    cudaStream_t passed as void*.  Calls are stream-ordered and never
 *    synchronise the host, except spdkfac_*_info readers that say so.
 *  - No allocation inside calls: every call that needs scratch takes a
 *    caller-provided device workspace whose size the matching
 *    *_workspace_size() returns.  The workspace must stay alive until the
 *    stream work of the call (or of the plan) completes.
 *  - Arithmetic: fp32 storage; contractions on tcgen05 tensor cores with
 *    split-precision operands (3 x bf16 for factors and preconditioning,
 *    3 x tf32 for inverse updates), fp32 accumulation in TMEM.
 *  - Packed symmetric layout = the reference's: row-major upper triangle
 *    including the diagonal, element (i<=j) at i*(2d-i+1)/2 + (j-i)
 *    (pack_upper, linalg.py:181-184).
 *  - Return codes mirror the reference's exceptions.
 */
#ifndef SPDKFAC_H_
#define SPDKFAC_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SPDKFAC_API __attribute__((visibility("default")))
#else
#define SPDKFAC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SPDKFAC_OK 0
#define SPDKFAC_ERR_NOT_PD 1   /* NotPositiveDefiniteError(pivot), linalg.py:37-46,141-145 */
#define SPDKFAC_ERR_SHAPE 2    /* ValueError on shape mismatch, linalg.py:108-112,161-166 */
#define SPDKFAC_ERR_ARG 3      /* ValueError on bad argument (gamma<0, empty batch), linalg.py:138-139 */
#define SPDKFAC_ERR_CUDA 4
#define SPDKFAC_ERR_NCCL 5
#define SPDKFAC_ERR_UNSUPPORTED 6 /* not an sm_100 device */

/* Human-readable description of the last error on this thread. */
SPDKFAC_API const char* spdkfac_last_error(void);
SPDKFAC_API int spdkfac_version(void);
/* 1 iff the current device is sm_100 (B200) and the kernels can launch. */
SPDKFAC_API int spdkfac_device_supported(void);

/* Launch accounting for benchmarks: every kernel launch is counted; launches
 * of the categories in `timing_mask` (bit c = category c, -1 = all) are
 * bracketed by CUDA events on their own stream (events pre-created with
 * spdkfac_stats_reserve so that timing adds no driver allocation).
 * Categories: 0 factor stage (im2col/transpose + split), 1 factor SYRK
 * (tcgen05), 2 factor reduce+pack, 3 small inverse, 4 pivot inverse,
 * 5 panel, 6 inverse update (tcgen05), 7 inverse unpack/finalize,
 * 8 precondition split, 9 precondition GEMMs (tcgen05), 10 update apply,
 * 11 pack/unpack.  flops = algorithmic flops; stats_read
 * synchronises on the recorded events. */
SPDKFAC_API void spdkfac_stats_reset(int timing_mask);
SPDKFAC_API int spdkfac_stats_reserve(int n_launches);
SPDKFAC_API uint64_t spdkfac_stats_launches(void);
SPDKFAC_API int spdkfac_stats_read(int category, double* ms, int64_t* launches, double* flops, double* bytes);
/* In-kernel launch probes for the categories in probe_mask (bit = category): the first CTA of a
 * launch stamps its start, the last CTA its end (%globaltimer), with no stream or graph node, so a
 * graphed step can be timed per kernel category without perturbing it.  n_slots probe slots are
 * allocated once (outside any capture); each probed launch after spdkfac_stats_reset takes one.
 * spdkfac_stats_read reports the probe time of the last run of each launch for those categories. */
SPDKFAC_API int spdkfac_stats_set_probes(int probe_mask, int n_slots);

/* ------------------------------------------------------------------ factors
 * Replaces compute_factor_A / compute_factor_G / _factor_from_batch
 * (linalg.py:106-127) and the running-average/aggregation prologue of
 * _mean_sym (emulator.py:199-200).  Computes, into the packed buffer:
 *
 *   packed <- world_scale * ( decay * packed + (1 - decay) * scale * X^T X )
 *
 * (decay == 0 never reads `packed`).  The reference's factor is scale = 1/rows,
 * decay = 0, world_scale = 1; world_scale = 1/P pre-scales a rank's share of
 * an all-reduce(sum) mean.  X is described by a layout:
 *   SPDKFAC_ROWS     x = [rows][d] row-major (ld = row stride)     linear layer input / output grad
 *   SPDKFAC_CONV_A   x = NCHW activation; rows = im2col patches (c,kh,kw order) per output position
 *   SPDKFAC_SPATIAL  x = NCHW output gradient; rows = (b,h,w) positions, d = C
 *   SPDKFAC_CONV_A_NHWC   x = channels-last activation; patch rows ordered (kh,kw,c), the column
 *                         order of a channels-last conv weight viewed as [cout][kh*kw*cin]
 *   SPDKFAC_SPATIAL_NHWC  x = channels-last output gradient (rows [b*h*w][C])
 * A plan binds the shapes once and owns the split-precision staging buffers
 * and tile tables inside the workspace; run() takes the per-step pointers.
 */
#define SPDKFAC_ROWS 0
#define SPDKFAC_CONV_A 1
#define SPDKFAC_SPATIAL 2
#define SPDKFAC_CONV_A_NHWC 3
#define SPDKFAC_SPATIAL_NHWC 4

typedef struct spdkfac_factor_geom {
  int32_t layout;       /* SPDKFAC_ROWS / CONV_A / SPATIAL */
  int64_t n, c, h, w;   /* ROWS: n = rows, c = d, ld = w (row stride, >= d); h unused */
  int32_t kh, kw, stride_h, stride_w, pad_h, pad_w, dil_h, dil_w; /* CONV_A only */
} spdkfac_factor_geom;

typedef struct spdkfac_factor_plan spdkfac_factor_plan;

/* rows and dim of the factor this geometry produces */
SPDKFAC_API int spdkfac_factor_dims(const spdkfac_factor_geom* g, int64_t* rows, int64_t* dim);
SPDKFAC_API size_t spdkfac_factor_workspace_size(const spdkfac_factor_geom* g);
SPDKFAC_API int spdkfac_factor_plan_create(spdkfac_factor_plan** out, const spdkfac_factor_geom* g, void* ws, size_t ws_bytes,
                               void* stream);
SPDKFAC_API int spdkfac_factor_plan_run(spdkfac_factor_plan* p, const float* x, float scale, float decay, float world_scale,
                            float* packed_inout, void* stream);
/* run() in two halves: stage() reads x (im2col / transpose + precision split into the
 * plan's staging buffer) on the stream that owns x; compute() (tensor-core SYRK +
 * packed epilogue) reads only plan memory, so it may run on a side stream ordered
 * after stage() without extending the lifetime of x. */
SPDKFAC_API int spdkfac_factor_plan_stage(spdkfac_factor_plan* p, const float* x, void* stream);
SPDKFAC_API int spdkfac_factor_plan_compute(spdkfac_factor_plan* p, float scale, float decay, float world_scale,
                                            float* packed_inout, void* stream);
SPDKFAC_API void spdkfac_factor_plan_destroy(spdkfac_factor_plan* p);

/* A factor group: n layer-sides staged independently (stage(member, x) on the stream that
 * owns x) and reduced by ONE persistent tensor-core launch over all members' tiles
 * (compute()).  Each member writes packed_out[k] <- world_scale*(decay*old + (1-decay)*
 * scales[k]*X_k^T X_k).  The optimizer builds one group per fusion group of the plan
 * (planner.py:94-121), so a group's all-reduce follows its single compute launch. */
typedef struct spdkfac_factor_group spdkfac_factor_group;
SPDKFAC_API size_t spdkfac_factor_group_workspace_size(int n, const spdkfac_factor_geom* geoms);
SPDKFAC_API int spdkfac_factor_group_create(spdkfac_factor_group** out, int n, const spdkfac_factor_geom* geoms,
                                            float* const* packed_out, const float* scales, void* ws,
                                            size_t ws_bytes, void* stream);
SPDKFAC_API int spdkfac_factor_group_stage(spdkfac_factor_group* g, int member, const float* x, void* stream);
SPDKFAC_API int spdkfac_factor_group_compute(spdkfac_factor_group* g, float decay, float world_scale, void* stream);
SPDKFAC_API void spdkfac_factor_group_destroy(spdkfac_factor_group* g);
/* Introspection of a group's tile-engine choice for one member (tests and diagnostics):
 * out[0] = engine: 0 = single-CTA engine on staged bf16 planes, 1 = CTA-pair engine (cta_group::2,
 * 256x256 super tiles), 2 = single-CTA engine reading the fp32 rows itself (opt-in for row layouts,
 * environment SPDKFAC_F32_ROWS = max 128-blocks: no staging pass; the input must then be 16-byte
 * aligned and stay valid until compute; at most 40 such members per group, the rest are staged),
 * 3 = single-CTA engine gathering im2col tiles of the staged activation by TMA im2col loads
 * (channels-last k x k convolutions with C % 64 == 0: the staging pass writes the activation, not
 * its im2col rows; opt-in: environment SPDKFAC_IM2COL=1),
 * out[1] = split-K slices, out[2] = rows M, out[3] = dim d.  No device work. */
SPDKFAC_API int spdkfac_factor_group_describe(const spdkfac_factor_group* g, int member, int64_t out[4]);

/* ------------------------------------------------------------------ packing
 * pack_upper / unpack_upper (linalg.py:181-199) on device. `ld` = row stride
 * of the full matrix.  unpack writes both triangles. */
SPDKFAC_API int spdkfac_pack_upper_f32(const float* full, int64_t d, int64_t ld, float* packed, void* stream);
SPDKFAC_API int spdkfac_unpack_upper_f32(const float* packed, int64_t d, float* full, int64_t ld, void* stream);
/* Batched over n matrices (host arrays of device pointers). */
SPDKFAC_API int spdkfac_pack_upper_batched_f32(int n, const int32_t* dims, const float* const* full, float* const* packed,
                                   void* stream);
SPDKFAC_API int spdkfac_unpack_upper_batched_f32(int n, const int32_t* dims, const float* const* packed, float* const* full,
                                     void* stream);

/* ------------------------------------------------------------------ damped inverse
 * Replaces damped_inverse (linalg.py:130-149) for a batch of n factors:
 *   out_t = (unpack(packed_t) + gamma I)^-1, symmetrised, full d_t x d_t (ld = d_t)
 * Blocked Gauss-Jordan sweep (pivot blocks of 128 inverted in shared memory,
 * trailing updates as 3 x tf32 tcgen05 rank-128 updates).  info_dev[t] = 0 or
 * LAPACK-style failing pivot + 1 (the reference raises
 * NotPositiveDefiniteError(info-1)).  The plan binds dims and the in/out
 * pointers (host arrays of device pointers, copied at create). */
typedef struct spdkfac_inverse_plan spdkfac_inverse_plan;
SPDKFAC_API size_t spdkfac_inverse_workspace_size(int n, const int32_t* dims);
SPDKFAC_API int spdkfac_inverse_plan_create(spdkfac_inverse_plan** out, int n, const int32_t* dims, const float* const* packed_in,
                                float* const* out_full, int32_t* info_dev, void* ws, size_t ws_bytes, void* stream);
SPDKFAC_API int spdkfac_inverse_plan_run(spdkfac_inverse_plan* p, float gamma, void* stream);
SPDKFAC_API void spdkfac_inverse_plan_destroy(spdkfac_inverse_plan* p);

/* ------------------------------------------------------------------ precondition + update
 * Replaces precondition (linalg.py:152-167) and _apply_update
 * (emulator.py:203-208) for n layers:
 *   P_l = G_l^-1 . grad_l . A_l^-1      ([d_out][d_in] row-major)
 *   W_l <- W_l - alpha * P_l            (skipped when weight == NULL)
 *   precond_out_l <- P_l                (skipped when precond_out == NULL)
 * Two tcgen05 3 x bf16 GEMMs per layer, batched over layers.
 * a_inv / g_inv == NULL: that side's inverses were already staged into the plan's
 * split-precision operands by spdkfac_precond_plan_stage_inverses (e.g. on the stream that
 * inverted them, while the backward pass still runs), so run() only splits the gradients. */
typedef struct spdkfac_precond_plan spdkfac_precond_plan;
SPDKFAC_API size_t spdkfac_precond_workspace_size(int n, const int32_t* d_out, const int32_t* d_in);
SPDKFAC_API int spdkfac_precond_plan_create(spdkfac_precond_plan** out, int n, const int32_t* d_out, const int32_t* d_in,
                                void* ws, size_t ws_bytes, void* stream);
SPDKFAC_API int spdkfac_precond_plan_run(spdkfac_precond_plan* p, const float* const* g_inv, const float* const* grad,
                             const float* const* a_inv, float* const* weight, float alpha, float* const* precond_out,
                             void* stream);
/* Stage the inverses of n_sel layers (layers[i] indexes the plan's layers; inv[i] its full
 * fp32 inverse) into the plan's bf16 hi/lo operand planes: which = 0 for A^-1, 1 for G^-1. */
SPDKFAC_API int spdkfac_precond_plan_stage_inverses(spdkfac_precond_plan* p, int which, int n_sel, const int32_t* layers,
                                                    const float* const* inv, void* stream);
/* Same from packed upper inverses (the owner broadcast, emulator.py:256-262): one pass writes the
 * full fp32 inverse (full_out[i], may be NULL) and the operand planes. */
SPDKFAC_API int spdkfac_precond_plan_stage_packed(spdkfac_precond_plan* p, int which, int n_sel, const int32_t* layers,
                                                  const float* const* packed, float* const* full_out, void* stream);
SPDKFAC_API void spdkfac_precond_plan_destroy(spdkfac_precond_plan* p);

/* ------------------------------------------------------------------ collectives
 * NCCL over NVLink/NVSwitch for the factor all-reduce (_mean_sym,
 * emulator.py:199-200) and the owner broadcast of CT inverses (placement walk,
 * emulator.py:256-262).  The communicator is created from a unique id that
 * the host exchanges out of band (torch.distributed store). */
typedef struct spdkfac_comm spdkfac_comm;
SPDKFAC_API int spdkfac_comm_unique_id(void* id_out /* 128 bytes */);
SPDKFAC_API int spdkfac_comm_create(spdkfac_comm** out, const void* id /* 128 bytes */, int rank, int world);
SPDKFAC_API int spdkfac_comm_allreduce_sum_f32(spdkfac_comm* c, float* buf, size_t count, void* stream);
SPDKFAC_API int spdkfac_comm_bcast_f32(spdkfac_comm* c, float* buf, size_t count, int root, void* stream);
/* In-place sum onto `root` only (the other ranks' buffers are left unchanged).  Replaces the
 * all-reduce of a CT factor, whose aggregate only its inverse's owner reads (factor_decay == 0):
 * the reference's _mean_sym (emulator.py:199-200) restricted to the placement walk's owner
 * (emulator.py:247-262). */
SPDKFAC_API int spdkfac_comm_reduce_sum_f32(spdkfac_comm* c, float* buf, size_t count, int root, void* stream);
SPDKFAC_API int spdkfac_comm_group_start(void);
SPDKFAC_API int spdkfac_comm_group_end(void);
SPDKFAC_API void spdkfac_comm_destroy(spdkfac_comm* c);

/* ------------------------------------------------------------------ peer-memory factor aggregation
 * factor_comm = "peer" (csrc/peer.cu): the reference's factor sum (_mean_sym, emulator.py:199-200,
 * 236-241) restricted to the owner of each CT inverse (emulator.py:247-262), done by the SYRK
 * epilogue itself: every rank's factor-group launch stores its 1/P-scaled packed tiles into the
 * owner's inbox (CUDA-IPC mapping, one slot per source rank) over NVLink, then signals; the owner
 * waits for the P-1 signals of the group and adds the slots into its packed factor.
 *   alloc / free        a device allocation of its own (an IPC handle maps exactly it), zeroed
 *   handle / open/close cudaIpcGetMemHandle / OpenMemHandle (64-byte handle) / CloseMemHandle
 *   copy                stream-ordered copy-engine push of a contiguous range into a peer's inbox
 *   scatter_f32         the same range pushed to n_dst peers by SM stores over NVLink (16-byte vectors when
 *                       every dst shares src's address mod 16, else 4-byte)
 *   epoch_advance       epoch[0] += 1 on the stream (once per step, on every rank)
 *   signal              flags[q][slot * world + rank] = *epoch for every peer q != rank (release, sys scope)
 *   wait_sum            poll flags[slot * world + q] == *epoch for q != rank (timeout_s: *err = slot + 1
 *                       instead of hanging), then packed[s + i] += sum_{q != rank} inbox[q * stride + s + i]
 *                       for the n_segs (start, count) int64 pairs at segs_dev (device memory) */
SPDKFAC_API int spdkfac_peer_alloc(size_t bytes, void** out);
SPDKFAC_API int spdkfac_peer_free(void* p);
SPDKFAC_API int spdkfac_peer_handle(void* p, void* handle_out /* 64 bytes */);
SPDKFAC_API int spdkfac_peer_open(const void* handle /* 64 bytes */, void** out);
SPDKFAC_API int spdkfac_peer_close(void* p);
SPDKFAC_API int spdkfac_peer_copy(void* dst, const void* src, size_t bytes, void* stream);
SPDKFAC_API int spdkfac_peer_scatter_f32(float* const* dsts, int n_dst, const float* src, int64_t count, void* stream);
SPDKFAC_API int spdkfac_peer_epoch_advance(int* epoch, void* stream);
SPDKFAC_API int spdkfac_peer_signal(int* const* flags, int world, int rank, int slot, const int* epoch, void* stream);
SPDKFAC_API int spdkfac_peer_wait_sum(const int* flags, int world, int rank, int slot, const int* epoch, int* err,
                                      double timeout_s, float* packed, const float* inbox, int64_t stride,
                                      int n_segs, const int64_t* segs_dev, int64_t max_count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPDKFAC_H_ */
