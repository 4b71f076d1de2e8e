// NCCL collectives of the SPD-KFAC step (factor all-reduce, owner broadcast of CT
// inverses).  One communicator per process/GPU; calls are enqueued on the caller's
// stream (the optimizer's side streams), never synchronising the host.
#include <nccl.h>

#include "runtime.cuh"

struct spdkfac_comm {
  ncclComm_t comm;
  int rank, world;
};

#define SPD_NCCL(call)                                                                      \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess) {                                                                \
      ::spd::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, ncclGetErrorString(r_)); \
      return SPDKFAC_ERR_NCCL;                                                              \
    }                                                                                       \
  } while (0)

extern "C" {

int spdkfac_comm_unique_id(void* id_out) {
  SPD_ARG(id_out != nullptr, SPDKFAC_ERR_ARG, "null id");
  static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
  ncclUniqueId id;
  SPD_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return SPDKFAC_OK;
}

int spdkfac_comm_create(spdkfac_comm** out, const void* id, int rank, int world) {
  SPD_ARG(out && id && world >= 1 && rank >= 0 && rank < world, SPDKFAC_ERR_ARG, "bad communicator arguments");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  auto* c = new spdkfac_comm();
  c->rank = rank;
  c->world = world;
  ncclResult_t r = ncclCommInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    spd::set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
    return SPDKFAC_ERR_NCCL;
  }
  *out = c;
  return SPDKFAC_OK;
}

int spdkfac_comm_allreduce_sum_f32(spdkfac_comm* c, float* buf, size_t count, void* stream) {
  SPD_ARG(c && (buf || count == 0), SPDKFAC_ERR_ARG, "bad all-reduce arguments");
  if (count == 0) return SPDKFAC_OK;
  SPD_NCCL(ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, c->comm, static_cast<cudaStream_t>(stream)));
  return SPDKFAC_OK;
}

int spdkfac_comm_bcast_f32(spdkfac_comm* c, float* buf, size_t count, int root, void* stream) {
  SPD_ARG(c && (buf || count == 0) && root >= 0 && root < c->world, SPDKFAC_ERR_ARG, "bad broadcast arguments");
  if (count == 0) return SPDKFAC_OK;
  SPD_NCCL(ncclBroadcast(buf, buf, count, ncclFloat32, root, c->comm, static_cast<cudaStream_t>(stream)));
  return SPDKFAC_OK;
}

int spdkfac_comm_reduce_sum_f32(spdkfac_comm* c, float* buf, size_t count, int root, void* stream) {
  SPD_ARG(c && (buf || count == 0) && root >= 0 && root < c->world, SPDKFAC_ERR_ARG, "bad reduce arguments");
  if (count == 0) return SPDKFAC_OK;
  SPD_NCCL(ncclReduce(buf, buf, count, ncclFloat32, ncclSum, root, c->comm, static_cast<cudaStream_t>(stream)));
  return SPDKFAC_OK;
}

int spdkfac_comm_group_start(void) {
  SPD_NCCL(ncclGroupStart());
  return SPDKFAC_OK;
}

int spdkfac_comm_group_end(void) {
  SPD_NCCL(ncclGroupEnd());
  return SPDKFAC_OK;
}

void spdkfac_comm_destroy(spdkfac_comm* c) {
  if (!c) return;
  ncclCommDestroy(c->comm);
  delete c;
}

}  // extern "C"
