// comm.cuh — the collectives of the multi-GPU path, internal to libfmm.so.
//
// One handle per rank (one process per GPU). The distributed evaluation in fmm_api.cu needs five
// stream-ordered collectives on device buffers; two transports implement them:
//   * NcclComm  — NCCL over NVLink / NVSwitch (fmm_create_dist). libnccl.so.2 is dlopen'ed on first
//                 use, so single-GPU users do not depend on it (and a process that already loaded
//                 torch's NCCL reuses that copy).
//   * LocalComm — the ranks are handles of ONE process (fmm_group_create / fmm_create_in_group),
//                 each driven by its own host thread; collectives are device-to-device copies and
//                 a reduction kernel between barrier points. It runs the identical distributed
//                 algorithm on a single GPU, which is how the multi-rank logic is tested here.
// Every call returns 0 or an FMM_E_* code; `err` holds the message.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>

enum CommType { CT_I32 = 0, CT_U32 = 1, CT_I64 = 2, CT_F32 = 3, CT_F64 = 4 };
enum CommOp { CO_SUM = 0, CO_MAX = 1, CO_MIN = 2 };

struct FmmComm {
  int nranks = 1, rank = 0;
  std::string err;
  virtual ~FmmComm() {}
  // in place on a device buffer
  virtual int allreduce(void *d_buf, size_t count, int type, int op, cudaStream_t st) = 0;
  // d_recv[r * bytes ...] = rank r's d_send[0 .. bytes)
  virtual int allgather(const void *d_send, void *d_recv, size_t bytes, cudaStream_t st) = 0;
  // byte counts / displacements on the host, per peer
  virtual int alltoallv(const void *d_send, const size_t *scnt, const size_t *sdsp, void *d_recv,
                        const size_t *rcnt, const size_t *rdsp, cudaStream_t st) = 0;
};

struct fmm_group;  // opaque (include/fmm.h): the shared state of a LocalComm group

int comm_nccl_unique_id(unsigned char id[128], std::string &err);
FmmComm *comm_nccl_create(int nranks, int rank, const unsigned char id[128], std::string &err);
fmm_group *comm_group_create(int nranks);
void comm_group_destroy(fmm_group *g);
FmmComm *comm_local_create(fmm_group *g, int rank, std::string &err);
