// comm.cu — NCCL and in-process transports of the multi-GPU collectives (see comm.cuh).
#include <dlfcn.h>
#include <nccl.h>  // types only: every NCCL function is resolved with dlsym

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/fmm.h"
#include "comm.cuh"

// ---- NCCL (dlopen) ------------------------------------------------------------------------------
namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl(std::string &err) {
  static NcclApi api;
  static std::once_flag once;
  static std::string load_err;
  std::call_once(once, [] {
    void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      load_err = std::string("dlopen libnccl.so.2: ") + dlerror();
      return;
    }
#define SYM(f)                                                     \
  *(void **)(&api.f) = dlsym(lib, "nccl" #f);                      \
  if (!api.f) {                                                    \
    load_err = "libnccl.so.2 lacks nccl" #f;                        \
    return;                                                        \
  }
    SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(AllReduce) SYM(AllGather) SYM(Send)
    SYM(Recv) SYM(GroupStart) SYM(GroupEnd) SYM(GetErrorString)
#undef SYM
    api.ok = true;
  });
  if (!api.ok) err = load_err;
  return api;
}

ncclDataType_t nccl_type(int t) {
  switch (t) {
    case CT_I32: return ncclInt32;
    case CT_U32: return ncclUint32;
    case CT_I64: return ncclInt64;
    case CT_F32: return ncclFloat32;
    default: return ncclFloat64;
  }
}

struct NcclComm : FmmComm {
  ncclComm_t c = nullptr;
  NcclApi *api = nullptr;
  int check(ncclResult_t r, const char *what) {
    if (r == ncclSuccess) return FMM_OK;
    err = std::string(what) + ": " + api->GetErrorString(r);
    return FMM_E_NCCL;
  }
  ~NcclComm() override {
    if (c) api->CommDestroy(c);
  }
  int allreduce(void *d_buf, size_t count, int type, int op, cudaStream_t st) override {
    if (!count) return FMM_OK;
    const ncclRedOp_t o = op == CO_SUM ? ncclSum : op == CO_MAX ? ncclMax : ncclMin;
    return check(api->AllReduce(d_buf, d_buf, count, nccl_type(type), o, c, st), "ncclAllReduce");
  }
  int allgather(const void *d_send, void *d_recv, size_t bytes, cudaStream_t st) override {
    return check(api->AllGather(d_send, d_recv, bytes, ncclChar, c, st), "ncclAllGather");
  }
  int alltoallv(const void *d_send, const size_t *scnt, const size_t *sdsp, void *d_recv,
                const size_t *rcnt, const size_t *rdsp, cudaStream_t st) override {
    // the self segment is a device copy; the peers exchange in one NCCL group (ncclSend/ncclRecv
    // pairs; NVSwitch gives every pair full bandwidth, so no ring / hypercube schedule is needed)
    if (scnt[rank]) {
      if (cudaMemcpyAsync((char *)d_recv + rdsp[rank], (const char *)d_send + sdsp[rank], scnt[rank],
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
        err = "alltoallv self copy failed";
        return FMM_E_CUDA;
      }
    }
    if (int rc = check(api->GroupStart(), "ncclGroupStart")) return rc;
    int rc = FMM_OK;
    for (int r = 0; r < nranks && !rc; ++r) {
      if (r == rank) continue;
      if (scnt[r]) rc = check(api->Send((const char *)d_send + sdsp[r], scnt[r], ncclChar, r, c, st), "ncclSend");
      if (!rc && rcnt[r]) rc = check(api->Recv((char *)d_recv + rdsp[r], rcnt[r], ncclChar, r, c, st), "ncclRecv");
    }
    const int rc2 = check(api->GroupEnd(), "ncclGroupEnd");
    return rc ? rc : rc2;
  }
};
}  // namespace

int comm_nccl_unique_id(unsigned char id[128], std::string &err) {
  NcclApi &api = nccl(err);
  if (!api.ok) return FMM_E_NCCL;
  ncclUniqueId u;
  const ncclResult_t r = api.GetUniqueId(&u);
  if (r != ncclSuccess) {
    err = std::string("ncclGetUniqueId: ") + api.GetErrorString(r);
    return FMM_E_NCCL;
  }
  memcpy(id, u.internal, 128);
  return FMM_OK;
}

FmmComm *comm_nccl_create(int nranks, int rank, const unsigned char id[128], std::string &err) {
  NcclApi &api = nccl(err);
  if (!api.ok) return nullptr;
  ncclUniqueId u;
  memcpy(u.internal, id, 128);
  NcclComm *c = new NcclComm();
  c->api = &api;
  c->nranks = nranks;
  c->rank = rank;
  const ncclResult_t r = api.CommInitRank(&c->c, nranks, u, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + api.GetErrorString(r);
    c->c = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

// ---- in-process group ---------------------------------------------------------------------------
struct fmm_group {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  // per-rank slots posted between barriers
  std::vector<const void *> ptr;
  std::vector<const size_t *> cnt, dsp;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

fmm_group *comm_group_create(int nranks) {
  fmm_group *g = new fmm_group();
  g->n = nranks;
  g->ptr.assign(nranks, nullptr);
  g->cnt.assign(nranks, nullptr);
  g->dsp.assign(nranks, nullptr);
  return g;
}
void comm_group_destroy(fmm_group *g) { delete g; }

namespace {
constexpr int kMaxLocal = 16;
struct SrcPtrs {
  const void *p[kMaxLocal];
};

template <class T, int OP>
__global__ void k_reduce(T *dst, SrcPtrs s, int nsrc, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    T v = ((const T *)s.p[0])[i];
    for (int r = 1; r < nsrc; ++r) {
      const T w = ((const T *)s.p[r])[i];
      v = OP == CO_SUM ? v + w : OP == CO_MAX ? (w > v ? w : v) : (w < v ? w : v);
    }
    dst[i] = v;
  }
}

template <class T>
void launch_reduce(void *dst, const SrcPtrs &s, int nsrc, size_t count, int op, cudaStream_t st) {
  const int blocks = (int)std::min<size_t>((count + 255) / 256, 148 * 8);
  if (op == CO_SUM) k_reduce<T, CO_SUM><<<blocks, 256, 0, st>>>((T *)dst, s, nsrc, count);
  else if (op == CO_MAX) k_reduce<T, CO_MAX><<<blocks, 256, 0, st>>>((T *)dst, s, nsrc, count);
  else k_reduce<T, CO_MIN><<<blocks, 256, 0, st>>>((T *)dst, s, nsrc, count);
}

size_t type_size(int t) { return t == CT_I64 || t == CT_F64 ? 8 : 4; }

struct LocalComm : FmmComm {
  fmm_group *g = nullptr;
  void *tmp = nullptr;
  size_t tmp_cap = 0;
  ~LocalComm() override {
    if (tmp) cudaFree(tmp);
  }
  int cuda(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return FMM_OK;
    err = std::string(what) + ": " + cudaGetErrorString(e);
    return FMM_E_CUDA;
  }
  int allreduce(void *d_buf, size_t count, int type, int op, cudaStream_t st) override {
    // every rank reduces all ranks' buffers into its own scratch, then (after a second barrier,
    // when nobody reads the inputs any more) copies the result over its buffer
    const size_t bytes = count * type_size(type);
    int rc = FMM_OK;
    if (bytes > tmp_cap) {
      if (tmp) cudaFree(tmp);
      tmp = nullptr;
      tmp_cap = 0;
      rc = cuda(cudaMalloc(&tmp, bytes), "cudaMalloc");
      if (!rc) tmp_cap = bytes;
    }
    if (!rc) rc = cuda(cudaStreamSynchronize(st), "sync");
    g->ptr[rank] = d_buf;
    g->barrier();
    if (!rc && count) {
      SrcPtrs s{};
      for (int r = 0; r < nranks; ++r) s.p[r] = g->ptr[r];
      switch (type) {
        case CT_I32: launch_reduce<int>(tmp, s, nranks, count, op, st); break;
        case CT_U32: launch_reduce<unsigned>(tmp, s, nranks, count, op, st); break;
        case CT_I64: launch_reduce<long long>(tmp, s, nranks, count, op, st); break;
        case CT_F32: launch_reduce<float>(tmp, s, nranks, count, op, st); break;
        default: launch_reduce<double>(tmp, s, nranks, count, op, st); break;
      }
      rc = cuda(cudaStreamSynchronize(st), "reduce");
    }
    g->barrier();
    if (!rc && count) rc = cuda(cudaMemcpyAsync(d_buf, tmp, bytes, cudaMemcpyDeviceToDevice, st), "copy");
    if (!rc) rc = cuda(cudaStreamSynchronize(st), "sync");
    return rc;
  }
  int allgather(const void *d_send, void *d_recv, size_t bytes, cudaStream_t st) override {
    int rc = cuda(cudaStreamSynchronize(st), "sync");
    g->ptr[rank] = d_send;
    g->barrier();
    for (int r = 0; r < nranks && !rc && bytes; ++r)
      rc = cuda(cudaMemcpyAsync((char *)d_recv + r * bytes, g->ptr[r], bytes, cudaMemcpyDeviceToDevice, st), "copy");
    if (!rc) rc = cuda(cudaStreamSynchronize(st), "sync");
    g->barrier();
    return rc;
  }
  int alltoallv(const void *d_send, const size_t *scnt, const size_t *sdsp, void *d_recv,
                const size_t *rcnt, const size_t *rdsp, cudaStream_t st) override {
    int rc = cuda(cudaStreamSynchronize(st), "sync");
    g->ptr[rank] = d_send;
    g->cnt[rank] = scnt;
    g->dsp[rank] = sdsp;
    g->barrier();
    for (int r = 0; r < nranks && !rc; ++r) {
      const size_t b = g->cnt[r][rank];
      if (b != rcnt[r]) {
        err = "alltoallv: send/receive sizes disagree";
        rc = FMM_E_INVALID;
        break;
      }
      if (b) rc = cuda(cudaMemcpyAsync((char *)d_recv + rdsp[r], (const char *)g->ptr[r] + g->dsp[r][rank], b,
                                       cudaMemcpyDeviceToDevice, st), "copy");
    }
    if (!rc) rc = cuda(cudaStreamSynchronize(st), "sync");
    g->barrier();
    return rc;
  }
};
}  // namespace

FmmComm *comm_local_create(fmm_group *g, int rank, std::string &err) {
  if (!g || rank < 0 || rank >= g->n || g->n > kMaxLocal) {
    err = "bad in-process group or rank";
    return nullptr;
  }
  LocalComm *c = new LocalComm();
  c->g = g;
  c->nranks = g->n;
  c->rank = rank;
  return c;
}
