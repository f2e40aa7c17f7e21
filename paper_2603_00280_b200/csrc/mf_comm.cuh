// mf_comm.cuh -- the multi-GPU exchange of a sharded render (SURVEY.md
// 8(b) "mf_reduce", 8(e)): included at the end of mf_kernels.cu (uses its
// fail / MF_CUDA / g_launches).
//
// NCCL is resolved at run time with dlopen: the copy already loaded in the
// process (torch's libnccl.so.2) when there is one, else the system's, or
// $MF_NCCL_PATH.  Only the handful of entry points below are bound; the
// types are the stable parts of nccl.h's ABI (ncclUniqueId = 128 bytes,
// ncclFloat32 = 7, ncclSum = 0, ncclComm_t an opaque pointer).
#pragma once

#include <dlfcn.h>

#include <cstdlib>

namespace {

struct NcclId {
  char internal[MF_COMM_ID_BYTES];
};
typedef int (*nccl_get_unique_id_t)(NcclId*);
typedef int (*nccl_comm_init_rank_t)(void**, int, NcclId, int);
typedef int (*nccl_comm_destroy_t)(void*);
typedef int (*nccl_comm_count_t)(const void*, int*);
typedef int (*nccl_comm_user_rank_t)(const void*, int*);
typedef int (*nccl_reduce_t)(const void*, void*, size_t, int, int, int, void*, cudaStream_t);
typedef int (*nccl_send_t)(const void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_recv_t)(void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_group_t)(void);
typedef const char* (*nccl_error_string_t)(int);

constexpr int kNcclFloat32 = 7;
constexpr int kNcclSum = 0;

struct NcclApi {
  bool ok = false;
  std::string why;
  nccl_get_unique_id_t get_unique_id = nullptr;
  nccl_comm_init_rank_t comm_init_rank = nullptr;
  nccl_comm_destroy_t comm_destroy = nullptr;
  nccl_comm_count_t comm_count = nullptr;
  nccl_comm_user_rank_t comm_user_rank = nullptr;
  nccl_reduce_t reduce = nullptr;
  nccl_send_t send = nullptr;
  nccl_recv_t recv = nullptr;
  nccl_group_t group_start = nullptr;
  nccl_group_t group_end = nullptr;
  nccl_error_string_t error_string = nullptr;
};

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  std::call_once(once, [] {
    void* h = nullptr;
    const char* env = std::getenv("MF_NCCL_PATH");
    if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "not found");
      return;
    }
#define MF_NCCL_SYM(field, name)                                        \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));    \
  if (!api.field) {                                                     \
    api.why = std::string("libnccl lacks ") + name;                     \
    return;                                                             \
  }
    MF_NCCL_SYM(get_unique_id, "ncclGetUniqueId");
    MF_NCCL_SYM(comm_init_rank, "ncclCommInitRank");
    MF_NCCL_SYM(comm_destroy, "ncclCommDestroy");
    MF_NCCL_SYM(comm_count, "ncclCommCount");
    MF_NCCL_SYM(comm_user_rank, "ncclCommUserRank");
    MF_NCCL_SYM(reduce, "ncclReduce");
    MF_NCCL_SYM(send, "ncclSend");
    MF_NCCL_SYM(recv, "ncclRecv");
    MF_NCCL_SYM(group_start, "ncclGroupStart");
    MF_NCCL_SYM(group_end, "ncclGroupEnd");
    MF_NCCL_SYM(error_string, "ncclGetErrorString");
#undef MF_NCCL_SYM
    api.ok = true;
  });
  return api;
}

#define MF_NCCL(call)                                                                  \
  do {                                                                                 \
    int r_ = (call);                                                                   \
    if (r_ != 0)                                                                       \
      return fail(MF_ERR_CUDA, std::string(#call) + ": " + nccl().error_string(r_));  \
  } while (0)

// root's fixed-order sum: buf[i] = v_0[i] + v_1[i] + ... + v_{n-1}[i], the
// root's own contribution read from buf, the others from the receive slots
__global__ void __launch_bounds__(256) ordered_sum_kernel(float* buf, const float* slots,
                                                          size_t count, int nranks, int root) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    float own = buf[i];
    float acc = 0.0f;
    for (int r = 0; r < nranks; ++r) {
      float v = r == root ? own : __ldg(slots + (size_t)r * count + i);
      acc = r == 0 ? v : acc + v;
    }
    buf[i] = acc;
  }
}

}  // namespace

extern "C" {

int mf_comm_unique_id(unsigned char id_out[MF_COMM_ID_BYTES]) {
  if (!id_out) return fail(MF_ERR_PARAM, "null argument");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(MF_ERR_UNSUPPORTED, n.why);
  NcclId id;
  MF_NCCL(n.get_unique_id(&id));
  std::memcpy(id_out, id.internal, MF_COMM_ID_BYTES);
  return MF_OK;
}

int mf_comm_init(const unsigned char id[MF_COMM_ID_BYTES], int nranks, int rank, void** comm_out) {
  if (!id || !comm_out) return fail(MF_ERR_PARAM, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(MF_ERR_PARAM, "bad rank / nranks");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(MF_ERR_UNSUPPORTED, n.why);
  NcclId nid;
  std::memcpy(nid.internal, id, MF_COMM_ID_BYTES);
  void* comm = nullptr;
  MF_NCCL(n.comm_init_rank(&comm, nranks, nid, rank));
  *comm_out = comm;
  return MF_OK;
}

int mf_comm_destroy(void* comm) {
  if (!comm) return MF_OK;
  const NcclApi& n = nccl();
  if (!n.ok) return fail(MF_ERR_UNSUPPORTED, n.why);
  MF_NCCL(n.comm_destroy(comm));
  return MF_OK;
}

int mf_reduce(void* comm, float* d_buf, size_t count, int root, int mode, void* stream) {
  if (!comm || (!d_buf && count)) return fail(MF_ERR_PARAM, "null argument");
  if (mode != MF_REDUCE_NCCL && mode != MF_REDUCE_ORDERED)
    return fail(MF_ERR_PARAM, "unknown reduce mode " + std::to_string(mode));
  const NcclApi& n = nccl();
  if (!n.ok) return fail(MF_ERR_UNSUPPORTED, n.why);
  int nranks = 0, rank = 0;
  MF_NCCL(n.comm_count(comm, &nranks));
  MF_NCCL(n.comm_user_rank(comm, &rank));
  if (root < 0 || root >= nranks) return fail(MF_ERR_PARAM, "root out of range");
  cudaStream_t st = (cudaStream_t)stream;
  if (count == 0) return MF_OK;
  if (mode == MF_REDUCE_NCCL) {
    MF_NCCL(n.reduce(d_buf, d_buf, count, kNcclFloat32, kNcclSum, root, comm, st));
    return MF_OK;
  }
  if (nranks == 1) return MF_OK;
  if (rank != root) {
    MF_NCCL(n.send(d_buf, count, kNcclFloat32, root, comm, st));
    return MF_OK;
  }
  int rc = retain_pool_memory();
  if (rc) return rc;
  float* slots = nullptr;
  MF_CUDA(cudaMallocAsync((void**)&slots, count * nranks * sizeof(float), st));
  MF_NCCL(n.group_start());
  for (int r = 0; r < nranks; ++r)
    if (r != root) {
      int e = n.recv(slots + (size_t)r * count, count, kNcclFloat32, r, comm, st);
      if (e != 0) {
        n.group_end();
        cudaFreeAsync(slots, st);
        return fail(MF_ERR_CUDA, std::string("ncclRecv: ") + n.error_string(e));
      }
    }
  MF_NCCL(n.group_end());
  int sms = 148, dev = 0;
  MF_CUDA(cudaGetDevice(&dev));
  MF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  size_t blocks = std::min<size_t>((count + 255) / 256, (size_t)sms * 8);
  ordered_sum_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_buf, slots, count, nranks, root);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  MF_CUDA(cudaFreeAsync(slots, st));
  return MF_OK;
}

}  // extern "C"
