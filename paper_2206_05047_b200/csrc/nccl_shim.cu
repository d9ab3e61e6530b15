// nccl_shim.cu — NCCL entry points loaded at run time (dlopen), so liblfsr.so has
// no link-time NCCL dependency and single-GPU users never load it.  Only the
// handful of calls the strip decomposition needs.
#include "nccl_shim.h"

#include <dlfcn.h>
#include <cstdlib>
#include <mutex>

namespace lfsr {

namespace {
struct Api {
  bool ok = false;
  std::string err;
  int (*GetUniqueId)(NcclUniqueId*) = nullptr;
  int (*CommInitRank)(void**, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*CommAbort)(void*) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
Api g_api;
std::once_flag g_once;

void load() {
  // LFSR_NCCL_LIB: an explicit library path (tests point it at their NCCL test double,
  // tests/fake_nccl, to run this path with several processes on one GPU)
  const char* env = getenv("LFSR_NCCL_LIB");
  const char* names[] = {env && env[0] ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) {
    g_api.err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
    return;
  }
#define SYM(field, name)                                                    \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, name));   \
  if (!g_api.field) {                                                       \
    g_api.err = std::string("missing NCCL symbol ") + name;                 \
    return;                                                                 \
  }
  SYM(GetUniqueId, "ncclGetUniqueId")
  SYM(CommInitRank, "ncclCommInitRank")
  SYM(CommDestroy, "ncclCommDestroy")
  SYM(CommAbort, "ncclCommAbort")
  SYM(Send, "ncclSend")
  SYM(Recv, "ncclRecv")
  SYM(AllReduce, "ncclAllReduce")
  SYM(Broadcast, "ncclBroadcast")
  SYM(GroupStart, "ncclGroupStart")
  SYM(GroupEnd, "ncclGroupEnd")
  SYM(GetErrorString, "ncclGetErrorString")
#undef SYM
  g_api.ok = true;
}
}  // namespace

bool nccl_available(std::string* why) {
  std::call_once(g_once, load);
  if (!g_api.ok && why) *why = g_api.err;
  return g_api.ok;
}

const char* nccl_error(int code) { return g_api.GetErrorString ? g_api.GetErrorString(code) : "NCCL unavailable"; }

int nccl_comm_init(void** comm, int nranks, const void* uid, int rank) {
  NcclUniqueId id;
  memcpy(id.internal, uid, sizeof id.internal);
  return g_api.CommInitRank(comm, nranks, id, rank);
}
int nccl_comm_destroy(void* comm) { return g_api.CommDestroy(comm); }
int nccl_comm_abort(void* comm) { return g_api.CommAbort(comm); }
int nccl_group_start() { return g_api.GroupStart(); }
int nccl_group_end() { return g_api.GroupEnd(); }
int nccl_send_f32(const float* buf, size_t n, int peer, void* comm, cudaStream_t st) {
  return g_api.Send(buf, n, kNcclFloat32, peer, comm, st);
}
int nccl_recv_f32(float* buf, size_t n, int peer, void* comm, cudaStream_t st) {
  return g_api.Recv(buf, n, kNcclFloat32, peer, comm, st);
}
int nccl_allreduce_sum_f64(double* buf, size_t n, void* comm, cudaStream_t st) {
  return g_api.AllReduce(buf, buf, n, kNcclFloat64, kNcclSum, comm, st);
}
int nccl_bcast_f32(float* buf, size_t n, int root, void* comm, cudaStream_t st) {
  return g_api.Broadcast(buf, buf, n, kNcclFloat32, root, comm, st);
}

}  // namespace lfsr
