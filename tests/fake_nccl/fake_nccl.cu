// fake_nccl.cu — TEST DOUBLE of the NCCL subset liblfsr's strip mode calls (nccl_shim.cu):
// ncclCommInitRank / Destroy / Abort, ncclSend / ncclRecv, ncclAllReduce (f64 sum),
// ncclBroadcast (f32), ncclGroupStart / End, ncclGetUniqueId, ncclGetErrorString.
//
// It lets the library's own NCCL code path (capi.cu: xfill / xfold / xallreduce inside the
// captured CUDA graph) run with several PROCESSES on ONE GPU, which is all this project's GPU
// boxes have: every rank exports a device "region" with cudaIpcGetMemHandle, the ranks meet
// through files under /tmp named after the unique id, and each call is a single-CTA kernel on
// the caller's stream (so it is captured into graphs like real NCCL kernels):
//   send:  wait for a free mailbox slot in the peer's region (ack counter), copy, fence,
//          publish the message count in the peer's flag word;
//   recv:  wait for the peer's flag, copy out of my mailbox (L1 bypassed), fence, ack;
//   allreduce: write my values into every rank's box slot, publish, wait for all ranks,
//          sum in rank order (identical bits on every rank, like NCCL's tree/ring results
//          are identical across ranks).
// Counters live in device memory and advance inside the kernels, so a graph replay continues
// the message sequence.  Not a product path: tests set LFSR_NCCL_LIB to this library.
#include <cuda_runtime.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <sys/stat.h>
#include <thread>
#include <vector>

namespace {

constexpr int kMaxRanks = 8;
constexpr int kSlots = 8;
constexpr size_t kSlotBytes = 1 << 20;
constexpr int kArSlots = 4;
constexpr int kArMax = 64;   // doubles per all-reduce

struct Header {
  unsigned long long send_seq[kMaxRanks];   // mine: messages I posted to peer j
  unsigned long long recv_seq[kMaxRanks];   // mine: messages I consumed from peer j
  unsigned long long flag[kMaxRanks];       // written by peer j: messages j posted to me
  unsigned long long ack[kMaxRanks];        // written by peer j: my messages j consumed
  unsigned long long ar_seq;                // mine
  unsigned long long ar_flag[kMaxRanks];    // written by rank j: its all-reduce count
  double ar_box[kArSlots][kMaxRanks][kArMax];
};

size_t region_bytes(int n) {
  return ((sizeof(Header) + 255) & ~(size_t)255) + (size_t)n * kSlots * kSlotBytes;
}

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ char* mailbox(char* region, int src, int slot) {
  return region + ((sizeof(Header) + 255) & ~(size_t)255) + ((size_t)src * kSlots + slot) * kSlotBytes;
}

__device__ void copy_bytes(char* dst, const char* src, size_t n) {
  if ((((uintptr_t)dst | (uintptr_t)src | n) & 15) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (size_t i = threadIdx.x; i < n / 16; i += blockDim.x) d4[i] = __ldcg(s4 + i);
  } else {
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];   // plain: bytes in L2
  }
}

__global__ void k_send(const char* src, size_t n, char* mine, char* peer_region, int me, int peer) {
  Header* H = reinterpret_cast<Header*>(mine);
  Header* P = reinterpret_cast<Header*>(peer_region);
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) {
    s = H->send_seq[peer];
    while (ld_acq(&H->ack[peer]) + kSlots <= s) __nanosleep(200);   // the peer freed slot s % kSlots
  }
  __syncthreads();
  copy_bytes(mailbox(peer_region, me, (int)(s % kSlots)), src, n);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    st_rel(&P->flag[me], s + 1);
    H->send_seq[peer] = s + 1;
  }
}

__global__ void k_recv(char* dst, size_t n, char* mine, char* peer_region, int me, int peer) {
  Header* H = reinterpret_cast<Header*>(mine);
  Header* P = reinterpret_cast<Header*>(peer_region);
  __shared__ unsigned long long r;
  if (threadIdx.x == 0) {
    r = H->recv_seq[peer];
    while (ld_acq(&H->flag[peer]) <= r) __nanosleep(200);
  }
  __syncthreads();
  copy_bytes(dst, mailbox(mine, peer, (int)(r % kSlots)), n);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    st_rel(&P->ack[me], r + 1);
    H->recv_seq[peer] = r + 1;
  }
}

struct Peers {
  char* p[kMaxRanks];
};

__global__ void k_allreduce(const double* in, double* out, int count, Peers regions, int me, int n) {
  Header* H = reinterpret_cast<Header*>(regions.p[me]);
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = H->ar_seq + 1;
  __syncthreads();
  const int slot = (int)(s % kArSlots);
  for (int j = 0; j < n; ++j) {
    Header* R = reinterpret_cast<Header*>(regions.p[j]);
    for (int i = threadIdx.x; i < count; i += blockDim.x) R->ar_box[slot][me][i] = in[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < n; ++j) st_rel(&reinterpret_cast<Header*>(regions.p[j])->ar_flag[me], s);
    for (int j = 0; j < n; ++j)
      while (ld_acq(&H->ar_flag[j]) < s) __nanosleep(200);
    H->ar_seq = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc += __ldcg(&H->ar_box[slot][j][i]);   // rank order: same bits everywhere
    out[i] = acc;
  }
}

struct Comm {
  int rank = 0, n = 0;
  char* mine = nullptr;
  Peers regions{};
  std::string dir;
};

std::string id_dir(const char* id) {
  char hex[33];
  for (int i = 0; i < 16; ++i) snprintf(hex + 2 * i, 3, "%02x", (unsigned char)id[i]);
  return std::string("/tmp/lfsr_fake_nccl_") + hex;
}

}  // namespace

extern "C" {

struct ncclUniqueIdFake {
  char internal[128];
};

int ncclGetUniqueId(ncclUniqueIdFake* id) {
  srand((unsigned)time(nullptr) ^ (unsigned)getpid());
  for (int i = 0; i < 128; ++i) id->internal[i] = (char)(rand() & 0xff);
  return 0;
}

int ncclCommInitRank(void** comm, int nranks, ncclUniqueIdFake id, int rank) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return 4;   // ncclInvalidArgument
  Comm* c = new Comm;
  c->rank = rank;
  c->n = nranks;
  c->dir = id_dir(id.internal);
  mkdir(c->dir.c_str(), 0700);
  const size_t bytes = region_bytes(nranks);
  if (cudaMalloc(&c->mine, bytes) != cudaSuccess || cudaMemset(c->mine, 0, bytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return 1;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, c->mine) != cudaSuccess) return 1;
  const std::string f = c->dir + "/rank" + std::to_string(rank), tmp = f + ".tmp";
  FILE* fp = fopen(tmp.c_str(), "wb");
  if (!fp) return 2;
  fwrite(&h, sizeof h, 1, fp);
  fclose(fp);
  rename(tmp.c_str(), f.c_str());
  c->regions.p[rank] = c->mine;
  const auto t0 = std::chrono::steady_clock::now();
  for (int j = 0; j < nranks; ++j) {
    if (j == rank) continue;
    const std::string g = c->dir + "/rank" + std::to_string(j);
    FILE* q = nullptr;
    while (!(q = fopen(g.c_str(), "rb"))) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) return 2;   // ncclSystemError
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
    cudaIpcMemHandle_t hj;
    const size_t got = fread(&hj, sizeof hj, 1, q);
    fclose(q);
    if (got != 1) return 2;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hj, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return 1;
    c->regions.p[j] = (char*)p;
  }
  *comm = c;
  return 0;
}

static int destroy(void* comm) {
  Comm* c = (Comm*)comm;
  if (!c) return 0;
  cudaDeviceSynchronize();
  for (int j = 0; j < c->n; ++j)
    if (j != c->rank && c->regions.p[j]) cudaIpcCloseMemHandle(c->regions.p[j]);
  cudaFree(c->mine);
  remove((c->dir + "/rank" + std::to_string(c->rank)).c_str());
  rmdir(c->dir.c_str());   // the last rank out removes the directory
  delete c;
  return 0;
}
int ncclCommDestroy(void* comm) { return destroy(comm); }
int ncclCommAbort(void* comm) { return destroy(comm); }

static size_t dsize(int dtype) { return dtype == 8 ? 8 : 4; }   // ncclFloat64 = 8, ncclFloat32 = 7

int ncclSend(const void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t st) {
  Comm* c = (Comm*)comm;
  const size_t n = count * dsize(dtype);
  for (size_t off = 0; off < n || (n == 0 && off == 0); off += kSlotBytes) {
    const size_t b = n - off < kSlotBytes ? n - off : kSlotBytes;
    k_send<<<1, 1024, 0, st>>>((const char*)buf + off, b, c->mine, c->regions.p[peer], c->rank, peer);
    if (n == 0) break;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int ncclRecv(void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t st) {
  Comm* c = (Comm*)comm;
  const size_t n = count * dsize(dtype);
  for (size_t off = 0; off < n || (n == 0 && off == 0); off += kSlotBytes) {
    const size_t b = n - off < kSlotBytes ? n - off : kSlotBytes;
    k_recv<<<1, 1024, 0, st>>>((char*)buf + off, b, c->mine, c->regions.p[peer], c->rank, peer);
    if (n == 0) break;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int ncclAllReduce(const void* in, void* out, size_t count, int dtype, int op, void* comm, cudaStream_t st) {
  Comm* c = (Comm*)comm;
  if (dtype != 8 || op != 0 || count > (size_t)kArMax) return 4;   // only what liblfsr uses: f64 sum
  k_allreduce<<<1, 64, 0, st>>>((const double*)in, (double*)out, (int)count, c->regions, c->rank, c->n);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int ncclBroadcast(const void* in, void* out, size_t count, int dtype, int root, void* comm, cudaStream_t st) {
  Comm* c = (Comm*)comm;
  if (c->rank == root) {
    if (in != out) cudaMemcpyAsync(out, in, count * dsize(dtype), cudaMemcpyDeviceToDevice, st);
    for (int j = 0; j < c->n; ++j)
      if (j != root) ncclSend(in, count, dtype, j, comm, st);
    return 0;
  }
  return ncclRecv(out, count, dtype, root, comm, st);
}

int ncclGroupStart() { return 0; }
int ncclGroupEnd() { return 0; }

const char* ncclGetErrorString(int code) {
  switch (code) {
    case 0: return "success (fake NCCL)";
    case 1: return "CUDA error (fake NCCL)";
    case 2: return "system error (fake NCCL: rendezvous)";
    case 4: return "invalid argument (fake NCCL)";
    default: return "error (fake NCCL)";
  }
}

}  // extern "C"
