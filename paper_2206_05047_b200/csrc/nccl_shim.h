// nccl_shim.h — the NCCL calls of the strip decomposition, resolved with dlopen.
#pragma once
#include <cstddef>
#include <cstring>
#include <string>
#include <cuda_runtime.h>

namespace lfsr {

struct NcclUniqueId {
  char internal[128];
};
// ncclDataType_t / ncclRedOp_t values of the NCCL 2.x ABI
constexpr int kNcclFloat32 = 7;
constexpr int kNcclFloat64 = 8;
constexpr int kNcclSum = 0;

bool nccl_available(std::string* why);
const char* nccl_error(int code);
int nccl_comm_init(void** comm, int nranks, const void* uid, int rank);
int nccl_comm_destroy(void* comm);
int nccl_comm_abort(void* comm);
int nccl_group_start();
int nccl_group_end();
int nccl_send_f32(const float* buf, size_t n, int peer, void* comm, cudaStream_t st);
int nccl_recv_f32(float* buf, size_t n, int peer, void* comm, cudaStream_t st);
int nccl_allreduce_sum_f64(double* buf, size_t n, void* comm, cudaStream_t st);
int nccl_bcast_f32(float* buf, size_t n, int root, void* comm, cudaStream_t st);

}  // namespace lfsr
