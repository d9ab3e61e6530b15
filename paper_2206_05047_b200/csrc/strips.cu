// strips.cu — kernels of the HR row-strip decomposition (DESIGN.md §10,
// SURVEY §8e): folding the accumulated halo ring of a strip into the
// neighbour's own rows, and the in-process scalar all-reduce used by the
// "virtual ranks" mode (all strips of one problem on one device; the NCCL
// mode uses ncclSend/ncclRecv/ncclAllReduce instead).
#include "internal.h"

namespace lfsr {

// dst[i] += src[i]; src[i] = 0 (src: the ring rows of one strip, dst: the same
// rows, owned by the neighbour).  n is a multiple of 4 (whole pitched rows).
__global__ void k_fold_rows(float* __restrict__ dst, float* __restrict__ src, size_t n4, int zero_src) {
  float4* d = reinterpret_cast<float4*>(dst);
  float4* s = reinterpret_cast<float4*>(src);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 a = d[i], b = s[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    d[i] = a;
    if (zero_src) s[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Sum cur[slot0 .. slot0+count) over the strips' control blocks and write the
// total back to every strip (the in-process stand-in for ncclAllReduce).
__global__ void k_allreduce_local(Control* const* ctls, int nparts, int slot0, int count) {
  const int i = threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += ctls[p]->cur[slot0 + i];
  for (int p = 0; p < nparts; ++p) ctls[p]->cur[slot0 + i] = s;
}

cudaError_t launch_fold_rows(float* dst, float* src, size_t n, int zero_src, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  size_t n4 = n / 4;
  int blocks = (int)((n4 + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  k_fold_rows<<<blocks, 256, 0, st>>>(dst, src, n4, zero_src);
  return cudaGetLastError();
}

cudaError_t launch_allreduce_local(Control* const* ctls, int nparts, int slot0, int count, cudaStream_t st) {
  k_allreduce_local<<<1, 32 * ((count + 31) / 32), 0, st>>>(ctls, nparts, slot0, count);
  return cudaGetLastError();
}

}  // namespace lfsr
