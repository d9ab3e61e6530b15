// Microbenchmark: throughput of the candidate scatter/gather primitives for
// the exact bilinear warp adjoint on sm_100a (design input).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
#define NT 256
template<int MODE>
__global__ void __launch_bounds__(NT) kbench(float* gout, float* gacc, int seed) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += NT) s[i] = 0.f;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float v = 1.0f + lane * 1e-3f;
  float acc = 0.f;
  unsigned st = seed * 747796405u + threadIdx.x;
  #pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    st = st * 1664525u + 1013904223u;
    int off = (st >> 28);                 // 0..15 "shift"
    int row = (w * 7 + i) & 63;
    int col = lane + off;                 // distinct within warp
    int a = row * 80 + col;
    if (MODE == 0) {          // float atomicAdd in smem (CAS spin)
      atomicAdd(&s[a], v);
    } else if (MODE == 1) {   // int32 ATOMS.ADD
      atomicAdd((int*)&s[a], (int)st);
    } else if (MODE == 2) {   // warp-private RMW (LDS+FADD+STS)
      int pa = (w * 1024) + ((i & 7) * 80 + col) % 1024;
      s[pa] += v; __syncwarp();
    } else if (MODE == 3) {   // 4 scalar LDS (bilinear gather)
      acc += s[a] + s[a + 1] + s[a + 80] + s[a + 81];
    } else if (MODE == 4) {   // 1 LDS.128 gather
      float4 q = *reinterpret_cast<float4*>(&s[(a & ~3)]);
      acc += q.x + q.y + q.z + q.w;
    } else if (MODE == 5) {   // global RED.ADD.F32 to an L2-resident buffer
      atomicAdd(&gacc[(blockIdx.x * 4096 + a) & ((1 << 18) - 1)], v);
    } else if (MODE == 6) {   // 1 scalar LDS
      acc += s[a];
    } else if (MODE == 8) {   // one int64 ATOMS.ADD.64 per cell (hi/lo in one word)
      atomicAdd(reinterpret_cast<unsigned long long*>(s) + (a & 4095), (unsigned long long)(long long)(int)st);
    } else if (MODE == 9) {   // two int32 ATOMS.ADD per cell (the hi / lo accumulators, LO words apart)
      atomicAdd((int*)&s[a & 4095], (int)st);
      atomicAdd((int*)&s[4096 + (a & 4095)], (int)(st >> 7));
    } else if (MODE == 7) {   // 4 shuffles
      acc += __shfl_sync(0xffffffffu, v, (lane + off) & 31) + __shfl_down_sync(0xffffffffu, acc, 1)
           + __shfl_up_sync(0xffffffffu, v, 1) + __shfl_xor_sync(0xffffffffu, acc, 2);
      v += 1e-7f;
    }
  }
  __syncthreads();
  float r = acc;
  for (int i = threadIdx.x; i < 8192; i += NT) r += s[i];
  if (r == 12345.f) gout[blockIdx.x] = r;
}
int main() {
  float *gout, *gacc; cudaMalloc(&gout, 1 << 20); cudaMalloc(&gacc, 1 << 20);
  cudaMemset(gacc, 0, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"smem f32 atomicAdd (CAS)", "smem i32 ATOMS.ADD", "warp-private RMW",
                         "4x LDS.32 gather", "1x LDS.128 gather", "global REDG.F32", "1x LDS.32", "4x SHFL",
                         "smem i64 ATOMS.ADD.64", "2x smem i32 ATOMS (hi+lo)"};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 10; ++mode) {
    for (int occ : {4, 8}) {
      int grid = sms * occ;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        switch (mode) {
          case 0: kbench<0><<<grid, NT>>>(gout, gacc, rep); break;
          case 1: kbench<1><<<grid, NT>>>(gout, gacc, rep); break;
          case 2: kbench<2><<<grid, NT>>>(gout, gacc, rep); break;
          case 3: kbench<3><<<grid, NT>>>(gout, gacc, rep); break;
          case 4: kbench<4><<<grid, NT>>>(gout, gacc, rep); break;
          case 5: kbench<5><<<grid, NT>>>(gout, gacc, rep); break;
          case 6: kbench<6><<<grid, NT>>>(gout, gacc, rep); break;
          case 7: kbench<7><<<grid, NT>>>(gout, gacc, rep); break;
          case 8: kbench<8><<<grid, NT>>>(gout, gacc, rep); break;
          case 9: kbench<9><<<grid, NT>>>(gout, gacc, rep); break;
        }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) {
          double warp_ops = (double)grid * (NT / 32) * ITERS;
          double per_sm_cyc = ms * 1e-3 * clk * 1e3 / (warp_ops / sms);
          printf("%-28s occ=%d  %.3f ms  %.2f cyc per warp-op per SM (clk %d MHz nominal)\n",
                 names[mode], occ, ms, per_sm_cyc, clk / 1000);
        }
      }
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
