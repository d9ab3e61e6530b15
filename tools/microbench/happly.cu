// Microbenchmark: an assembled normal matrix applied as a per-pixel window stencil,
// q(c) = sum_o Hw[o][c] p(c + o), o in [-WY, WY] x [-WX, WX], Hw plane-major.
// Design input for the CG normal-operator path: achievable HBM
// streaming rate for the window sizes the light-field geometries need.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int BY = 8, BX = 128;

template <int WY, int WX>
__global__ void __launch_bounds__(256) k_happly(const float* __restrict__ Hw, const float* __restrict__ p,
                                                float* __restrict__ q, int H, int W, int ps) {
  constexpr int PX = BX + 2 * 12;            // halo columns (aligned loads cover WX <= 12)
  constexpr int PY = BY + 2 * WY;
  __shared__ __align__(16) float ps_[PY][PX];
  const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
  for (int e = threadIdx.x; e < PY * PX; e += 256) {
    const int r = e / PX, c = e - r * PX;
    const int gy = y0 - WY + r, gx = x0 - 12 + c;
    ps_[r][c] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? p[(size_t)gy * ps + gx] : 0.f;
  }
  __syncthreads();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int y = y0 + ty, x = x0 + 4 * tx;
  if (y >= H || x >= W) return;
  const size_t plane = (size_t)H * ps;
  const float4* Hp = reinterpret_cast<const float4*>(Hw + (size_t)y * ps + x);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int dy = -WY; dy <= WY; ++dy) {
    float pr[4 + 24];
    const float4* row = reinterpret_cast<const float4*>(&ps_[ty + WY + dy][4 * tx]);
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      const float4 v = row[j];
      pr[4 * j] = v.x; pr[4 * j + 1] = v.y; pr[4 * j + 2] = v.z; pr[4 * j + 3] = v.w;
    }
    const float4* hrow = Hp + (size_t)((dy + WY) * (2 * WX + 1)) * (plane / 4);
    float4 h[2 * WX + 1];
#pragma unroll
    for (int dx = 0; dx <= 2 * WX; ++dx) h[dx] = __ldcs(hrow + (size_t)dx * (plane / 4));
#pragma unroll
    for (int dx = 0; dx <= 2 * WX; ++dx) {
      const int j = 12 - WX + dx;
      acc.x = fmaf(h[dx].x, pr[j], acc.x);
      acc.y = fmaf(h[dx].y, pr[j + 1], acc.y);
      acc.z = fmaf(h[dx].z, pr[j + 2], acc.z);
      acc.w = fmaf(h[dx].w, pr[j + 3], acc.w);
    }
  }
  *reinterpret_cast<float4*>(q + (size_t)y * ps + x) = acc;
}

template <int WY, int WX>
int run(int Hh, int Ww) {
  const int ps = (Ww + 127) / 128 * 128;
  const size_t plane = (size_t)Hh * ps, npl = (size_t)(2 * WY + 1) * (2 * WX + 1);
  float *Hw, *p, *q;
  CK(cudaMalloc(&Hw, plane * npl * 4));
  CK(cudaMalloc(&p, plane * 4));
  CK(cudaMalloc(&q, plane * 4));
  CK(cudaMemset(Hw, 0, plane * npl * 4));
  CK(cudaMemset(p, 0, plane * 4));
  dim3 grid((Ww + BX - 1) / BX, (Hh + BY - 1) / BY);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k_happly<WY, WX><<<grid, 256>>>(Hw, p, q, Hh, Ww, ps);
  const int N = 20;
  cudaEventRecord(a);
  for (int i = 0; i < N; ++i) k_happly<WY, WX><<<grid, 256>>>(Hw, p, q, Hh, Ww, ps);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= N;
  const double bytes = (double)plane * npl * 4 + 2.0 * plane * 4;
  printf("H=%d W=%d window %dx%d (%zu planes): %.1f us, %.0f MB, %.2f TB/s\n", Hh, Ww, 2 * WY + 1, 2 * WX + 1,
         npl, ms * 1e3, bytes / 1e6, bytes / (ms * 1e-3) / 1e12);
  cudaFree(Hw); cudaFree(p); cudaFree(q);
  return 0;
}

int main() {
  run<5, 5>(512, 512);
  run<6, 6>(512, 512);
  run<9, 9>(512, 512);
  run<8, 8>(512, 512);
  run<8, 8>(2048, 2048);
  run<7, 7>(2048, 2048);
  return 0;
}
