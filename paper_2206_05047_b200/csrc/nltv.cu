// nltv.cu — the NLTV half of the wz-step as an HBM-streaming kernel (k_wz_nltv).
//
// Per own HR pixel z and offset d of the 5x5 window (A9), the z/w steps of the NLTV rows of F
// (Alg.1 lines 5-8, clamp form A5/A6, A10):
//     g_d(z)   = W_d(z) (x(z) - x(z+d))  if z+d in Omega, else 0,   W_d = w_d m
//     w_S+     = clamp(g_d + w_S, +-1/theta),  f = 2 w_S+ - w_S
//     v(z)    += (theta/2) [W_d(z) f_d(z) - 1{z-d in Omega} W_d(z-d) f_d(z-d)]
// with the backward neighbour's f_d(z-d) recomputed from its old dual (gather form: no atomics),
// and the J term sum |g| and the primal residual |w+ - w|^2.  r = -v (A3) is updated in place
// (the tile kernel has already accumulated the data part of -v into r, stream order).
//
// The w_S planes are the largest stream of the method (48 B per HR pixel per iteration, SURVEY
// §8a a5); the tile kernel's in-CTA version read them a scalar per lane per offset between its
// view passes (26 % of HBM peak at M2).  Here a CTA owns 128 x 8 pixels and streams the 24
// planes through shared memory with cp.async, three planes in flight (tile + the 2-pixel halo the
// backward neighbours need, 16-byte chunks, zero-filled outside the image): every w_S element is
// read from HBM once and written once, coalesced; a warp owns a row, a lane the pixels lane + 32 j
// (j < 4), and x and m come from a shared tile with the window halo (conflict-free reads).
#include "internal.h"

namespace lfsr {

namespace {
constexpr int kRad = 2;                 // 5x5 window
#ifndef LFSR_NLTV_TH
#define LFSR_NLTV_TH 8
#endif
#ifndef LFSR_NLTV_NBUF
#define LFSR_NLTV_NBUF 4
#endif
#ifndef LFSR_NLTV_MINB
#define LFSR_NLTV_MINB 4
#endif
constexpr int kTW = 128, kTH = LFSR_NLTV_TH;   // own pixels per CTA: 8 warps x kTH/8 rows x (32 lanes x 4 pixels)
constexpr int kRW = kTH / 8;                   // rows per warp
constexpr int kSW = kTW + 2 * kRad + 1, kSH = kTH + 2 * kRad;   // x / m tiles with halo (+1: odd pitch)
constexpr int kPW = kTW + 8;            // staged w_S plane rows: X0 - 4 .. X0 + kTW + 4 (16-byte chunks)
constexpr int kPH = kTH + 2 * kRad;
constexpr int kNBUF = LFSR_NLTV_NBUF;   // planes in flight (cp.async groups)
constexpr int kChunks = kPH * (kPW / 4);
}  // namespace

__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// stage plane d of w_S^{n-1} (tile + 2-row/col halo; chunks outside the image or the pitch read as 0)
__device__ __forceinline__ void stage_plane(float* buf, const float* plane_base, int Y0, int X0, int H, int ps, int tid) {
  for (int c = tid; c < kChunks; c += 256) {
    const int r = c / (kPW / 4), q = c - r * (kPW / 4);
    const int gy = Y0 - kRad + r, gx = X0 - 4 + 4 * q;
    const bool ok = gy >= 0 && gy < H && gx >= 0 && gx + 4 <= ps;
    const float* src = plane_base + (ok ? (size_t)gy * ps + gx : 0);
    cp_async16(buf + r * kPW + 4 * q, src, ok);
  }
}

__global__ void __launch_bounds__(256, LFSR_NLTV_MINB) k_wz_nltv(const Geom G, const float* __restrict__ x, const float* __restrict__ m,
                                                    const float* wS0, float* wS1_, float* r, Control* ctl, int row0,
                                                    int row1) {
  extern __shared__ __align__(16) float dyn[];
  float (*sx)[kSW] = reinterpret_cast<float (*)[kSW]>(dyn);                    // [kSH][kSW]
  float (*sm)[kSW] = reinterpret_cast<float (*)[kSW]>(dyn + kSH * kSW);        // [kSH][kSW]
  float* swb = dyn + ((2 * kSH * kSW + 3) & ~3);                               // [kNBUF][kPH * kPW]
  __shared__ double red[8 * 2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int X0 = blockIdx.x * kTW, Y0 = row0 + blockIdx.y * kTH;
  const int H = G.H, W = G.W, ps = G.ps;
  // this iteration's w_S buffers (Alg.1: read w^{n-1}, write w^n; ping-pong by the iteration parity)
  const int rd = ctl->iter & 1;
  const float* wSr = rd ? wS1_ : wS0;
  float* wSw = rd ? const_cast<float*>(wS0) : wS1_;
  const size_t plane = (size_t)H * ps;
  // planes 0 .. kNBUF - 2 in flight while x and m are staged
#pragma unroll
  for (int b = 0; b + 1 < kNBUF; ++b) {
    stage_plane(swb + b * kPH * kPW, wSr + (size_t)b * plane, Y0, X0, H, ps, tid);
    cp_commit();
  }
  // x and m with the window halo (m = 0, x replicated outside: those terms are masked anyway)
  for (int e = tid; e < kSH * kSW; e += 256) {
    const int ly = e / kSW, lx = e - ly * kSW;
    const int gy = Y0 - kRad + ly, gx = X0 - kRad + lx;
    const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
    const size_t gi = (size_t)min(max(gy, 0), H - 1) * ps + min(max(gx, 0), W - 1);
    sx[ly][lx] = __ldg(x + gi);
    sm[ly][lx] = in ? __ldg(m + gi) : 0.f;
  }
  const float ith = G.inv_theta;
  const bool cols_in = X0 >= kRad && X0 + kTW <= W - kRad;
  float acc[kRW][4];
#pragma unroll
  for (int t = 0; t < kRW; ++t)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[t][j] = 0.f;
  float freg = 0.f, fres = 0.f;
#pragma unroll
  for (int dy = -kRad; dy <= kRad; ++dy) {
#pragma unroll
    for (int dx = -kRad; dx <= kRad; ++dx) {
      if (dy == 0 && dx == 0) continue;
      const int lin = (dy + kRad) * (2 * kRad + 1) + (dx + kRad);
      const int d = lin > (2 * kRad + 1) * kRad + kRad ? lin - 1 : lin;   // A9 order, centre skipped
      cp_wait<kNBUF - 2>();  // plane d has landed (later planes may still be in flight)
      __syncthreads();       // ... for every thread; plane d - 1's buffer is free
      if (d + kNBUF - 1 < 24)
        stage_plane(swb + ((d + kNBUF - 1) % kNBUF) * kPH * kPW, wSr + (size_t)(d + kNBUF - 1) * plane, Y0, X0, H,
                    ps, tid);
      cp_commit();           // (an empty group at the tail keeps the wait count uniform)
      const float* pl = swb + (d % kNBUF) * kPH * kPW;
      const float wd = G.wd[d];
#pragma unroll
      for (int t = 0; t < kRW; ++t) {
        const int Y = Y0 + warp + 8 * t, ly = warp + 8 * t + kRad;
        if (Y >= row1) continue;
        const bool inner = cols_in && Y >= kRad && Y < H - kRad;
        float* wp = wSw + (size_t)d * plane + (size_t)Y * ps + X0 + lane;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int xg = X0 + lane + 32 * j, lx = lane + 32 * j + kRad, px = lane + 32 * j + 4;
          const bool fin = inner || (Y + dy >= 0 && Y + dy < H && xg + dx >= 0 && xg + dx < W);
          const bool bin = inner || (Y - dy >= 0 && Y - dy < H && xg - dx >= 0 && xg - dx < W);
          const float o = pl[ly * kPW + px];
          const float nb = pl[(ly - dy) * kPW + px - dx];    // z - d
          const float xz = sx[ly][lx], mz = sm[ly][lx];
          const float wz = wd * mz;
          const float g = fin ? wz * (xz - sx[ly + dy][lx + dx]) : 0.f;   // W_d (.) Delta_d x
          const float w = fminf(fmaxf(g + o, -ith), ith);
          freg += fabsf(g);
          fres = fmaf(w - o, w - o, fres);
          if (fin) acc[t][j] = fmaf(wz, 2.f * w - o, acc[t][j]);
          if (bin) {
            const float wb = wd * sm[ly - dy][lx - dx];
            const float wnb = fminf(fmaxf(fmaf(wb, sx[ly - dy][lx - dx] - xz, nb), -ith), ith);
            acc[t][j] = fmaf(-wb, 2.f * wnb - nb, acc[t][j]);
          }
          if (xg < W) wp[32 * j] = w;
        }
      }
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int t = 0; t < kRW; ++t) {
    const int Y = Y0 + warp + 8 * t;
    if (Y >= row1) continue;
    float* rp = r + (size_t)Y * ps + X0 + lane;
#pragma unroll
    for (int j = 0; j < 4; ++j)   // r = -v (A3): subtract (theta/2) times the NLTV part
      if (X0 + lane + 32 * j < W) rp[32 * j] -= G.cS * acc[t][j];
  }
  // J's regulariser term and the primal residual (fp64 block partials, a7)
  double a = (double)freg, b = (double)fres;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    red[warp * 2] = a;
    red[warp * 2 + 1] = b;
  }
  __syncthreads();
  if (tid == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < 8; ++w) {
      s0 += red[w * 2];
      s1 += red[w * 2 + 1];
    }
    if (s0 != 0.0) atomicAdd(&ctl->cur[S_REG], s0);
    if (s1 != 0.0) atomicAdd(&ctl->cur[S_RES2], s1);
  }
}

cudaError_t launch_wz_nltv(const Geom& G, const float* x, const float* m, float* wS0, float* wS1, float* r,
                           Control* ctl, int row0, int row1, cudaStream_t st) {
  if (row1 <= row0) return cudaSuccess;
  constexpr size_t smem = (((size_t)2 * kSH * kSW + 3) & ~(size_t)3) * 4 + (size_t)kNBUF * kPH * kPW * 4;
  const cudaError_t e = cudaFuncSetAttribute(k_wz_nltv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;   // (per device; a host-side call, legal during graph capture)
  dim3 grid((G.W + kTW - 1) / kTW, (row1 - row0 + kTH - 1) / kTH);
  k_wz_nltv<<<grid, 256, smem, st>>>(G, x, m, wS0, wS1, r, ctl, row0, row1);
  return cudaGetLastError();
}

}  // namespace lfsr
