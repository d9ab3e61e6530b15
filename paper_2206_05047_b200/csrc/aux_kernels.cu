// aux_kernels.cu — setup, CG update and test-operator kernels of liblfsr.
#include "internal.h"
#include <algorithm>
#include <cfloat>

namespace lfsr {

// ---------------------------------------------------------------------------
// Setup (once per solve).
// ---------------------------------------------------------------------------

// Bilinear sample of an LR image at continuous LR (row, col), clamped (reading A17).
__device__ __forceinline__ float bilin_lr(const float* img, int h, int w, int lps, float r, float c) {
  r = fminf(fmaxf(r, 0.f), (float)(h - 1));
  c = fminf(fmaxf(c, 0.f), (float)(w - 1));
  float fr = floorf(r), fc = floorf(c);
  int r0 = (int)fr, c0 = (int)fc;
  int r1 = min(r0 + 1, h - 1), c1 = min(c0 + 1, w - 1);
  float a = r - fr, b = c - fc;
  return (1.f - a) * ((1.f - b) * img[(size_t)r0 * lps + c0] + b * img[(size_t)r0 * lps + c1]) +
         a * ((1.f - b) * img[(size_t)r1 * lps + c0] + b * img[(size_t)r1 * lps + c1]);
}

// Static occlusion weight w_o (Eq. weight_occ; readings A16/A17):
//   b = min(0, forward-difference divergence of omega), p = mean over non-reference
//   views of |y_ref(z/zeta) - y_k((z - dtheta_k omega(z))/zeta)|.
__global__ void k_setup_wo(const Geom G, const Views V, const float* __restrict__ y,
                           const float* __restrict__ omega, float* __restrict__ wo) {
  int X = blockIdx.x * blockDim.x + threadIdx.x, Y = blockIdx.y;
  if (X >= G.W || Y >= G.H) return;
  const int ps = G.ps;
  float om = omega[(size_t)Y * ps + X];
  float dx = X + 1 < G.W ? omega[(size_t)Y * ps + X + 1] - om : 0.f;
  float dy = Y + 1 < G.H ? omega[(size_t)(Y + 1) * ps + X] - om : 0.f;
  float b = fminf(dx + dy, 0.f);
  const float iz = 1.f / (float)G.scale;
  const size_t lstride = (size_t)G.h * G.lps;
  float ref = bilin_lr(y + G.ref_view * lstride, G.h, G.w, G.lps, Y * iz, X * iz);
  float acc = 0.f;
  int cnt = 0;
  for (int k = 0; k < G.n_views; ++k) {
    if (k == G.ref_view) continue;
    float2 o = V.off[k];
    float v = bilin_lr(y + k * lstride, G.h, G.w, G.lps, ((float)Y - o.y * om) * iz, ((float)X - o.x * om) * iz);
    acc += fabsf(ref - v);
    ++cnt;
  }
  float p = cnt > 0 ? acc / (float)cnt : 0.f;
  wo[(size_t)Y * ps + X] = expf(-b * b * G.inv_2s1sq) * expf(-p * p * G.inv_2s2sq);
}

// Splat density D(z) = sum_k (W_k^T 1)(z): the total bilinear weight all views'
// exact adjoint warps deposit on cell z.  Its maximum bounds the fixed-point
// accumulators of the tile kernels.  Setup only.
__global__ void k_density(const Geom G, const Views V, const float* __restrict__ omega, float* __restrict__ D) {
  int X = blockIdx.x * blockDim.x + threadIdx.x, Y = blockIdx.y;
  if (X >= G.W || Y >= G.H) return;
  const int ps = G.ps;
  const size_t pv_stride = G.per_view ? (size_t)G.H * ps : 0;   // omega_k (A34)
  for (int k = 0; k < G.n_views; ++k) {
    const float om = omega[k * pv_stride + (size_t)Y * ps + X];
    const float2 o = V.off[k];
    const float sy = fminf(fmaxf((float)Y + o.y * om, 0.f), (float)(G.H - 1));
    const float sx = fminf(fmaxf((float)X + o.x * om, 0.f), (float)(G.W - 1));
    const float fy = floorf(sy), fx = floorf(sx);
    const int y0 = (int)fy, x0 = (int)fx;
    const int y1 = min(y0 + 1, G.H - 1), x1 = min(x0 + 1, G.W - 1);
    const float a = sy - fy, b = sx - fx;
    atomicAdd(&D[(size_t)y0 * ps + x0], (1.f - a) * (1.f - b));
    atomicAdd(&D[(size_t)y0 * ps + x1], (1.f - a) * b);
    atomicAdd(&D[(size_t)y1 * ps + x0], a * (1.f - b));
    atomicAdd(&D[(size_t)y1 * ps + x1], a * b);
  }
}

__device__ __forceinline__ float keys_cubic(float t) {  // Catmull-Rom, a = -0.5 (reading A15)
  const float a = -0.5f;
  t = fabsf(t);
  if (t <= 1.f) return ((a + 2.f) * t - (a + 3.f)) * t * t + 1.f;
  if (t < 2.f) return ((a * t - 5.f * a) * t + 8.f * a) * t - 4.f * a;
  return 0.f;
}

// x0 = bicubic up-sampling of the reference LR view at (Y/zeta, X/zeta) (A15).
__global__ void k_bicubic(const Geom G, const float* __restrict__ y, float* __restrict__ x) {
  int X = blockIdx.x * blockDim.x + threadIdx.x, Y = blockIdx.y;
  if (X >= G.W || Y >= G.H) return;
  const float* yr = y + (size_t)G.ref_view * G.h * G.lps;
  float fy = (float)Y / (float)G.scale, fx = (float)X / (float)G.scale;
  float iyf = floorf(fy), ixf = floorf(fx);
  int iy = (int)iyf, ix = (int)ixf;
  float ty = fy - iyf, tx = fx - ixf;
  float s = 0.f;
#pragma unroll
  for (int a = -1; a <= 2; ++a) {
    int rr = min(max(iy + a, 0), G.h - 1);
    float wy = keys_cubic(ty - (float)a);
    float row = 0.f;
#pragma unroll
    for (int b = -1; b <= 2; ++b) row += keys_cubic(tx - (float)b) * yr[(size_t)rr * G.lps + min(max(ix + b, 0), G.w - 1)];
    s += wy * row;
  }
  x[(size_t)Y * G.ps + X] = s;
}

// m = lambda_R w_o exp(-|grad x|^2/sigma_e) (A8, A17, A19).
__global__ void k_weights(const Geom G, const float* __restrict__ x, const float* __restrict__ wo,
                          float* __restrict__ m) {
  int X = blockIdx.x * blockDim.x + threadIdx.x, Y = blockIdx.y;
  if (X >= G.W || Y >= G.H) return;
  const int ps = G.ps;
  const float* row = x + (size_t)Y * ps;
  float gx = 0.5f * (row[min(X + 1, G.W - 1)] - row[max(X - 1, 0)]);
  float gy = 0.5f * (x[(size_t)min(Y + 1, G.H - 1) * ps + X] - x[(size_t)max(Y - 1, 0) * ps + X]);
  m[(size_t)Y * ps + X] = G.lambda_reg * wo[(size_t)Y * ps + X] * expf(-(gx * gx + gy * gy) * G.inv_sigma_e);
}

// max |v| over an [H][ps] array (non-negative floats order like their bit patterns).
// (n is a multiple of 4: pitched rows of 32 floats; float4 loads)
__global__ void k_absmax(const float* __restrict__ v, size_t n, unsigned* out) {
  // max over the bit patterns of |v| as unsigned integers: for non-negative floats the order of
  // the bits is the order of the values, and a NaN (exponent all ones, mantissa != 0) sorts above
  // +inf, so a single NaN makes the result NaN (fmaxf would drop it and let it through validation)
  unsigned mx = 0u;
  const float4* v4 = reinterpret_cast<const float4*>(v);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = __ldg(v4 + i);
    const unsigned b0 = __float_as_uint(a.x) & 0x7fffffffu, b1 = __float_as_uint(a.y) & 0x7fffffffu;
    const unsigned b2 = __float_as_uint(a.z) & 0x7fffffffu, b3 = __float_as_uint(a.w) & 0x7fffffffu;
    mx = max(mx, max(max(b0, b1), max(b2, b3)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// ---------------------------------------------------------------------------
// CG update (Alg.2 lines 8-9 and 11 with readings A1-A4):
//   alpha = pi_{k-1} / <p_k, q_k>; x += alpha p_k; r -= alpha q_k; pi_k = <r, r>.
// Also zeroes q (the next normal operator accumulates into it) and, at k = K,
// zeroes r for the next wz-step.  The last block to finish closes the step:
// it records CG bookkeeping and, at k = K, writes the iteration's stats record
// and resets the scalar slots (threadfence reduction pattern).
// ---------------------------------------------------------------------------
// Record of the finished ADMM iteration and reset of the scalar slots (run by one
// thread: the last block of the final CG update, or k_close in the strip mode).
__device__ void close_iteration(const Geom& G, Control* ctl) {
  volatile double* cur = ctl->cur;
  const int cgit = (int)cur[S_CGIT];
  const double J = (double)G.lambda1 * cur[S_L1] + (double)G.lambda2 * cur[S_L2] + cur[S_REG];
  const double pil = cur[S_PI + cgit];
  double* rec = ctl->ring + (size_t)(ctl->iter % ctl->cap) * T_COUNT;
  rec[T_ITER] = (double)(ctl->iter + 1);
  rec[T_CGIT] = (double)cgit;
  rec[T_BREAK] = cur[S_BREAK];
  rec[T_NF] = (cur[S_NF] > 0.0 || !isfinite(J) || !isfinite(pil)) ? 1.0 : 0.0;
  rec[T_J] = J;
  rec[T_L1] = cur[S_L1];
  rec[T_L2] = cur[S_L2];
  rec[T_REG] = cur[S_REG];
  rec[T_RES] = sqrt(cur[S_RES2]);
  rec[T_PI0] = cur[S_PI];
  rec[T_PILAST] = pil;
  for (int s = 0; s < S_COUNT; ++s) cur[s] = 0.0;
  ctl->iter = ctl->iter + 1;
}

__global__ void k_close(const Geom G, Control* ctl) {
  if (threadIdx.x == 0 && blockIdx.x == 0) close_iteration(G, ctl);
}

// ---------------------------------------------------------------------------
// CG update (Alg.2 lines 8-9 and 11 with readings A1-A4) on the own rows
// [row0, row0 + nrows):
//   alpha = pi_{k-1} / <p_k, q_k>; x += alpha p_k; r -= alpha q_k; pi_k = <r, r>.
// Also zeroes q (the next normal operator accumulates into it) and, at k = K,
// zeroes r for the next wz-step.  The last block to finish closes the step:
// CG bookkeeping (steps taken, stop / breakdown flags) and, at k = K when
// close_here, the iteration's stats record (threadfence reduction pattern).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_cg_update(const Geom G, float* __restrict__ x, float* __restrict__ r,
                                                   const float* __restrict__ p, float* __restrict__ q,
                                                   Control* ctl, int k, int row0, int nrows, int close_here) {
  __shared__ double red[8 * 2];
  __shared__ bool am_last;
  const double pi_prev = ctl->cur[S_PI + k - 1];
  const double pq = ctl->cur[S_PQ + k];
  const bool stopped = ctl->cur[S_STOP] != 0.0;
  const bool active = !stopped && !(pi_prev < (double)G.cg_tol) && pi_prev != 0.0 && pq > 0.0;
  const float alpha = active ? (float)(pi_prev / pq) : 0.f;
  const bool last = (k == G.K);
  double pi_part = 0.0, nf_part = 0.0;
  const size_t off4 = (size_t)row0 * G.ps / 4;
  const size_t n4 = (size_t)nrows * G.ps / 4;
  float4* x4 = reinterpret_cast<float4*>(x) + off4;
  float4* r4 = reinterpret_cast<float4*>(r) + off4;
  const float4* p4 = reinterpret_cast<const float4*>(p) + off4;
  float4* q4 = reinterpret_cast<float4*>(q) + off4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 qv = q4[i];
    if (active) {
      float4 xv = x4[i], rv = r4[i], pv = p4[i];
      xv.x += alpha * pv.x; xv.y += alpha * pv.y; xv.z += alpha * pv.z; xv.w += alpha * pv.w;
      rv.x -= alpha * qv.x; rv.y -= alpha * qv.y; rv.z -= alpha * qv.z; rv.w -= alpha * qv.w;
      pi_part += (double)rv.x * rv.x + (double)rv.y * rv.y + (double)rv.z * rv.z + (double)rv.w * rv.w;
      x4[i] = xv;
      if (!last) r4[i] = rv;
      if (last) nf_part += (float)(!isfinite(xv.x)) + (!isfinite(xv.y)) + (!isfinite(xv.z)) + (!isfinite(xv.w));
    } else if (last) {
      float4 xv = x4[i];
      nf_part += (float)(!isfinite(xv.x)) + (!isfinite(xv.y)) + (!isfinite(xv.z)) + (!isfinite(xv.w));
    }
    q4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (last) r4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pi_part += __shfl_xor_sync(0xffffffffu, pi_part, o);
    nf_part += __shfl_xor_sync(0xffffffffu, nf_part, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[warp * 2] = pi_part; red[warp * 2 + 1] = nf_part; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) { a += red[w * 2]; b += red[w * 2 + 1]; }
    if (active && a != 0.0) atomicAdd(&ctl->cur[S_PI + k], a);
    if (b != 0.0) atomicAdd(&ctl->cur[S_NF], b);
    __threadfence();
    unsigned prev = atomicAdd(&ctl->done, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last || threadIdx.x != 0) return;
  // ---- last block: close CG step k ----
  __threadfence();
  volatile double* cur = ctl->cur;
  if (active) {
    cur[S_CGIT] = cur[S_CGIT] + 1.0;
  } else if (!stopped) {
    cur[S_STOP] = 1.0;
    if (!(pi_prev < (double)G.cg_tol) && pi_prev != 0.0 && !(pq > 0.0)) cur[S_BREAK] = 1.0;
  }
  if (last && close_here) close_iteration(G, ctl);
  __threadfence();
  ctl->done = 0u;
}

// ---------------------------------------------------------------------------
// CG update of the strip decomposition in the Chronopoulos-Gear form: step j
// (0-based) has w_j = M r_j, gamma_j = <r_j, r_j> and delta_j = <r_j, w_j> from the operator
// kernel -- reduced across the strips in ONE all-reduce -- and
//   beta = gamma_j / gamma_{j-1},  alpha = gamma_j / (delta_j - beta gamma_j / alpha_{j-1})
//   p = r + beta p,  s = w + beta s,  x += alpha p,  r -= alpha s
// (j = 0: beta = 0, alpha = gamma_0 / delta_0).  Equivalent to Alg.2 (readings A1-A4) in exact
// arithmetic: s_j = M p_j, delta_j - beta gamma_j / alpha_{j-1} = <p_j, M p_j>.  Stop rule A1 on
// gamma_j (= pi_j), breakdown A28 on the denominator.  The last step also forms pi_K = |r_K|^2
// (own rows; the caller all-reduces it) for the stats record.  w is zeroed for the next step.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_cgcg_update(const Geom G, float* __restrict__ x, float* __restrict__ r,
                                                     float* __restrict__ p, float* __restrict__ sv,
                                                     float* __restrict__ w, Control* ctl, int j, int row0,
                                                     int nrows) {
  __shared__ double red[8 * 2];
  __shared__ bool am_last;
  const double gam = ctl->cur[S_CG + 2 * j], del = ctl->cur[S_CG + 2 * j + 1];
  const bool stopped = ctl->cur[S_STOP] != 0.0;
  const bool small = gam < (double)G.cg_tol || gam == 0.0;
  double beta = 0.0, den = del;
  if (j > 0) {
    beta = gam / ctl->cur[S_PI + j - 1];
    den = del - beta * gam / ctl->cur[S_ALPHA];
  }
  const bool active = !stopped && !small && den > 0.0;
  const float alpha = active ? (float)(gam / den) : 0.f, betaf = (float)beta;
  const bool last = (j == G.K - 1);
  double pi_part = 0.0, nf_part = 0.0;
  const size_t off4 = (size_t)row0 * G.ps / 4, n4 = (size_t)nrows * G.ps / 4;
  float4* x4 = reinterpret_cast<float4*>(x) + off4;
  float4* r4 = reinterpret_cast<float4*>(r) + off4;
  float4* p4 = reinterpret_cast<float4*>(p) + off4;
  float4* s4 = reinterpret_cast<float4*>(sv) + off4;
  float4* w4 = reinterpret_cast<float4*>(w) + off4;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 wv = w4[i];
    if (active) {
      float4 rv = r4[i], pv = j > 0 ? p4[i] : z4, s = j > 0 ? s4[i] : z4, xv = x4[i];
      pv.x = rv.x + betaf * pv.x; pv.y = rv.y + betaf * pv.y; pv.z = rv.z + betaf * pv.z; pv.w = rv.w + betaf * pv.w;
      s.x = wv.x + betaf * s.x; s.y = wv.y + betaf * s.y; s.z = wv.z + betaf * s.z; s.w = wv.w + betaf * s.w;
      xv.x += alpha * pv.x; xv.y += alpha * pv.y; xv.z += alpha * pv.z; xv.w += alpha * pv.w;
      rv.x -= alpha * s.x; rv.y -= alpha * s.y; rv.z -= alpha * s.z; rv.w -= alpha * s.w;
      p4[i] = pv;
      s4[i] = s;
      x4[i] = xv;
      if (last) pi_part += (double)rv.x * rv.x + (double)rv.y * rv.y + (double)rv.z * rv.z + (double)rv.w * rv.w;
      if (last) nf_part += (float)(!isfinite(xv.x)) + (!isfinite(xv.y)) + (!isfinite(xv.z)) + (!isfinite(xv.w));
      r4[i] = last ? z4 : rv;   // the next wz-step accumulates r = -v into zeros
    } else if (last) {
      const float4 xv = x4[i];
      nf_part += (float)(!isfinite(xv.x)) + (!isfinite(xv.y)) + (!isfinite(xv.z)) + (!isfinite(xv.w));
      r4[i] = z4;
    }
    w4[i] = z4;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pi_part += __shfl_xor_sync(0xffffffffu, pi_part, o);
    nf_part += __shfl_xor_sync(0xffffffffu, nf_part, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[warp * 2] = pi_part; red[warp * 2 + 1] = nf_part; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < (int)(blockDim.x / 32); ++q) { a += red[q * 2]; b += red[q * 2 + 1]; }
    if (a != 0.0) atomicAdd(&ctl->cur[S_PI + j + 1], a);   // pi_K (last step only; all-reduced by the caller)
    if (b != 0.0) atomicAdd(&ctl->cur[S_NF], b);
    __threadfence();
    const unsigned prev = atomicAdd(&ctl->done, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last || threadIdx.x != 0) return;
  __threadfence();
  volatile double* cur = ctl->cur;
  if (!stopped) cur[S_PI + j] = gam;   // pi_j for the record (Alg.2 bookkeeping)
  if (active) {
    cur[S_CGIT] = cur[S_CGIT] + 1.0;
    cur[S_ALPHA] = gam / den;
  } else if (!stopped) {
    cur[S_STOP] = 1.0;
    if (!small && !(den > 0.0)) cur[S_BREAK] = 1.0;
  }
  __threadfence();
  ctl->done = 0u;
}

cudaError_t launch_cgcg_update(const Geom& G, float* x, float* r, float* p, float* s, float* w, Control* ctl, int j,
                               int row0, int nrows, int num_sms, cudaStream_t st) {
  const size_t n4 = (size_t)nrows * G.ps / 4;
  int blocks = (int)((n4 + 255) / 256);
  if (blocks > num_sms * 4) blocks = num_sms * 4;
  if (blocks < 1) blocks = 1;
  k_cgcg_update<<<blocks, 256, 0, st>>>(G, x, r, p, s, w, ctl, j, row0, nrows);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// gd / gd-ls (the baselines of the paper's solver comparison, P:L910-933;
// readings A30-A33).  One iteration = k_tile<GRAD> (cost terms of x and the
// subgradient g, accumulated into a zeroed buffer) [+ k_gd_gnorm and L trial
// launches of k_tile<J> for the line search] + k_gd_update.
// ---------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_sum_to(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) red[warp * NV + i] = v[i];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < NV; ++i) {
      double a = 0.0;
      for (int w = 0; w < (int)(blockDim.x / 32); ++w) a += red[w * NV + i];
      v[i] = a;
    }
}

// |g|^2 -> cur[S_GN] (the Armijo right-hand side needs it before the trials)
__global__ void __launch_bounds__(256) k_gd_gnorm(const Geom G, const float* __restrict__ g, Control* ctl) {
  __shared__ double red[8];
  const size_t n4 = (size_t)G.H * G.ps / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  double v[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = g4[i];
    v[0] += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
  }
  block_sum_to<1>(v, red);
  if (threadIdx.x == 0 && v[0] != 0.0) atomicAdd(&ctl->cur[S_GN], v[0]);
}

// Step choice (A32; every block computes the same from the fp64 sums), x -= eta g
// (fmaf: the rounding the J trial applied to the same x and g), non-finite count,
// and in the last block the iteration record: T_CGIT = trials evaluated, T_BREAK =
// ls_failed, T_RES = eta, T_PI0 = |g|^2 (lfsr_gd_stats).
__global__ void __launch_bounds__(256) k_gd_update(const Geom G, float* __restrict__ x, const float* __restrict__ g,
                                                   Control* ctl, const GdCfg cfg) {
  __shared__ double red[8 * 2];
  __shared__ bool am_last;
  const double* cur = ctl->cur;
  const double J0 = (double)G.lambda1 * cur[S_L1] + (double)G.lambda2 * cur[S_L2] + cur[S_REG];
  float eta = cfg.eta0;
  int evals = 0, failed = 0;
  if (cfg.ls) {
    eta = 0.f;
    failed = 1;
    evals = cfg.L;
    for (int t = 0; t < cfg.L; ++t) {
      const double et = ldexp((double)cfg.eta0, -t);
      const double* jt = cur + S_TJ + 3 * t;
      const double Jt = (double)G.lambda1 * jt[0] + (double)G.lambda2 * jt[1] + jt[2];
      if (Jt <= J0 - (double)cfg.armijo_c * et * cur[S_GN]) {
        eta = ldexpf(cfg.eta0, -t);
        evals = t + 1;
        failed = 0;
        break;
      }
    }
  }
  const float beta = -eta;
  const size_t n4 = (size_t)G.H * G.ps / 4;
  float4* x4 = reinterpret_cast<float4*>(x);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  double v[2] = {0.0, 0.0};   // |g|^2 (fixed step), non-finite count
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 gv = g4[i];
    float4 xv = x4[i];
    xv.x = fmaf(beta, gv.x, xv.x); xv.y = fmaf(beta, gv.y, xv.y);
    xv.z = fmaf(beta, gv.z, xv.z); xv.w = fmaf(beta, gv.w, xv.w);
    x4[i] = xv;
    if (!cfg.ls) v[0] += (double)gv.x * gv.x + (double)gv.y * gv.y + (double)gv.z * gv.z + (double)gv.w * gv.w;
    v[1] += (double)(!isfinite(xv.x)) + (!isfinite(xv.y)) + (!isfinite(xv.z)) + (!isfinite(xv.w));
  }
  block_sum_to<2>(v, red);
  if (threadIdx.x == 0) {
    if (v[0] != 0.0) atomicAdd(&ctl->cur[S_GN], v[0]);
    if (v[1] != 0.0) atomicAdd(&ctl->cur[S_NF], v[1]);
    __threadfence();
    const unsigned prev = atomicAdd(&ctl->done, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last || threadIdx.x != 0) return;
  __threadfence();
  volatile double* vc = ctl->cur;
  double* rec = ctl->ring + (size_t)(ctl->iter % ctl->cap) * T_COUNT;
  rec[T_ITER] = (double)(ctl->iter + 1);
  rec[T_CGIT] = (double)evals;
  rec[T_BREAK] = (double)failed;
  rec[T_NF] = (vc[S_NF] > 0.0 || !isfinite(J0)) ? 1.0 : 0.0;
  rec[T_J] = J0;
  rec[T_L1] = vc[S_L1];
  rec[T_L2] = vc[S_L2];
  rec[T_REG] = vc[S_REG];
  rec[T_RES] = (double)eta;
  rec[T_PI0] = vc[S_GN];
  rec[T_PILAST] = 0.0;
  for (int s = 0; s < S_COUNT; ++s) vc[s] = 0.0;
  ctl->iter = ctl->iter + 1;
  __threadfence();
  ctl->done = 0u;
}

// ---------------------------------------------------------------------------
// Paper-mode adjoint (reading A37): out(z) += sign * sum_k (W_k^* B^T D^T rho_k)(z),
// (W_k^* u)(z) = u(z - dtheta_k omega_0(z)) bilinear (replicate-clamped).  Gather form: one
// thread per HR pixel, no atomics.  u at the four bilinear points is
// sum_{i,j} g(Y - zeta i) g(X - zeta j) rho(i, j) (B^T D^T, zero padding), and the bilinear
// weights factor per axis, so the sample is sum_i Wy(i) sum_j Wx(j) rho(i, j) over the <= 4 x 4
// LR pixels whose blur reaches the 2 x 2 points.  Optionally adds <p, data part> to
// ctl->cur[slot] (the CG <p, Mp>; M is not symmetric in this mode).  Runs after the tile
// kernel that wrote rho and the NLTV part of `out`.
// ---------------------------------------------------------------------------
// One axis of the gather: the LR indices i_lo .. i_lo + 3 whose blur reaches the two bilinear
// points p0 = floor(s), p0 + 1, and their weights w[t] = (1 - a) g(p0 - zeta i) + a g(p0 + 1 - zeta i)
// (g = the blur taps, zero outside [-R, R]).  With phi = (R - p0) mod zeta, i_lo = (p0 - R + phi) /
// zeta and the tap offsets are 2R - phi - zeta t (+1), so the tap pairs come from a per-phase table
// tp[phi][t] (shared memory, built once per block).  At the clamped last sample a = 0.
__device__ __forceinline__ void paper_axis(float s, int scale, int R, const float2* tp, int& i_lo, float (&w)[4]) {
  const float fs = floorf(s);
  const int p0 = (int)fs;
  const float a = s - fs;
  const int phi = ((R - p0) % scale + scale) % scale;
  i_lo = (p0 - R + phi) / scale;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float2 g = tp[phi * 4 + t];
    w[t] = fmaf(a, g.y - g.x, g.x);
  }
}

// LR window of one 32 x 8 HR pixel block: every bilinear point z - dtheta_k omega_0(z) of the
// block lies within the block +- (SY, SX) (+1 for the second point), so the rho the block
// reads lies in LR rows [i_lo, i_lo + RH) and columns [j_lo, j_lo + RW) for every view.
struct GatherWin {
  int i_lo, j_lo, RH, RW;
};
__host__ __device__ inline int floor_div_pos(int a, int b) { return (a + 64 * b) / b - 64; }   // a >= -64 b
__host__ __device__ inline GatherWin gather_window(const Geom& G, int by0, int bx0) {
  GatherWin w;
  const int ylo = max(by0 - G.SY, 0), yhi = min(by0 + 7 + G.SY, G.H - 1) + 1;
  const int xlo = max(bx0 - G.SX, 0), xhi = min(bx0 + 31 + G.SX, G.W - 1) + 1;
  w.i_lo = floor_div_pos(ylo - G.R + G.scale - 1, G.scale);
  w.j_lo = floor_div_pos(xlo - G.R + G.scale - 1, G.scale);
  w.RH = floor_div_pos(yhi + G.R, G.scale) - w.i_lo + 1;
  w.RW = floor_div_pos(xhi + G.R, G.scale) - w.j_lo + 1;
  return w;
}
// shared-memory words per staged view (+3 rows / columns of slack: the 4 x 4 read window
// of a pixel may run past the block window where its weights are zero)
static inline int gather_stride(const Geom& G) {
  const int RH = (8 + 2 * G.SY + 1 + 2 * G.R) / G.scale + 2, RW = (32 + 2 * G.SX + 1 + 2 * G.R) / G.scale + 2;
  return (RH + 3) * (RW + 3);
}

__global__ void __launch_bounds__(256) k_paper_gather(const Geom G, const Views V, const float* __restrict__ rho,
                                                      const float* __restrict__ omega0, const float* __restrict__ p,
                                                      float* __restrict__ out, float sign, Control* ctl, int slot,
                                                      int cg_k, int row0, int nrows, int vchunk, int stride) {
  extern __shared__ float s_rho[];   // vchunk views x stride words
  __shared__ double red[8];
  __shared__ float2 s_tp[4 * 4];     // tap pairs per phase (paper_axis)
  if (cg_k >= 2 && ctl->cur[S_STOP] != 0.0) return;   // CG stopped (the tile kernel returned too)
  if (threadIdx.x < 4 * G.scale) {
    const int phi = threadIdx.x / 4, t = threadIdx.x % 4;
    const int d = 2 * G.R - phi - G.scale * t;
    s_tp[threadIdx.x] = make_float2((d >= 0 && d <= 2 * G.R) ? G.taps[d] : 0.f,
                                    (d + 1 >= 0 && d + 1 <= 2 * G.R) ? G.taps[d + 1] : 0.f);
  }
  const int bx0 = blockIdx.x * 32, by0 = row0 + blockIdx.y * 8;
  const int X = bx0 + (threadIdx.x & 31);
  const int Y = by0 + (threadIdx.x >> 5);
  const bool valid = X < G.W && Y < row0 + nrows && Y < G.H;
  const GatherWin gw = gather_window(G, by0, bx0);
  const int PWs = gw.RW + 3, PHs = gw.RH + 3;
  const int h = G.h, w = G.w, Z = G.scale, R = G.R;
  const size_t lstride = (size_t)h * G.lps;
  const size_t gi = (size_t)min(Y, G.H - 1) * G.ps + min(X, G.W - 1);
  const float om = omega0[gi];
  float acc = 0.f;
  for (int k0 = 0; k0 < G.n_views; k0 += vchunk) {
    const int nk = min(vchunk, G.n_views - k0);
    __syncthreads();   // the previous chunk's reads are done
    for (int e = threadIdx.x; e < nk * PHs * PWs; e += blockDim.x) {
      const int kk = e / (PHs * PWs), r = e - kk * (PHs * PWs);
      const int i = gw.i_lo + r / PWs, j = gw.j_lo + r % PWs;
      s_rho[kk * stride + r] =
          (i >= 0 && i < h && j >= 0 && j < w) ? __ldg(rho + (k0 + kk) * lstride + (size_t)i * G.lps + j) : 0.f;
    }
    __syncthreads();
    if (valid) {
      for (int kk = 0; kk < nk; ++kk) {
        const float2 o = V.off[k0 + kk];
        const float sy = fminf(fmaxf((float)Y - o.y * om, 0.f), (float)(G.H - 1));
        const float sx = fminf(fmaxf((float)X - o.x * om, 0.f), (float)(G.W - 1));
        int iy, ix;
        float wy[4], wx[4];
        paper_axis(sy, Z, R, s_tp, iy, wy);
        paper_axis(sx, Z, R, s_tp, ix, wx);
        const float* base = s_rho + kk * stride + (iy - gw.i_lo) * PWs + (ix - gw.j_lo);
        float v = 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float* row = base + t * PWs;
          float r = wx[0] * row[0];
          r = fmaf(wx[1], row[1], r);
          r = fmaf(wx[2], row[2], r);
          r = fmaf(wx[3], row[3], r);
          v = fmaf(wy[t], r, v);
        }
        acc += v;
      }
    }
  }
  double part = 0.0;
  if (valid) {
    out[gi] += sign * acc;
    if (p) part = (double)p[gi] * (double)(sign * acc);
  }
  if (slot >= 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = 0; i < 8; ++i) s += red[i];
      if (s != 0.0) atomicAdd(&ctl->cur[slot], s);
    }
  }
}

// ---------------------------------------------------------------------------
// Test operators S / S^T (weighted directional gradient / divergence,
// P:L585-601, reading A10) on dense [s_d][H][ps] stacks.
// ---------------------------------------------------------------------------
__global__ void k_apply_S(const Geom G, const float* __restrict__ x, const float* __restrict__ m,
                          float* __restrict__ out) {
  int X = blockIdx.x * blockDim.x + threadIdx.x, Y = blockIdx.y;
  if (X >= G.W || Y >= G.H) return;
  const int ps = G.ps;
  float xz = x[(size_t)Y * ps + X], mz = m[(size_t)Y * ps + X];
  for (int d = 0; d < G.s_d; ++d) {
    int yy = Y + G.ody[d], xx = X + G.odx[d];
    float g = 0.f;
    if (yy >= 0 && yy < G.H && xx >= 0 && xx < G.W) g = G.wd[d] * mz * (xz - x[(size_t)yy * ps + xx]);
    out[((size_t)d * G.H + Y) * ps + X] = g;
  }
}

__global__ void k_apply_ST(const Geom G, const float* __restrict__ hin, const float* __restrict__ m,
                           float* __restrict__ out) {
  int X = blockIdx.x * blockDim.x + threadIdx.x, Y = blockIdx.y;
  if (X >= G.W || Y >= G.H) return;
  const int ps = G.ps;
  float s = 0.f;
  for (int d = 0; d < G.s_d; ++d) {
    int dy = G.ody[d], dx = G.odx[d];
    const float* hd = hin + (size_t)d * G.H * ps;
    if (Y + dy >= 0 && Y + dy < G.H && X + dx >= 0 && X + dx < G.W)
      s += G.wd[d] * m[(size_t)Y * ps + X] * hd[(size_t)Y * ps + X];
    if (Y - dy >= 0 && Y - dy < G.H && X - dx >= 0 && X - dx < G.W)
      s -= G.wd[d] * m[(size_t)(Y - dy) * ps + X - dx] * hd[(size_t)(Y - dy) * ps + X - dx];
  }
  out[(size_t)Y * ps + X] = s;
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
static dim3 hr_grid(const Geom& G, int bx) { return dim3((G.W + bx - 1) / bx, G.H); }

cudaError_t launch_setup_wo(const Geom& G, const Views& V, const float* y, const float* omega, float* wo,
                            cudaStream_t st) {
  k_setup_wo<<<hr_grid(G, 128), 128, 0, st>>>(G, V, y, omega, wo);
  return cudaGetLastError();
}
cudaError_t launch_density(const Geom& G, const Views& V, const float* omega, float* D, cudaStream_t st) {
  k_density<<<hr_grid(G, 128), 128, 0, st>>>(G, V, omega, D);
  return cudaGetLastError();
}
cudaError_t launch_bicubic(const Geom& G, const float* y, float* x, cudaStream_t st) {
  k_bicubic<<<hr_grid(G, 128), 128, 0, st>>>(G, y, x);
  return cudaGetLastError();
}
cudaError_t launch_weights(const Geom& G, const float* x, const float* wo, float* m, cudaStream_t st) {
  k_weights<<<hr_grid(G, 128), 128, 0, st>>>(G, x, wo, m);
  return cudaGetLastError();
}
cudaError_t launch_absmax(const float* v, size_t n, unsigned* out, cudaStream_t st) {
  const size_t n4 = n / 4;
  const int blocks = (int)std::max<size_t>(1, std::min<size_t>((n4 + 255) / 256, 148 * 8));
  k_absmax<<<blocks, 256, 0, st>>>(v, n, out);
  return cudaGetLastError();
}
cudaError_t launch_cg_update(const Geom& G, float* x, float* r, const float* p, float* q, Control* ctl, int k,
                             int row0, int nrows, int close_here, int num_sms, cudaStream_t st) {
  size_t n4 = (size_t)nrows * G.ps / 4;
  int blocks = (int)((n4 + 255) / 256);
  int cap = num_sms * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_cg_update<<<blocks, 256, 0, st>>>(G, x, r, p, q, ctl, k, row0, nrows, close_here);
  return cudaGetLastError();
}
cudaError_t launch_gd_gnorm(const Geom& G, const float* g, Control* ctl, int num_sms, cudaStream_t st) {
  k_gd_gnorm<<<num_sms * 2, 256, 0, st>>>(G, g, ctl);
  return cudaGetLastError();
}
cudaError_t launch_gd_update(const Geom& G, float* x, const float* g, Control* ctl, const GdCfg& cfg, int num_sms,
                             cudaStream_t st) {
  size_t n4 = (size_t)G.H * G.ps / 4;
  int blocks = (int)((n4 + 255) / 256);
  if (blocks > num_sms * 4) blocks = num_sms * 4;
  if (blocks < 1) blocks = 1;
  k_gd_update<<<blocks, 256, 0, st>>>(G, x, g, ctl, cfg);
  return cudaGetLastError();
}
// Colour handling of the paper's experiments ("solve the cost function
// for Y color channel while applying bi-cubic interpolation for Cb and Cr"): full-range
// ITU-R BT.601 YCbCr on [0, 1] (reading A35).  Planar fp32, n pixels per plane.
__global__ void k_rgb_to_ycbcr(const float* __restrict__ rgb, float* __restrict__ y, float* __restrict__ cb,
                               float* __restrict__ cr, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float r = rgb[i], g = rgb[n + i], b = rgb[2 * n + i];
    const float yy = 0.299f * r + 0.587f * g + 0.114f * b;
    y[i] = yy;
    cb[i] = 0.5f + (b - yy) * (1.f / 1.772f);
    cr[i] = 0.5f + (r - yy) * (1.f / 1.402f);
  }
}
__global__ void k_ycbcr_to_rgb(const float* __restrict__ y, const float* __restrict__ cb,
                               const float* __restrict__ cr, float* __restrict__ rgb, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float yy = y[i], u = cb[i] - 0.5f, v = cr[i] - 0.5f;
    const float r = yy + 1.402f * v, b = yy + 1.772f * u;
    rgb[i] = r;
    rgb[n + i] = (yy - 0.299f * r - 0.114f * b) * (1.f / 0.587f);
    rgb[2 * n + i] = b;
  }
}
cudaError_t launch_color(int to_ycbcr, const float* a, float* y, float* cb, float* cr, size_t n, int num_sms,
                         cudaStream_t st) {
  int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)num_sms * 8);
  if (blocks < 1) blocks = 1;
  if (to_ycbcr) k_rgb_to_ycbcr<<<blocks, 256, 0, st>>>(a, y, cb, cr, n);
  else k_ycbcr_to_rgb<<<blocks, 256, 0, st>>>(y, cb, cr, const_cast<float*>(a), n);
  return cudaGetLastError();
}
cudaError_t launch_paper_gather(const Geom& G, const Views& V, const float* rho, const float* omega0, const float* p,
                                float* out, float sign, Control* ctl, int slot, int cg_k, int row0, int nrows,
                                cudaStream_t st) {
  dim3 grid((G.W + 31) / 32, (nrows + 7) / 8);
  const int stride = gather_stride(G);
  int vchunk = std::max(1, std::min(16, (int)(40 * 1024 / (4 * (size_t)stride))));   // <= 40 KB staged
  vchunk = std::min(vchunk, G.n_views);
  k_paper_gather<<<grid, 256, (size_t)vchunk * stride * 4, st>>>(G, V, rho, omega0, p, out, sign, ctl, slot, cg_k,
                                                                 row0, nrows, vchunk, stride);
  return cudaGetLastError();
}
cudaError_t launch_close(const Geom& G, Control* ctl, cudaStream_t st) {
  k_close<<<1, 32, 0, st>>>(G, ctl);
  return cudaGetLastError();
}
cudaError_t launch_apply_S(const Geom& G, const float* x, const float* m, float* out, cudaStream_t st) {
  k_apply_S<<<hr_grid(G, 128), 128, 0, st>>>(G, x, m, out);
  return cudaGetLastError();
}
cudaError_t launch_apply_ST(const Geom& G, const float* h, const float* m, float* out, cudaStream_t st) {
  k_apply_ST<<<hr_grid(G, 128), 128, 0, st>>>(G, h, m, out);
  return cudaGetLastError();
}

}  // namespace lfsr
