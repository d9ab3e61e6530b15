// misr.cu — the translation-invariant fast path of the CG normal operator (SURVEY §8f NEXT-1,
// the MISR / global-shift workload of P:L1110-1123).
//
// With one constant disparity c (every view a global translation s_k = dtheta_k c, P:L580-583
// with omega constant), W_k is, away from the image border, a bilinear translation, B a
// convolution and D a decimation, so the data part of the normal operator
//     M_data = c_A sum_k W_k^T B^T D^T D B W_k                         (A7)
// is a zeta^2-phase periodic stencil: (M_data p)(z) = sum_Delta S[phase(z)][Delta] p(z + Delta)
// with |Delta| <= 2R + 1 per axis.  S is assembled once per set_observations on the host in
// fp64 (capi.cu: misr_setup) and travels in the kernel parameter block, so every tap is an
// FFMA with a constant-bank operand.  The weighted NLTV part (A10)
//     (S_W^T S_W p)(z) = sum_d (p(z) - p(z+d)) (w_d^2 m(z)^2 + w_{-d}^2 m(z+d)^2)
// is evaluated in the same register-streaming pass as three 24-tap stencils on p, m^2 and m^2 p.
// The stencil is exact only where every LR pixel that reaches z has an unclamped, unpadded row of
// A_k (the rectangle Z_s computed by misr_setup); the border band outside Z_s is computed by the
// exact tile kernel on the border tiles only, with its flush masked to the band (tile_impl.cuh).
//
// k_misr_normal: one thread = a zeta-wide column of RT = NB zeta output rows (all zeta^2 phases,
// so the stencil taps are warp-uniform); a warp = 32 such columns side by side; 8 warps stacked.
// The input rows stream through registers (LDS.64 / LDS.128 where the lane stride allows).
// CG step k >= 1: p = r + beta p_{k-1} is formed in the tile load (Alg.2 line 10, A2), written
// for the pixels this kernel owns, pi_0 (k = 1) over them; <p, q> over the whole image (the band
// from the q the border kernel already accumulated) goes to the step's slot (Alg.2 line 7).
#include "internal.h"
#include <cstdio>
#include <type_traits>

namespace lfsr {

template <int Z> struct MisrCfg {
  static constexpr int R = Z == 2 ? 2 : 3;
  static constexpr int WR = 2 * R + 1;        // stencil half width
  static constexpr int NB = Z == 2 ? 4 : 2;   // zeta x zeta blocks per thread, stacked
  static constexpr int RT = NB * Z;           // output rows per thread
  static constexpr int NW = Z == 4 ? 4 : 8;   // warps per CTA (stacked)
  static constexpr int TH = NW * RT, TW = 32 * Z;   // output tile
  static constexpr int PHh = TH + 2 * WR;
  static constexpr int VEC = (Z % 4 == 0) ? 4 : (Z % 2 == 0 ? 2 : 1);
  static constexpr int NC = Z + 2 * WR;                              // input columns per thread
  static constexpr int NCV = (NC + VEC - 1) / VEC * VEC;
  static constexpr int PWh = ((TW + 2 * WR + VEC) + 3) / 4 * 4;     // smem row pitch (>= 32 (Z-1) + NCV)
  static constexpr int RAD = 2;                                      // NLTV window 5x5
  static constexpr int PHm = TH + 2 * RAD, PWm = TW + 2 * RAD;       // m^2, m^2 p tiles
  static constexpr int NWT = 2 * WR + 1;                             // taps of the 1-D matrices
  static constexpr size_t kSmem = (size_t)(PHh * PWh + 2 * PHm * PWm + TH * NWT) * 4;
};

// compile-time loop: f(integral_constant<int, I>) for I in [I0, N) -- the streaming loop must be
// unrolled completely so that every stencil tap is an FFMA with a constant-bank operand
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

__device__ __forceinline__ double misr_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// SEP: the separable form (rank-1 data stencil per phase pair, separable NLTV weights): a
// horizontal pass per streamed row, then vertical taps -- 2 (2WR + 1) + 3 x 10 FMAs per pixel
// instead of (2WR + 1)^2 + 72.
template <int Z, bool SEP>
__global__ void __launch_bounds__(MisrCfg<Z>::NW * 32)
k_misr_normal(const Geom G, const __grid_constant__ MisrStencil S, const MisrArgs a) {
  using C = MisrCfg<Z>;
  constexpr int WR = C::WR, RT = C::RT, TH = C::TH, TW = C::TW, PHh = C::PHh, PWh = C::PWh;
  constexpr int NCV = C::NCV, VEC = C::VEC, RAD = C::RAD;
  constexpr int PHm = C::PHm, PWm = C::PWm;
  extern __shared__ __align__(16) float smem_misr[];
  float* sp = smem_misr;                 // p on tile + WR halo
  float* smm = sp + PHh * PWh;           // m^2 on tile + RAD halo (NLTV)
  float* smp = smm + PHm * PWm;          // m^2 p
  float* sty = smp + PHm * PWm;          // sep: T_y rows of the tile
  __shared__ double red[C::NW * 2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Y0 = blockIdx.y * TH, X0 = blockIdx.x * TW;
  const int H = G.H, W = G.W, ps = G.ps;
  Control* ctl = a.ctl;
  if (a.cg_k >= 2 && ctl->cur[S_STOP] != 0.0) return;   // CG stopped (as the tile kernel)
  float beta = 0.f;
  if (a.cg_k >= 2) beta = (float)(ctl->cur[S_PI + a.cg_k - 1] / ctl->cur[S_PI + a.cg_k - 2]);   // A2
  double pi0 = 0.0, pq = 0.0;

  // ---- tile load: p (formed from r, p_{k-1}), zero outside the image; then m^2 and m^2 p.
  // U independent loads in flight per thread (the load is latency bound: one CTA wave only
  // hides so much), the m tile's loads issued before the p tile is combined ----
  constexpr int NT = C::NW * 32, U = 8;
  const float* src1 = a.cg_k == 0 ? a.p_in : a.r;
  for (int e0 = tid; e0 < PHh * PWh; e0 += U * NT) {
    float v1[U], v2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      const int py = e / PWh, px = e - py * PWh;
      const int gy = Y0 - WR + py, gx = X0 - WR + px;
      const bool in = e < PHh * PWh && gy >= 0 && gy < H && gx >= 0 && gx < W && px < TW + 2 * WR;
      const size_t gi = in ? (size_t)gy * ps + gx : 0;
      v1[u] = in ? __ldg(src1 + gi) : 0.f;
      v2[u] = (in && a.cg_k >= 2) ? __ldg(a.p_prev + gi) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      if (e >= PHh * PWh) break;
      float pv = v1[u];
      if (a.cg_k >= 2) pv = pv + beta * v2[u];   // the tile kernel's rounding
      if (a.cg_k >= 1) {
        const int py = e / PWh, px = e - py * PWh;
        const int gy = Y0 - WR + py, gx = X0 - WR + px;
        const bool own = py >= WR && py < WR + TH && px >= WR && px < WR + TW;
        if (own && gy < H && gx < W && gy >= a.o_y0 && gy < a.o_y1 && gx >= a.o_x0 && gx < a.o_x1) {
          a.p_out[(size_t)gy * ps + gx] = pv;
          if (a.cg_k == 1) pi0 += (double)pv * pv;                 // pi_0 = <r_0, r_0> (Alg.2 line 3)
        }
      }
      sp[e] = pv;
    }
  }
  if constexpr (SEP)
    for (int e = tid; e < TH * C::NWT; e += NT) {
      const int gy = Y0 + e / C::NWT;
      sty[e] = gy < H ? __ldg(a.tyt + (size_t)Y0 * C::NWT + e) : 0.f;
    }
  if (a.do_nltv) {
    __syncthreads();
    for (int e0 = tid; e0 < PHm * PWm; e0 += U * NT) {
      float mv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * NT;
        const int py = e / PWm, px = e - py * PWm;
        const int gy = Y0 - RAD + py, gx = X0 - RAD + px;
        const bool in = e < PHm * PWm && gy >= 0 && gy < H && gx >= 0 && gx < W;
        mv[u] = in ? __ldg(a.m + (size_t)gy * ps + gx) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * NT;
        if (e >= PHm * PWm) break;
        const int py = e / PWm, px = e - py * PWm;
        const float mm = mv[u] * mv[u];
        smm[e] = mm;
        smp[e] = mm * sp[(py + WR - RAD) * PWh + px + WR - RAD];
      }
    }
  }
  __syncthreads();

  // ---- streaming stencil: thread = columns X0 + Z lane + [0, Z), rows Y0 + RT warp + [0, RT) ----
  constexpr int NWT = C::NWT;
  float txr[SEP ? Z : 1][SEP ? NWT : 1];   // sep: this thread's columns of T_x (registers)
  if constexpr (SEP) {
#pragma unroll
    for (int c = 0; c < Z; ++c) {
      const int gx = X0 + Z * lane + c;
#pragma unroll
      for (int t = 0; t < NWT; ++t) txr[c][t] = gx < W ? __ldg(a.txt + (size_t)gx * NWT + t) : 0.f;
    }
  }
  float acc[RT][Z], nA[RT][Z], nB[RT][Z], nC[RT][Z];
#pragma unroll
  for (int o = 0; o < RT; ++o)
#pragma unroll
    for (int c = 0; c < Z; ++c) acc[o][c] = nA[o][c] = nB[o][c] = nC[o][c] = 0.f;
  const int row0 = RT * warp, col0 = Z * lane;
  static_for<0, RT + 2 * WR>([&](auto IYc) {
    constexpr int iy = decltype(IYc)::value;
    float v[NCV];
    const float* src = sp + (row0 + iy) * PWh + col0;
    if constexpr (VEC == 4) {
#pragma unroll
      for (int j = 0; j < NCV; j += 4) {
        const float4 t = *reinterpret_cast<const float4*>(src + j);
        v[j] = t.x; v[j + 1] = t.y; v[j + 2] = t.z; v[j + 3] = t.w;
      }
    } else if constexpr (VEC == 2) {
#pragma unroll
      for (int j = 0; j < NCV; j += 2) {
        const float2 t = *reinterpret_cast<const float2*>(src + j);
        v[j] = t.x; v[j + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < NCV; ++j) v[j] = src[j];
    }
    if constexpr (SEP) {
      float h[Z];   // horizontal pass of this row at the thread's columns (phase px = c)
#pragma unroll
      for (int c = 0; c < Z; ++c) {
        float t = 0.f;
#pragma unroll
        for (int dx = 0; dx <= 2 * WR; ++dx) t = fmaf(txr[c][dx], v[c + dx], t);
        h[c] = t;
      }
#pragma unroll
      for (int o = 0; o < RT; ++o) {
        const int dy = iy - o;   // compile time
        if (dy < 0 || dy > 2 * WR) continue;
        const float ty = sty[(row0 + o) * NWT + dy];   // warp-uniform (broadcast)
#pragma unroll
        for (int c = 0; c < Z; ++c) acc[o][c] = fmaf(ty, h[c], acc[o][c]);
      }
    } else {
#pragma unroll
      for (int o = 0; o < RT; ++o) {
        const int dy = iy - o;   // compile time
        if (dy < 0 || dy > 2 * WR) continue;
#pragma unroll
        for (int c = 0; c < Z; ++c) {
          const int ph = (o % Z) * Z + c;
          float t = acc[o][c];
#pragma unroll
          for (int dx = 0; dx <= 2 * WR; ++dx) t = fmaf(S.s[(ph * (2 * WR + 1) + dy) * (2 * WR + 1) + dx], v[c + dx], t);
          acc[o][c] = t;
        }
      }
    }
    // NLTV rows within RAD of an output row
    if (iy >= WR - RAD && iy <= RT - 1 + WR + RAD && a.do_nltv) {
      float mmv[Z + 2 * RAD], mpv[Z + 2 * RAD];
      const int off = (row0 + iy - WR + RAD) * PWm + col0;
#pragma unroll
      for (int j = 0; j < Z + 2 * RAD; ++j) {
        mmv[j] = smm[off + j];
        mpv[j] = smp[off + j];
      }
      if constexpr (SEP) {   // u (x) u over the full 5x5 window; the centre is removed in the epilogue
        float hp[Z], hm[Z], hc[Z];
#pragma unroll
        for (int c = 0; c < Z; ++c) {
          float t0 = 0.f, t1 = 0.f, t2 = 0.f;
#pragma unroll
          for (int dx = -RAD; dx <= RAD; ++dx) {
            t0 = fmaf(S.u[dx + RAD], v[c + WR + dx], t0);
            t1 = fmaf(S.u[dx + RAD], mmv[c + RAD + dx], t1);
            t2 = fmaf(S.u[dx + RAD], mpv[c + RAD + dx], t2);
          }
          hp[c] = t0; hm[c] = t1; hc[c] = t2;
        }
#pragma unroll
        for (int o = 0; o < RT; ++o) {
          const int dn = iy - WR - o;
          if (dn < -RAD || dn > RAD) continue;
#pragma unroll
          for (int c = 0; c < Z; ++c) {
            nA[o][c] = fmaf(S.u[dn + RAD], hp[c], nA[o][c]);
            nB[o][c] = fmaf(S.u[dn + RAD], hm[c], nB[o][c]);
            nC[o][c] = fmaf(S.u[dn + RAD], hc[c], nC[o][c]);
          }
        }
      } else {
#pragma unroll
        for (int o = 0; o < RT; ++o) {
          const int dn = iy - WR - o;
          if (dn < -RAD || dn > RAD) continue;
#pragma unroll
          for (int c = 0; c < Z; ++c) {
#pragma unroll
            for (int dx = -RAD; dx <= RAD; ++dx) {
              if (dn == 0 && dx == 0) continue;
              const int lin = (dn + RAD) * (2 * RAD + 1) + (dx + RAD);
              const int d = lin > (2 * RAD + 1) * RAD + RAD ? lin - 1 : lin;   // A9 order, centre skipped
              nA[o][c] = fmaf(S.w2[d], v[c + WR + dx], nA[o][c]);
              nB[o][c] = fmaf(S.w2f[d], mmv[c + RAD + dx], nB[o][c]);
              nC[o][c] = fmaf(S.w2f[d], mpv[c + RAD + dx], nC[o][c]);
            }
          }
        }
      }
    }
  });

  // ---- epilogue: q on Z_s (store), <p, q> over the tile (band: the border kernel's q) ----
#pragma unroll
  for (int o = 0; o < RT; ++o) {
    const int gy = Y0 + row0 + o;
#pragma unroll
    for (int c = 0; c < Z; ++c) {
      const int gx = X0 + col0 + c;
      if (gy >= H || gx >= W) continue;
      const int li = (row0 + o + WR) * PWh + col0 + c + WR;
      const float pz = sp[li];
      const size_t gi = (size_t)gy * ps + gx;
      float qz;
      if (gy >= a.zs_y0 && gy < a.zs_y1 && gx >= a.zs_x0 && gx < a.zs_x1) {
        qz = acc[o][c];
        if (a.do_nltv) {
          const int lm = (row0 + o + RAD) * PWm + col0 + c + RAD;
          const float mz = smm[lm];
          float A_ = nA[o][c], B_ = nB[o][c], C_ = nC[o][c];
          float W2z = S.W2;
          if constexpr (SEP) {   // drop the centre term u0^2 of the separable window; only pairs inside (A10)
            const float u00 = S.u[RAD] * S.u[RAD];
            A_ = fmaf(-u00, pz, A_);
            B_ = fmaf(-u00, mz, B_);
            C_ = fmaf(-u00, smp[lm], C_);
            float uy = 0.f, ux = 0.f;
#pragma unroll
            for (int t = -RAD; t <= RAD; ++t) {
              uy += (gy + t >= 0 && gy + t < H) ? S.u[t + RAD] : 0.f;
              ux += (gx + t >= 0 && gx + t < W) ? S.u[t + RAD] : 0.f;
            }
            W2z = fmaf(uy, ux, -u00);
          }
          qz += G.cS * (pz * fmaf(mz, W2z, B_) - fmaf(mz, A_, C_));
        }
        a.q[gi] = qz;
      } else {
        qz = a.cg_k >= 1 ? a.q[gi] : 0.f;   // band: exact tile kernel (already in q)
      }
      if (a.cg_k >= 1) pq += (double)pz * qz;
    }
  }
  if (a.cg_k >= 1) {
    pq = misr_warp_sum(pq);
    pi0 = misr_warp_sum(pi0);
    if (lane == 0) {
      red[warp * 2] = pq;
      red[warp * 2 + 1] = pi0;
    }
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int w = 0; w < C::NW; ++w) {
        s0 += red[w * 2];
        s1 += red[w * 2 + 1];
      }
      if (s0 != 0.0) atomicAdd(&ctl->cur[S_PQ + a.cg_k], s0);
      if (s1 != 0.0) atomicAdd(&ctl->cur[S_PI], s1);
    }
  }
}

__global__ void k_omega_const(const float* __restrict__ om, int H, int W, int ps, unsigned* flag) {
  const float c0 = om[0];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)H * W; i += (size_t)gridDim.x * blockDim.x) {
    const size_t y = i / W, x = i - y * W;
    const float v = om[y * ps + x];
    if (!(v == c0)) {   // NaN counts as not constant
      atomicOr(flag, 1u);
      return;
    }
  }
}

cudaError_t launch_omega_const(const Geom& G, const float* omega, unsigned* flag, cudaStream_t st) {
  k_omega_const<<<256, 256, 0, st>>>(omega, G.H, G.W, G.ps, flag);
  return cudaGetLastError();
}

size_t misr_coef_count(int scale) {
  const int R = scale == 2 ? 2 : 3, n = 4 * R + 3;
  return (size_t)scale * scale * n * n;
}

template <int Z, bool SEP>
static cudaError_t prep_one() {
  return cudaFuncSetAttribute(k_misr_normal<Z, SEP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)MisrCfg<Z>::kSmem);
}

cudaError_t prepare_misr_kernels() {
  cudaError_t e;
  if ((e = prep_one<2, false>()) || (e = prep_one<2, true>()) || (e = prep_one<3, false>()) ||
      (e = prep_one<3, true>()) || (e = prep_one<4, false>()) || (e = prep_one<4, true>()))
    return e;
  return cudaSuccess;
}

template <int Z>
static void launch_z(const Geom& G, const MisrStencil& S, const MisrArgs& a, cudaStream_t st) {
  using C = MisrCfg<Z>;
  dim3 grid((G.W + C::TW - 1) / C::TW, (G.H + C::TH - 1) / C::TH);
  if (S.sep) k_misr_normal<Z, true><<<grid, C::NW * 32, C::kSmem, st>>>(G, S, a);
  else k_misr_normal<Z, false><<<grid, C::NW * 32, C::kSmem, st>>>(G, S, a);
}

cudaError_t launch_misr_normal(const Geom& G, const MisrStencil& S, const MisrArgs& a, cudaStream_t st) {
  switch (G.scale) {
    case 2: launch_z<2>(G, S, a, st); break;
    case 3: launch_z<3>(G, S, a, st); break;
    case 4: launch_z<4>(G, S, a, st); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace lfsr
