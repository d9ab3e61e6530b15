// tile_kernels.cu — the fused observation-operator tile kernel of liblfsr.
//
// One CTA owns an LR tile of LY x LX pixels (an HR tile of zeta*LY x zeta*LX)
// and a group of views.  For each view k it runs, entirely in shared memory:
//   P1  warp W_k: bilinear gather of the HR input at z + dtheta_k*omega(z) for
//       every HR position z of the "E region" (the positions whose blurred
//       value reaches an own LR pixel)                     P:L580-583, A12/A13
//   P2  horizontal Gaussian blur evaluated at LR columns only        P:L579, A11
//   P3  vertical blur at LR rows = D B W_k x (A_k x)   + the per-LR-pixel
//       epilogue: (WZ) e = A_k x - y_k, clamp-form prox + scaled dual update
//       (Alg.1 lines 4-8, A5/A6) -> rho_k; (NORMAL) rho = c_A A_k p
//   P4  vertical adjoint blur (polyphase: only LR taps)          B^T D^T (A11/A14)
//   P5  horizontal adjoint blur + exact bilinear scatter W_k^T into a shared
//       accumulator (the transpose of P1, reading A12)
// then the weighted NLTV part for the own HR pixels, and finally
// flushes the accumulator (tile + halo) to global memory with RED.ADD so that
// neighbouring tiles' halo contributions sum up.  MODE_WZ is the whole wz-step
// of Alg.1 (lines 4-9) and writes r = -v (Alg.2 line 2 with reading A3);
// MODE_NORMAL is q = M p with the CG direction update
// p_k = r_k + beta p_{k-1} fused into the tile load (Alg.2 line 10, A2).
#include "internal.h"
#include <cfloat>

namespace lfsr {

template <int Z> struct TileCfg;
template <> struct TileCfg<2> { static constexpr int R = 2, LY = 16, LX = 32; };
template <> struct TileCfg<3> { static constexpr int R = 3, LY = 11, LX = 22; };
template <> struct TileCfg<4> { static constexpr int R = 3, LY = 8, LX = 16; };

template <int Z> struct TileC {
  static constexpr int R = TileCfg<Z>::R, LY = TileCfg<Z>::LY, LX = TileCfg<Z>::LX;
  static constexpr int TY = Z * LY, TX = Z * LX;
  static constexpr int EY = Z * (LY - 1) + 2 * R + 1, EX = Z * (LX - 1) + 2 * R + 1;
  static constexpr int E = EY * EX;
  static constexpr int MAXP = (E + kThreads - 1) / kThreads;
};


__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV doubles, then one atomicAdd per value into dst[slot[i]].
template <int NV>
__device__ __forceinline__ void block_reduce_add(double (&v)[NV], double* red, double* dst,
                                                 const int (&slot)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[warp * NV + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w * NV + threadIdx.x];
    if (s != 0.0) atomicAdd(dst + slot[threadIdx.x], s);
  }
}

template <int Z, int MODE>
__global__ void __launch_bounds__(kThreads, 2)
k_tile(const Geom G, const Views V, const TileGeom T, const TileIO io) {
  using C = TileC<Z>;
  constexpr int R = C::R, LY = C::LY, LX = C::LX, TY = C::TY, TX = C::TX;
  constexpr int EY = C::EY, EX = C::EX, E = C::E, MAXP = C::MAXP;
  constexpr bool kFwd = (MODE != MODE_AT);
  constexpr bool kAdj = (MODE != MODE_A);

  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x;
  const int ntiles = T.ntY * T.ntX;
  const int tile = blockIdx.x % ntiles;
  const int grp = blockIdx.x / ntiles;
  const int ti = tile / T.ntX, tj = tile % T.ntX;
  const int i0 = ti * LY, j0 = tj * LX;     // LR origin
  const int Y0 = i0 * Z, X0 = j0 * Z;       // HR origin of the own tile
  const int PY0 = Y0 - T.HY, PX0 = X0 - T.HX;  // p-tile origin
  const int PH = T.PH, PW = T.PW;
  const int H = G.H, W = G.W, ps = G.ps;

  Control* ctl = io.ctl;
  if (MODE == MODE_NORMAL && io.cg_k >= 2 && ctl->cur[S_STOP] != 0.0) return;  // CG stopped

  float* P = smem;                  // PH*PW   input tile
  float* ACC = P + PH * PW;         // PH*PW   adjoint accumulator
  float* WP = ACC + PH * PW;        // E       warped input on the E region
  float* T1 = WP + E;               // EY*LX   forward horizontal blur
  float* T1b = T1 + EY * LX;        // EY*LX   adjoint vertical blur
  float* RHO = T1b + EY * LX;       // LY*LX   LR residual / weights
  float* MT = RHO + LY * LX;        // MH*MW   m tile (NORMAL with NLTV)
  // reduction scratch: first 8-byte aligned slot after MT
  const size_t red_off = ((size_t)(MT - smem) + (size_t)T.MH * T.MW + 1) & ~(size_t)1;
  double* RED = reinterpret_cast<double*>(smem + red_off);

  // ---- tile load (and CG direction update) --------------------------------
  double pi0_part = 0.0;
  float beta = 0.f;
  if (MODE == MODE_NORMAL && io.cg_k >= 2) {
    double pim1 = ctl->cur[S_PI + io.cg_k - 1], pim2 = ctl->cur[S_PI + io.cg_k - 2];
    beta = (float)(pim1 / pim2);    // Alg.2 line 10 (reading A2): p_k = r_k + beta p_{k-1}
  }
  for (int e = tid; e < PH * PW; e += kThreads) {
    int py = e / PW, px = e - py * PW;
    int gy = PY0 + py, gx = PX0 + px;
    float v = 0.f;
    if (kFwd && gy >= 0 && gy < H && gx >= 0 && gx < W) {
      size_t gi = (size_t)gy * ps + gx;
      v = io.in_hr[gi];
      if (MODE == MODE_NORMAL && io.cg_k >= 1) {
        bool own = gy >= Y0 && gy < Y0 + TY && gx >= X0 && gx < X0 + TX;
        if (io.cg_k == 1) {
          if (own && grp == 0) pi0_part += (double)v * v;   // pi_0 = <r_0, r_0> (Alg.2 line 3)
        } else {
          v = v + beta * io.in_hr2[gi];
        }
        if (own && grp == 0) io.p_out[gi] = v;
      }
    }
    if (kFwd) P[e] = v;
    if (kAdj) ACC[e] = 0.f;
  }
  // m tile for the NLTV normal term (own + radius halo)
  const int rr = G.radius;
  if (MODE == MODE_NORMAL && io.do_nltv && grp == 0) {
    for (int e = tid; e < T.MH * T.MW; e += kThreads) {
      int my = e / T.MW, mx = e - my * T.MW;
      int gy = Y0 - rr + my, gx = X0 - rr + mx;
      MT[e] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? io.m[(size_t)gy * ps + gx] : 0.f;
    }
  }
  // disparity on the E region, kept in registers for all views
  float om[MAXP];
#pragma unroll
  for (int s = 0; s < MAXP; ++s) {
    int e = tid + s * kThreads;
    om[s] = 0.f;
    if (e < E) {
      int er = e / EX, ec = e - er * EX;
      int Y = Y0 - R + er, X = X0 - R + ec;
      if (Y >= 0 && Y < H && X >= 0 && X < W) om[s] = io.omega[(size_t)Y * ps + X];
    }
  }
  __syncthreads();

  // ---- per-view observation operator (forward + adjoint) -------------------
  double red_a = 0.0, red_b = 0.0, red_c = 0.0;  // WZ: l1, l2, res2 ; NORMAL: pq
  const int kbeg = grp * T.vpg;
  const int kend = min(G.n_views, kbeg + T.vpg);
  const float lam1 = G.lambda1, lam2 = G.lambda2, ith = G.inv_theta;
  for (int k = kbeg; k < kend; ++k) {
    const float drho = V.off[k].x, dtau = V.off[k].y;
    int cidx[MAXP];
    float ca[MAXP], cb[MAXP];
    // P1: W_k (bilinear gather, replicate-clamped coordinate)
#pragma unroll
    for (int s = 0; s < MAXP; ++s) {
      int e = tid + s * kThreads;
      cidx[s] = -1;
      ca[s] = 0.f;
      cb[s] = 0.f;
      if (e < E) {
        int er = e / EX, ec = e - er * EX;
        int Y = Y0 - R + er, X = X0 - R + ec;
        float wp = 0.f;
        if (Y >= 0 && Y < H && X >= 0 && X < W) {
          float sy = fminf(fmaxf((float)Y + dtau * om[s], 0.f), (float)(H - 1));
          float sx = fminf(fmaxf((float)X + drho * om[s], 0.f), (float)(W - 1));
          float fy = floorf(sy), fx = floorf(sx);
          float a = sy - fy, b = sx - fx;
          int idx = ((int)fy - PY0) * PW + ((int)fx - PX0);
          cidx[s] = idx;
          ca[s] = a;
          cb[s] = b;
          if (kFwd) {
            float p00 = P[idx], p01 = P[idx + 1], p10 = P[idx + PW], p11 = P[idx + PW + 1];
            wp = (1.f - a) * ((1.f - b) * p00 + b * p01) + a * ((1.f - b) * p10 + b * p11);
          }
        }
        if (kFwd) WP[e] = wp;
      }
    }
    __syncthreads();
    if (kFwd) {
      // P2: horizontal blur at LR columns
      for (int e = tid; e < EY * LX; e += kThreads) {
        int er = e / LX, lj = e - er * LX;
        const float* row = WP + er * EX + Z * lj;
        float s = 0.f;
#pragma unroll
        for (int v = 0; v <= 2 * R; ++v) s += G.taps[v] * row[v];
        T1[e] = s;
      }
      __syncthreads();
      // P3: vertical blur at LR rows -> A_k x ; per-pixel epilogue
      for (int l = tid; l < LY * LX; l += kThreads) {
        int li = l / LX, lj = l - li * LX;
        int i = i0 + li, j = j0 + lj;
        float a = 0.f;
#pragma unroll
        for (int u = 0; u <= 2 * R; ++u) a += G.taps[u] * T1[(Z * li + u) * LX + lj];
        float rho = 0.f;
        if (i < G.h && j < G.w) {
          size_t li_g = ((size_t)k * G.h + i) * G.lps + j;
          if (MODE == MODE_A) {
            io.out_lr[li_g] = a;
          } else if (MODE == MODE_NORMAL) {
            rho = G.cA * a;
            red_a += (double)G.cA * (double)a * (double)a;   // <p, c_A A^T A p> = c_A |A p|^2
          } else if (MODE == MODE_WZ) {
            float e_ = a - io.y[li_g];                        // e = A_k x - y_k (Alg.1 line 4)
            float wa = io.wA[li_g];
            float u = lam1 * e_ + wa;                          // u = F x - b' + w (line 5)
            float wn = fminf(fmaxf(u, -ith), ith);             // w+ = u - prox(u) = clamp (A5/A6)
            float f = 2.f * wn - wa;                           // f = 2w^n - w^{n-1} (line 8)
            rho = lam2 * e_ + G.cS * lam1 * f;                 // A^T a + (th/2) F^T f, data rows
            io.wA[li_g] = wn;
            red_a += fabs((double)e_);
            red_b += (double)e_ * e_;
            red_c += (double)(wn - wa) * (wn - wa);
          }
        }
        RHO[l] = rho;
      }
      __syncthreads();
    } else {
      for (int l = tid; l < LY * LX; l += kThreads) {
        int li = l / LX, lj = l - li * LX;
        int i = i0 + li, j = j0 + lj;
        RHO[l] = (i < G.h && j < G.w) ? io.in_lr[((size_t)k * G.h + i) * G.lps + j] : 0.f;
      }
      __syncthreads();
    }
    if (kAdj) {
      // P4: vertical adjoint blur (polyphase: only the LR rows within R)
      for (int e = tid; e < EY * LX; e += kThreads) {
        int er = e / LX, lj = e - er * LX;
        int lo = er - 2 * R;
        int li_lo = lo <= 0 ? 0 : (lo + Z - 1) / Z;
        int li_hi = min(LY - 1, er / Z);
        float s = 0.f;
        for (int li = li_lo; li <= li_hi; ++li) s += G.taps[er - Z * li] * RHO[li * LX + lj];
        T1b[e] = s;
      }
      __syncthreads();
      // P5: horizontal adjoint blur + exact bilinear scatter (W_k^T)
#pragma unroll
      for (int s = 0; s < MAXP; ++s) {
        int e = tid + s * kThreads;
        if (e < E && cidx[s] >= 0) {
          int er = e / EX, ec = e - er * EX;
          int lo = ec - 2 * R;
          int lj_lo = lo <= 0 ? 0 : (lo + Z - 1) / Z;
          int lj_hi = min(LX - 1, ec / Z);
          float t = 0.f;
          for (int lj = lj_lo; lj <= lj_hi; ++lj) t += G.taps[ec - Z * lj] * T1b[er * LX + lj];
          if (t != 0.f) {
            float a = ca[s], b = cb[s];
            int idx = cidx[s];
            atomicAdd(&ACC[idx], (1.f - a) * (1.f - b) * t);
            atomicAdd(&ACC[idx + 1], (1.f - a) * b * t);
            atomicAdd(&ACC[idx + PW], a * (1.f - b) * t);
            atomicAdd(&ACC[idx + PW + 1], a * b * t);
          }
        }
      }
      // no barrier: the next view's P1 writes WP only; T1b/RHO are rewritten
      // after three more barriers.
    }
  }

  // ---- NLTV part (group 0) ---------------------------------------------------
  double red_reg = 0.0;
  if ((MODE == MODE_WZ || (MODE == MODE_NORMAL && io.do_nltv)) && grp == 0) {
    if (MODE == MODE_NORMAL) __syncthreads();  // MT visible (loaded before the view loop)
    const int sd = G.s_d;
    for (int e = tid; e < TY * TX; e += kThreads) {
      int oy = e / TX, ox = e - oy * TX;
      int Y = Y0 + oy, X = X0 + ox;
      if (Y >= H || X >= W) continue;
      const int pz = (Y - PY0) * PW + (X - PX0);
      const float xz = P[pz];
      if (MODE == MODE_WZ) {
        // m = lambda_R w_o exp(-|grad x|^2 / sigma_e), central differences, replicate
        // border (readings A8/A17/A19), recomputed from x^{n-1}
        float mz;
        size_t gi = (size_t)Y * ps + X;
        if (io.reweight) {
          float xr = P[(Y - PY0) * PW + (min(X + 1, W - 1) - PX0)];
          float xl = P[(Y - PY0) * PW + (max(X - 1, 0) - PX0)];
          float xd = P[(min(Y + 1, H - 1) - PY0) * PW + (X - PX0)];
          float xu = P[(max(Y - 1, 0) - PY0) * PW + (X - PX0)];
          float gx = 0.5f * (xr - xl), gy = 0.5f * (xd - xu);
          mz = G.lambda_reg * io.wo[gi] * expf(-(gx * gx + gy * gy) * G.inv_sigma_e);
          if (grp == 0) io.m[gi] = mz;
        } else {
          mz = io.m[gi];
        }
        float vown = 0.f;
        for (int d = 0; d < sd; ++d) {
          const int dy = G.ody[d], dx = G.odx[d];
          const bool in = (Y + dy >= 0) && (Y + dy < H) && (X + dx >= 0) && (X + dx < W);
          const float Wd = G.wd[d] * mz;
          float g = 0.f;
          if (in) g = Wd * (xz - P[pz + dy * PW + dx]);       // W_d (.) Delta_d x
          float* wsp = io.wS + (size_t)d * H * ps + gi;
          float wso = *wsp;
          float u = g + wso;                                    // u = F x - b' + w, NLTV rows
          float wn = fminf(fmaxf(u, -ith), ith);                // clamp form of z/w steps
          float f = 2.f * wn - wso;
          *wsp = wn;
          red_reg += fabs((double)g);
          red_c += (double)(wn - wso) * (wn - wso);
          if (in) {                                             // (th/2) Delta_d^T (W_d f_d)
            float hcon = G.cS * Wd * f;
            vown += hcon;
            atomicAdd(&ACC[pz + dy * PW + dx], -hcon);
          }
        }
        atomicAdd(&ACC[pz], vown);
      } else {
        // (th/2) sum_d Delta_d^T (W_d^2 Delta_d p) in gather form, using the m tile
        const int MW = T.MW;
        const int mzi = (oy + rr) * MW + (ox + rr);
        const float mz = MT[mzi];
        float qs = 0.f, pq = 0.f;
        for (int d = 0; d < sd; ++d) {
          const int dy = G.ody[d], dx = G.odx[d];
          const float wd = G.wd[d];
          if ((Y + dy >= 0) && (Y + dy < H) && (X + dx >= 0) && (X + dx < W)) {
            float dp = xz - P[pz + dy * PW + dx];
            float w2 = (wd * mz) * (wd * mz);
            qs += w2 * dp;
            pq += w2 * dp * dp;
          }
          if ((Y - dy >= 0) && (Y - dy < H) && (X - dx >= 0) && (X - dx < W)) {
            float dpb = P[pz - dy * PW - dx] - xz;
            float mb = wd * MT[mzi - dy * MW - dx];
            qs -= mb * mb * dpb;
          }
        }
        atomicAdd(&ACC[pz], G.cS * qs);
        red_b += (double)G.cS * pq;
      }
    }
  }
  if (MODE == MODE_A) return;
  __syncthreads();

  // ---- flush the accumulator (tile + halo) with RED.ADD --------------------
  if (kAdj) {
    const float sign = (MODE == MODE_WZ) ? -1.f : 1.f;   // WZ writes r = -v (reading A3)
    for (int e = tid; e < PH * PW; e += kThreads) {
      float v = ACC[e];
      if (v == 0.f) continue;
      int py = e / PW, px = e - py * PW;
      int gy = PY0 + py, gx = PX0 + px;
      if (gy >= 0 && gy < H && gx >= 0 && gx < W) atomicAdd(&io.out_hr[(size_t)gy * ps + gx], sign * v);
    }
  }
  // ---- reductions --------------------------------------------------------------
  if (MODE == MODE_WZ) {
    double v[4] = {red_a, red_b, red_reg, red_c};
    const int slot[4] = {S_L1, S_L2, S_REG, S_RES2};
    block_reduce_add<4>(v, RED, ctl->cur, slot);
  } else if (MODE == MODE_NORMAL && io.cg_k >= 1) {
    double v[2] = {red_a + red_b, pi0_part};
    const int slot[2] = {S_PQ + io.cg_k, S_PI + 0};
    block_reduce_add<2>(v, RED, ctl->cur, slot);
  }
}

// --------------------------------------------------------------------------------
// Host-side geometry and launchers
// --------------------------------------------------------------------------------
TileGeom make_tile_geom(const Geom& G, int num_sms) {
  TileGeom T{};
  int LY = 0, LX = 0, R = 0, EY = 0, EX = 0;
  switch (G.scale) {
    case 2: LY = TileC<2>::LY; LX = TileC<2>::LX; R = TileC<2>::R; EY = TileC<2>::EY; EX = TileC<2>::EX; break;
    case 3: LY = TileC<3>::LY; LX = TileC<3>::LX; R = TileC<3>::R; EY = TileC<3>::EY; EX = TileC<3>::EX; break;
    default: LY = TileC<4>::LY; LX = TileC<4>::LX; R = TileC<4>::R; EY = TileC<4>::EY; EX = TileC<4>::EX; break;
  }
  T.LY = LY; T.LX = LX; T.TY = G.scale * LY; T.TX = G.scale * LX;
  T.EY = EY; T.EX = EX;
  int sy = G.SY > G.radius ? G.SY : G.radius;
  int sx = G.SX > G.radius ? G.SX : G.radius;
  T.HY = R + sy;
  T.HX = R + sx;
  T.PH = EY + 2 * sy + 1;
  T.PW = EX + 2 * sx + 1;
  T.MH = T.TY + 2 * G.radius;
  T.MW = T.TX + 2 * G.radius;
  T.ntY = (G.h + LY - 1) / LY;
  T.ntX = (G.w + LX - 1) / LX;
  int tiles = T.ntY * T.ntX;
  int groups = (2 * num_sms + tiles - 1) / tiles;
  if (groups > G.n_views) groups = G.n_views;
  if (groups < 1) groups = 1;
  T.vpg = (G.n_views + groups - 1) / groups;
  T.groups = (G.n_views + T.vpg - 1) / T.vpg;
  size_t floats = 2 * (size_t)T.PH * T.PW + (size_t)EY * EX + 2 * (size_t)EY * LX + (size_t)LY * LX +
                  (size_t)T.MH * T.MW + 2;  // +2: 8-byte alignment of the reduction scratch
  T.smem = floats * sizeof(float) + (kThreads / 32) * 4 * sizeof(double);
  return T;
}

template <int Z, int MODE>
static cudaError_t prepare_z(size_t smem) {
  return cudaFuncSetAttribute(k_tile<Z, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t prepare_tile_kernels(int scale, size_t smem) {
  cudaError_t e = cudaSuccess;
#define PREP(Z)                                                        \
  if (scale == Z) {                                                    \
    if ((e = prepare_z<Z, MODE_WZ>(smem)) != cudaSuccess) return e;     \
    if ((e = prepare_z<Z, MODE_NORMAL>(smem)) != cudaSuccess) return e; \
    if ((e = prepare_z<Z, MODE_A>(smem)) != cudaSuccess) return e;      \
    if ((e = prepare_z<Z, MODE_AT>(smem)) != cudaSuccess) return e;     \
  }
  PREP(2) PREP(3) PREP(4)
#undef PREP
  return e;
}

template <int Z, int MODE>
static cudaError_t launch_z(const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                            cudaStream_t st, int groups) {
  auto kern = k_tile<Z, MODE>;
  dim3 grid(T.ntY * T.ntX * groups);
  kern<<<grid, kThreads, T.smem, st>>>(G, V, T, io);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_mode(const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                               cudaStream_t st, int groups) {
  switch (G.scale) {
    case 2: return launch_z<2, MODE>(G, V, T, io, st, groups);
    case 3: return launch_z<3, MODE>(G, V, T, io, st, groups);
    case 4: return launch_z<4, MODE>(G, V, T, io, st, groups);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_tile(int mode, const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                        cudaStream_t st) {
  switch (mode) {
    case MODE_WZ: return launch_mode<MODE_WZ>(G, V, T, io, st, T.groups);
    case MODE_NORMAL: return launch_mode<MODE_NORMAL>(G, V, T, io, st, T.groups);
    case MODE_A: return launch_mode<MODE_A>(G, V, T, io, st, T.groups);
    case MODE_AT: return launch_mode<MODE_AT>(G, V, T, io, st, T.groups);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lfsr
