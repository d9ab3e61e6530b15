// asm.cu — the assembled data normal operator of the CG x-step.
//
// The CG normal operator (A7)
//     M = c_A sum_k A_k^T A_k + (th/2) S_W^T S_W,      A_k = D B W_k
// has a data part that does not change during a solve: omega, the blur and the views are fixed
// once set_observations returns, only the NLTV weights m change per ADMM iteration.
// Written row by row of the stacked A (one row per view k and LR pixel i,
//     a_{k,i} = sum_{u,v} g[u] g[v] bil_k(zeta i + (u, v))       (positions outside Omega dropped, A11)
// with bil_k(z) the four bilinear weights of the sample z + dtheta_k omega(z), A12/A13), the data
// part is the sum of outer products c_A sum_{k,i} a a^T.  A row whose cells fit a (2R + 2)^2
// window ("regular": everywhere except where the blur window straddles a depth edge, ~96 % of the
// rows of the HCI-shaped C3 light field) only couples cells at most SR = 2R + 1 apart per axis,
// so the regular rows sum to a banded operator stored as a stencil per HR pixel, (2 SR + 1)^2
// coefficients of which the symmetric half (NH = 61 at zeta = 2, 113 at zeta = 3, 4) is kept:
//     st[h][a] = c_A sum_{regular (k,i)} a_{k,i}[a] a_{k,i}[a + d_h],   d_h = (h / NSW, h % NSW) (see hoff)
//     (M_reg p)(a) = st[0][a] p(a) + sum_{h>0} st[h][a] p(a + d_h) + st[h][a - d_h] p(a - d_h).
// The irregular rows are applied exactly as rows, through the HR positions of their blur windows:
// u = W_k p there, t = c_A a . p = c_A sum g g u per row, T = sum over the irregular rows holding a
// position of g g t, and T bil_k added into q.
//
// Kernels:
//   k_asm_rows      setup: every row of the stacked A_k evaluated once: regular rows -> a record
//                   (window weights + base), irregular rows -> a compact list (k, iy << 16 | ix)
//                   and a bitmask of their window positions (k_asm_plist compacts it)
//   k_asm_stencil   setup: the stored half of the stencil, one CTA per 16 x 16 output cells,
//                   thread = cell (owner computes: every coefficient is summed by one thread in a
//                   fixed order, no atomics), the footprint's row records loaded view by view
//   k_asm_normal    per CG step: q = M_reg p + (th/2) S_W^T S_W p on a 128 x 4 output tile -- p =
//                   r + beta p_{k-1} formed in the tile load and written for the own pixels, the
//                   half stencil (HBM stream of NH planes; the transposed half read at the
//                   neighbour, L1/L2 hits), the weighted NLTV part from m (as k_misr_normal),
//                   <p, q> and pi_0 into the CG slots (Alg.2 lines 3, 6-7)
//   k_asm_irr_u     per CG step: u at the positions (on a side stream beside k_asm_normal)
//   k_asm_irr_t     per CG step: t of every irregular row, <p, M_irr p> = sum t^2 / c_A
//   k_asm_irr_scatter  per CG step: T at the positions, T bil_k into q (RED.ADD, after the join)
#include "internal.h"
#include <climits>
#include <type_traits>

namespace lfsr {

template <int Z> struct AsmCfg {
  static constexpr int R = Z == 2 ? 2 : 3;            // Gaussian blur radius (A11)
  static constexpr int NP = 2 * R + 1;                // positions per axis of a row
  static constexpr int WRr = 2 * R + 2;               // regular row window (cells per axis)
  static constexpr int WR2 = WRr * WRr;
  static constexpr int WR2P = WR2 + 1;                // odd shared-memory stride of a row
  static constexpr int RS = WR2 + 4;                  // global row record: weights, base, pad (16 B aligned)
  static constexpr int RB = Z == 2 ? 8 : 4;           // k_asm_rows: LR rows per CTA (32 x RB threads)
  static constexpr int SR = WRr - 1;                  // stencil radius
  static constexpr int NSW = 2 * SR + 1;
  static constexpr int NH = (NSW * NSW + 1) / 2;      // stored half (incl. the centre)
  // setup kernel: 16 x 16 cells per CTA, rows of the footprint in chunks of CAP
  static constexpr int TA = 16, NTA = TA * TA;
  static constexpr int CAP = Z == 2 ? 288 : 160;
  static constexpr size_t kSmemStencil = (size_t)NH * NTA * 4 + (size_t)CAP * (WR2P + 2) * 4;
  // CG-step kernel: 128 x 8 output pixels, warp = row, lane = 4 pixels
  static constexpr int TH = 4, TW = 128;              // 4 warps (one output row each)
  static constexpr int PC = TW + 16;                  // tile columns [X0 - 8, X0 + TW + 8)
  static constexpr int PR = TH + 2 * SR, MR = TH + 4;
  static constexpr size_t kSmemNormal = (size_t)(PR * PC + 2 * MR * PC) * 4;
};

// half-window offset of coefficient h: h = dy * NSW + dx with dy = 0, dx in [0, SR] or dy in
// [1, SR], dx in [-SR, SR]
template <int NSW, int SR>
__host__ __device__ constexpr int hoff_dy(int h) { return (h + SR) / NSW; }
template <int NSW, int SR>
__host__ __device__ constexpr int hoff_dx(int h) { return h - hoff_dy<NSW, SR>(h) * NSW; }

__device__ __forceinline__ int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }   // floor, b > 0
__device__ __forceinline__ int cdiv(int a, int b) { return -fdiv(-a, b); }                            // ceil

// The bilinear sample of view k at HR position (Y, X), replicate-clamped (A12/A13); the same
// arithmetic in every kernel of this file so that the regular / irregular split is consistent.
struct Samp {
  int y0, x0, y1, x1;
  float fy, fx;
};
__device__ __forceinline__ Samp asm_sample(const Geom& G, const float* om, float drho, float dtau, int Y, int X) {
  // integer and fractional parts of the shift d = dtheta omega in fp32 at its own (small) magnitude,
  // the integer part added to the pixel index: absolute fp32 coordinates near 2048 would keep only
  // ~12 fraction bits.  clamp(z + d, 0, N - 1) (A12/A13) in index form: below 0 -> cell 0, weight 0;
  // at or past N - 1 -> cell N - 1, weight 0.
  const float o = __ldg(om + (size_t)Y * G.ps + X);
  const float dy = dtau * o, dx = drho * o;
  const float fdy = floorf(dy), fdx = floorf(dx);
  Samp s;
  s.y0 = Y + (int)fdy;
  s.x0 = X + (int)fdx;
  s.fy = dy - fdy;
  s.fx = dx - fdx;
  if (s.y0 < 0) { s.y0 = 0; s.fy = 0.f; }
  else if (s.y0 >= G.H - 1) { s.y0 = G.H - 1; s.fy = 0.f; }
  if (s.x0 < 0) { s.x0 = 0; s.fx = 0.f; }
  else if (s.x0 >= G.W - 1) { s.x0 = G.W - 1; s.fx = 0.f; }
  s.y1 = min(s.y0 + 1, G.H - 1);
  s.x1 = min(s.x0 + 1, G.W - 1);
  return s;
}

__device__ __forceinline__ const float* asm_omega(const Geom& G, const float* omega, int k) {
  return omega + (G.per_view ? (size_t)k * G.H * G.ps : 0);
}

// Cell bounding box of row (k, iy, ix); returns true when it is regular.
template <int Z>
__device__ __forceinline__ bool asm_row_bbox(const Geom& G, const float* om, float drho, float dtau, int iy, int ix,
                                             int& by, int& bx, int* ey = nullptr, int* ex = nullptr) {
  using C = AsmCfg<Z>;
  int y0 = 1 << 30, y1 = -(1 << 30), x0 = 1 << 30, x1 = -(1 << 30);
#pragma unroll
  for (int u = -C::R; u <= C::R; ++u) {
    const int Y = Z * iy + u;
    if (Y < 0 || Y >= G.H) continue;
#pragma unroll
    for (int v = -C::R; v <= C::R; ++v) {
      const int X = Z * ix + v;
      if (X < 0 || X >= G.W) continue;
      const Samp s = asm_sample(G, om, drho, dtau, Y, X);
      y0 = min(y0, s.y0);
      y1 = max(y1, s.y1);
      x0 = min(x0, s.x0);
      x1 = max(x1, s.x1);
    }
  }
  by = y0;
  bx = x0;
  if (ey) *ey = y1;
  if (ex) *ex = x1;
  return y1 - y0 < C::WRr && x1 - x0 < C::WRr;
}

// ---------------------------------------------------------------------------------------------
// setup 1: irregular rows -> compact list (k, i) + cell boxes
// ---------------------------------------------------------------------------------------------
template <int Z>
__global__ void __launch_bounds__(256) k_asm_rows(const Geom G, const Views V, const float* __restrict__ omega,
                                                  float* __restrict__ rows, unsigned* count, int2* __restrict__ list,
                                                  unsigned* __restrict__ pmask, int pmw) {
  using C = AsmCfg<Z>;
  constexpr int WRr = C::WRr, WR2 = C::WR2, RS = C::RS;
  __shared__ float sw[32 * C::RB * (WR2 + 1)];   // per-thread row window, odd stride
  const int lane = threadIdx.x, ix = blockIdx.x * 32 + lane, iy = blockIdx.y * C::RB + threadIdx.y, k = blockIdx.z;
  const int tid = threadIdx.y * 32 + lane;
  const bool in = ix < G.w && iy < G.h;
  bool irr = false;
  int by = 0, bx = 0;
  const float drho = V.off[k].x, dtau = V.off[k].y;
  const float* om = asm_omega(G, omega, k);
  if (in) irr = !asm_row_bbox<Z>(G, om, drho, dtau, iy, ix, by, bx);
  float* w = sw + tid * (WR2 + 1);
  if (in && !irr) {
#pragma unroll
    for (int e = 0; e < WR2; ++e) w[e] = 0.f;
#pragma unroll
    for (int u = -C::R; u <= C::R; ++u) {
      const int Y = Z * iy + u;
      if (Y < 0 || Y >= G.H) continue;
#pragma unroll
      for (int v = -C::R; v <= C::R; ++v) {
        const int X = Z * ix + v;
        if (X < 0 || X >= G.W) continue;
        const Samp s = asm_sample(G, om, drho, dtau, Y, X);
        const float gg = G.taps[u + C::R] * G.taps[v + C::R];
        const float a0 = gg * (1.f - s.fy), a1 = gg * s.fy;
        const int r0 = (s.y0 - by) * WRr, r1 = (s.y1 - by) * WRr, c0 = s.x0 - bx, c1 = s.x1 - bx;
        w[r0 + c0] += a0 * (1.f - s.fx);
        w[r0 + c1] += a0 * s.fx;
        w[r1 + c0] += a1 * (1.f - s.fx);
        w[r1 + c1] += a1 * s.fx;
      }
    }
  }
  if (in) {   // the record: WR2 weights, then the window base (y << 16 | x), INT_MIN when irregular
    float* rec = rows + (((size_t)k * G.h + iy) * G.w + ix) * RS;
    if (!irr) {
#pragma unroll
      for (int e = 0; e < WR2; e += 4) *reinterpret_cast<float4*>(rec + e) = make_float4(w[e], w[e + 1], w[e + 2], w[e + 3]);
    }
    reinterpret_cast<int*>(rec)[WR2] = irr ? INT_MIN : ((by << 16) | bx);
  }
  const unsigned b = __ballot_sync(0xffffffffu, irr);
  if (!b) return;
  unsigned base = 0;
  if (lane == 0) base = atomicAdd(count, (unsigned)__popc(b));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (!irr) return;
  list[base + __popc(b & ((1u << lane) - 1u))] = make_int2(k, (iy << 16) | ix);
  // the HR positions of the row's blur window (inside Omega) join the position set P_k
  for (int u = -C::R; u <= C::R; ++u) {
    const int Y = Z * iy + u;
    if (Y < 0 || Y >= G.H) continue;
    for (int v = -C::R; v <= C::R; ++v) {
      const int X = Z * ix + v;
      if (X < 0 || X >= G.W) continue;
      atomicOr(pmask + ((size_t)k * G.H + Y) * pmw + (X >> 5), 1u << (X & 31));
    }
  }
}

// setup 2: P_k as a compact list (k, Y << 16 | X) (warp ballots over the mask)
__global__ void __launch_bounds__(256) k_asm_plist(const Geom G, const unsigned* __restrict__ pmask, int pmw,
                                                   unsigned* count, uint2* __restrict__ plist) {
  const size_t nwords = (size_t)G.n_views * G.H * pmw;
  const int lane = threadIdx.x & 31;
  for (size_t w0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(size_t)31; w0 < nwords;
       w0 += (size_t)gridDim.x * blockDim.x) {
    // each lane holds one mask word; the warp walks the 32 words' bits together
    const size_t wi = w0 + lane;
    const unsigned word = wi < nwords ? __ldg(pmask + wi) : 0u;
    const size_t row = wi / pmw;   // k H + Y
    const int xw = (int)(wi - row * pmw) * 32;
    const int n = __popc(word);
    unsigned base = 0;
    int tot = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {   // inclusive scan of the counts
      const int t = __shfl_up_sync(0xffffffffu, tot, o);
      if (lane >= o) tot += t;
    }
    const int all = __shfl_sync(0xffffffffu, tot, 31);
    if (lane == 31 && all) base = atomicAdd(count, (unsigned)all);
    base = __shfl_sync(0xffffffffu, base, 31) + (unsigned)(tot - n);
    unsigned wb = word;
    while (wb) {
      const int bpos = __ffs(wb) - 1;
      wb &= wb - 1;
      const size_t k = row / G.H, Y = row - k * G.H;
      plist[base++] = make_uint2((unsigned)k, ((unsigned)Y << 16) | (unsigned)(xw + bpos));
    }
  }
}

template <int Z>
__global__ void __launch_bounds__(256, 2) k_asm_stencil(const Geom G, const Views V, const float* __restrict__ rows,
                                                     float om_max, float* __restrict__ st, int psS, size_t plane) {
  using C = AsmCfg<Z>;
  constexpr int WRr = C::WRr, WR2P = C::WR2P, NH = C::NH, NSW = C::NSW, NTA = C::NTA, CAP = C::CAP;
  extern __shared__ __align__(16) float sm_asm[];
  float* acc = sm_asm;                               // [NH][NTA]
  float* rw = acc + NH * NTA;                        // [CAP][WR2P] row windows
  int* rby = reinterpret_cast<int*>(rw + CAP * WR2P);   // [CAP] window base row (INT_MIN: irregular)
  int* rbx = rby + CAP;
  __shared__ int s_oy[2], s_ox[2];                   // min / max of (base - zeta i) over the chunk's regular rows
  const int tid = threadIdx.x;
  const int A0y = blockIdx.y * C::TA, A0x = blockIdx.x * C::TA;
  const int Ay = A0y + tid / C::TA, Ax = A0x + tid % C::TA;
  for (int h = 0; h < NH; ++h) acc[h * NTA + tid] = 0.f;

  for (int k = 0; k < G.n_views; ++k) {
    const float drho = V.off[k].x, dtau = V.off[k].y;
    const int sY = (int)ceilf(fabsf(dtau) * om_max), sX = (int)ceilf(fabsf(drho) * om_max);
    // LR rows whose cells can reach the tile: cells of row i lie in [zeta i - R - s, zeta i + R + s + 1]
    const int iy0 = max(0, cdiv(A0y - C::R - sY - 1, Z)), iy1 = min(G.h - 1, fdiv(A0y + C::TA - 1 + C::R + sY, Z));
    const int ix0 = max(0, cdiv(A0x - C::R - sX - 1, Z)), ix1 = min(G.w - 1, fdiv(A0x + C::TA - 1 + C::R + sX, Z));
    if (iy0 > iy1 || ix0 > ix1) continue;
    const int nx = ix1 - ix0 + 1;
    const int cx = min(nx, CAP), cy = max(1, CAP / cx);
    for (int cy0 = iy0; cy0 <= iy1; cy0 += cy) {
      for (int cx0 = ix0; cx0 <= ix1; cx0 += cx) {
        const int ny_c = min(cy, iy1 - cy0 + 1), nx_c = min(cx, ix1 - cx0 + 1);
        __syncthreads();   // the previous chunk's rows are consumed
        if (tid == 0) {
          s_oy[0] = s_ox[0] = 1 << 30;
          s_oy[1] = s_ox[1] = -(1 << 30);
        }
        __syncthreads();
        for (int r = tid; r < ny_c * nx_c; r += NTA) {   // the chunk's row records (k_asm_rows)
          const int iy = cy0 + r / nx_c, ix = cx0 + r % nx_c;
          const float* rec = rows + (((size_t)k * G.h + iy) * G.w + ix) * C::RS;
          const int pk = __ldg(reinterpret_cast<const int*>(rec) + C::WR2);
          if (pk == INT_MIN) {
            rby[r] = INT_MIN;
            continue;
          }
          const int by = pk >> 16, bx = pk & 0xffff;
          float* w = rw + r * WR2P;
#pragma unroll
          for (int e = 0; e < C::WR2; e += 4) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(rec + e));
            w[e] = t.x; w[e + 1] = t.y; w[e + 2] = t.z; w[e + 3] = t.w;
          }
          atomicMin(&s_oy[0], by - Z * iy);
          atomicMax(&s_oy[1], by - Z * iy);
          atomicMin(&s_ox[0], bx - Z * ix);
          atomicMax(&s_ox[1], bx - Z * ix);
          rby[r] = by;
          rbx[r] = bx;
        }
        __syncthreads();
        if (s_oy[0] > s_oy[1]) continue;   // no regular row in this chunk (uniform)
        // candidate rows of this thread's cell: zeta i + o <= A <= zeta i + o + WRr - 1, o in [omin, omax]
        const int jy0 = max(cy0, cdiv(Ay - s_oy[1] - WRr + 1, Z)), jy1 = min(cy0 + ny_c - 1, fdiv(Ay - s_oy[0], Z));
        const int jx0 = max(cx0, cdiv(Ax - s_ox[1] - WRr + 1, Z)), jx1 = min(cx0 + nx_c - 1, fdiv(Ax - s_ox[0], Z));
        for (int iy = jy0; iy <= jy1; ++iy) {
          for (int ix = jx0; ix <= jx1; ++ix) {
            const int r = (iy - cy0) * nx_c + (ix - cx0);
            const int by = rby[r];
            if (by == INT_MIN) continue;
            const int oy = Ay - by, ox = Ax - rbx[r];
            if ((unsigned)oy >= (unsigned)WRr || (unsigned)ox >= (unsigned)WRr) continue;
            const float* w = rw + r * WR2P;
            const float wa = w[oy * WRr + ox];
            if (wa == 0.f) continue;
            // coefficients of the half window: cells (jy, jx) of the row with (jy, jx) >= (oy, ox)
            // in row-major order, acc index (jy - oy) NSW + (jx - ox)
            float* ab = acc + (-(oy * NSW) - ox) * NTA + tid;
            for (int jy = oy; jy < WRr; ++jy) {
#pragma unroll
              for (int jx = 0; jx < WRr; ++jx) {
                if (jy == oy && jx < ox) continue;
                const int i2 = (jy * NSW + jx) * NTA;
                ab[i2] = fmaf(wa, w[jy * WRr + jx], ab[i2]);
              }
            }
          }
        }
      }
    }
  }
  if (Ay < G.H && Ax < G.W) {
    const size_t o = (size_t)(Ay + kAsmPad) * psS + Ax + kAsmPad;
    for (int h = 0; h < NH; ++h) st[h * plane + o] = G.cA * acc[h * NTA + tid];
  }
}

// ---------------------------------------------------------------------------------------------
// per CG step 1: t = c_A a . p for every irregular row
// ---------------------------------------------------------------------------------------------
struct AsmStepArgs {
  const float* r;        // CG residual (k >= 1)
  const float* p_prev;   // previous direction (k >= 2)
  const float* p_in;     // k = 0: the operator input
  int p_form;            // k_asm_irr_u: form p_k = r + beta p_{k-1} itself (runs beside k_asm_normal)
  float* p_out;          // k >= 1: p_k (own pixels)
  const float* m;        // NLTV weight map
  float* q;              // output (stored)
  Control* ctl;
  int cg_k;
  const float* omega;
  const unsigned* count; // [0] irregular rows, [1] positions of their windows (device)
  const int2* list;      // irregular rows (k, iy * w + ix)
  const uint2* plist;    // the positions P_k, (k, Y << 16 | X)
  float* tdense;         // [n_views][h][w] t of the irregular rows (0 elsewhere)
  float* udense;         // [n_views][H][W] u = W_k p at the positions of P_k
  const float* st;       // stencil planes
  int psS;
  size_t plane;
  float om_max;
};

__device__ __forceinline__ float asm_beta(const Control* ctl, int k) {
  return k >= 2 ? (float)(ctl->cur[S_PI + k - 1] / ctl->cur[S_PI + k - 2]) : 0.f;   // A2
}

// p_k (k >= 1: formed and written by k_asm_normal, which runs first) or the plain input (k = 0)
__device__ __forceinline__ const float* asm_pk(const AsmStepArgs& a) { return a.cg_k == 0 ? a.p_in : a.p_out; }

// per CG step 2: u = (W_k p)(z) at every position of P_k (p_k as k_asm_normal formed it)
__global__ void __launch_bounds__(256) k_asm_irr_u(const Geom G, const Views V, const AsmStepArgs a) {
  if (a.cg_k >= 2 && a.ctl->cur[S_STOP] != 0.0) return;   // CG stopped
  const float* pk = asm_pk(a);
  const unsigned n = a.count[1];
  // p_k at a cell: read (k_asm_normal formed it) or formed here exactly as its tile load does
  const bool form = a.p_form && a.cg_k >= 1;
  const float beta = asm_beta(a.ctl, a.cg_k);
  auto pat = [&](size_t i) -> float {
    if (!form) return __ldcg(pk + i);
    const float rv = __ldg(a.r + i);
    return a.cg_k >= 2 ? fmaf(beta, __ldg(a.p_prev + i), rv) : rv;
  };
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const uint2 kz = __ldg(a.plist + e);
    const int k = (int)kz.x, Y = (int)(kz.y >> 16), X = (int)(kz.y & 0xffffu);
    const Samp s = asm_sample(G, asm_omega(G, a.omega, k), V.off[k].x, V.off[k].y, Y, X);
    const size_t r0 = (size_t)s.y0 * G.ps, r1 = (size_t)s.y1 * G.ps;
    const float p00 = pat(r0 + s.x0), p01 = pat(r0 + s.x1);
    const float p10 = pat(r1 + s.x0), p11 = pat(r1 + s.x1);
    const float top = fmaf(s.fx, p01 - p00, p00), bot = fmaf(s.fx, p11 - p10, p10);
    a.udense[((size_t)k * G.H + Y) * G.W + X] = fmaf(s.fy, bot - top, top);
  }
}

// per CG step 3: t = c_A a . p = c_A sum_{u,v} g[u] g[v] u(zeta i + (u, v)) of every irregular row
// (one row per thread, its window values all in flight), and <p, M_irr p> = sum t^2 / c_A into the step's <p, q>
template <int Z>
__global__ void __launch_bounds__(256) k_asm_irr_t(const Geom G, const AsmStepArgs a) {
  using C = AsmCfg<Z>;
  constexpr int NP = C::NP;
  __shared__ double s_tt[8];
  if (a.cg_k >= 2 && a.ctl->cur[S_STOP] != 0.0) return;   // CG stopped
  const unsigned n = a.count[0];
  double tt = 0.0;
  // one row per thread, its NP x NP window values all in flight (positions outside Omega read 0:
  // the clamped index is multiplied by a zero tap)
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int2 ki = __ldg(a.list + e);
    const int k = ki.x, iy = ki.y >> 16, ix = ki.y & 0xffff;
    const float* uk = a.udense + (size_t)k * G.H * G.W;
    float vals[NP][NP];
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      const int Y = min(max(Z * iy + u - C::R, 0), G.H - 1);
#pragma unroll
      for (int v = 0; v < NP; ++v) {
        const int X = min(max(Z * ix + v - C::R, 0), G.W - 1);
        vals[u][v] = __ldcg(uk + (size_t)Y * G.W + X);
      }
    }
    float t = 0.f;
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      const int Y = Z * iy + u - C::R;
      float tr = 0.f;
#pragma unroll
      for (int v = 0; v < NP; ++v) {
        const int X = Z * ix + v - C::R;
        tr = fmaf((X >= 0 && X < G.W) ? G.taps[v] : 0.f, vals[u][v], tr);
      }
      t = fmaf((Y >= 0 && Y < G.H) ? G.taps[u] : 0.f, tr, t);
    }
    const float tv = G.cA * t;
    a.tdense[((size_t)k * G.h + iy) * G.w + ix] = tv;
    tt += (double)tv * t;
  }
  // one atomic per CTA (same-address double atomics serialise in L2)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, o);
  if ((threadIdx.x & 31) == 0) s_tt[threadIdx.x >> 5] = tt;
  __syncthreads();
  if (threadIdx.x == 0 && a.cg_k >= 1) {
    double sum = 0.0;
    for (int w = 0; w < 8; ++w) sum += s_tt[w];
    if (sum != 0.0) atomicAdd(&a.ctl->cur[S_PQ + a.cg_k], sum);
  }
}

// per CG step 4: T(z) = sum_{irregular i: z in win(i)} g g t_i at every position of P_k, scattered
// bilinearly into q (W_k^T; RED.ADD)
template <int Z>
__global__ void __launch_bounds__(256) k_asm_irr_scatter(const Geom G, const Views V, const AsmStepArgs a) {
  using C = AsmCfg<Z>;
  __shared__ float s_g[2 * C::R + 1];
  if (threadIdx.x <= 2 * C::R) s_g[threadIdx.x] = G.taps[threadIdx.x];
  __syncthreads();
  if (a.cg_k >= 2 && a.ctl->cur[S_STOP] != 0.0) return;   // CG stopped
  const unsigned n = a.count[1];
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const uint2 kz = __ldg(a.plist + e);
    const int k = (int)kz.x, Y = (int)(kz.y >> 16), X = (int)(kz.y & 0xffffu);
    // LR pixels whose window holds (Y, X): i = floor(Y / zeta) - 1 + j, j = 0..2 (u = Y - zeta i in
    // [-R, R] for at most three of them at zeta <= 4); taps from a per-phase table, 0 where u leaves
    // the window or i leaves the image -- a fixed 3 x 3 gather with no data-dependent trip counts
    const int cy = Y / Z, cx = X / Z;
    const float* tk = a.tdense + (size_t)k * G.h * G.w;
    float gyv[3], gxv[3];
    int ry[3], rx[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int iy = cy - 1 + j, ix = cx - 1 + j;
      const int uy = Y - Z * iy, ux = X - Z * ix;
      const float ty = s_g[min(max(uy + C::R, 0), 2 * C::R)], tx = s_g[min(max(ux + C::R, 0), 2 * C::R)];
      gyv[j] = (uy >= -C::R && uy <= C::R && iy >= 0 && iy < G.h) ? ty : 0.f;
      gxv[j] = (ux >= -C::R && ux <= C::R && ix >= 0 && ix < G.w) ? tx : 0.f;
      ry[j] = min(max(iy, 0), G.h - 1);
      rx[j] = min(max(ix, 0), G.w - 1);
    }
    float T = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const float* trow = tk + (size_t)ry[j] * G.w;
      const float tr = fmaf(gxv[0], __ldcg(trow + rx[0]), fmaf(gxv[1], __ldcg(trow + rx[1]), gxv[2] * __ldcg(trow + rx[2])));
      T = fmaf(gyv[j], tr, T);
    }
    if (T == 0.f) continue;
    const Samp s = asm_sample(G, asm_omega(G, a.omega, k), V.off[k].x, V.off[k].y, Y, X);
    const float a0 = T * (1.f - s.fy), a1 = T * s.fy;
    float* q0 = a.q + (size_t)s.y0 * G.ps;
    float* q1 = a.q + (size_t)s.y1 * G.ps;
    atomicAdd(q0 + s.x0, a0 * (1.f - s.fx));
    atomicAdd(q0 + s.x1, a0 * s.fx);
    atomicAdd(q1 + s.x0, a1 * (1.f - s.fx));
    atomicAdd(q1 + s.x1, a1 * s.fx);
  }
}

__device__ __forceinline__ double asm_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Stencil planes: the stored half, plane h = dy NSW + dx (dy = 0: dx in [0, SR]; dy in [1, SR]:
// dx in [-SR, SR]) holds M_reg[a][a + d_h] at pixel a; the other half is read at the neighbour
// (M[a][a - d] = M[a - d][a]).  Stored-full planes (a mirror pass at setup, one coalesced LDG.128
// per coefficient) measured slower: 30.2 vs 24.6 us per pass at C3.
//
#ifndef LFSR_ASM_MINB
#define LFSR_ASM_MINB 4
#endif
#ifndef LFSR_ASM_DY_UNROLL
#define LFSR_ASM_DY_UNROLL 1
#endif
constexpr int kAsmDyUnroll = LFSR_ASM_DY_UNROLL;   // development knobs (tools/build_variants.sh)
template <int Z>
__global__ void __launch_bounds__(128, LFSR_ASM_MINB) k_asm_normal(const Geom G, const Views V, const AsmStepArgs a) {
  using C = AsmCfg<Z>;
  constexpr int SR = C::SR, NSW = C::NSW, TH = C::TH, TW = C::TW, PC = C::PC, PR = C::PR, MR = C::MR, NT = TH * 32;
  constexpr int RAD = 2, CX = 8;   // NLTV radius (5 x 5 window); tile column offset (>= SR, mult. of 4)
  extern __shared__ __align__(16) float sm_an[];
  float* sp = sm_an;                 // p  rows [-SR, TH + SR), columns [X0 - CX, X0 + TW + CX)
  float* smm = sp + PR * PC;         // m^2 rows [-RAD, TH + RAD), same columns
  float* smp = smm + MR * PC;        // m^2 p
  __shared__ double red[TH * 2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Y0 = blockIdx.y * TH, X0 = blockIdx.x * TW;
  const int H = G.H, W = G.W, ps = G.ps;
  Control* ctl = a.ctl;
  if (a.cg_k >= 2 && ctl->cur[S_STOP] != 0.0) return;   // CG stopped
  const float beta = asm_beta(ctl, a.cg_k);
  double pi0 = 0.0, pq = 0.0;

  // ---- tile load: p = r + beta p_{k-1} (Alg.2 line 10, A2), zero outside Omega; own pixels -> p_out,
  // pi_0 = <r_0, r_0> at k = 1 (Alg.2 line 3).  Chunks of 4 columns ----
  const float* src1 = a.cg_k == 0 ? a.p_in : a.r;
  for (int c = tid; c < PR * (PC / 4); c += NT) {
    const int py = c / (PC / 4), cx = (c - py * (PC / 4)) * 4;
    const int gy = Y0 - SR + py, gx = X0 - CX + cx;
    float v[4];
    if (gy >= 0 && gy < H && gx >= 0 && gx + 3 < W) {
      const float4 r4 = __ldg(reinterpret_cast<const float4*>(src1 + (size_t)gy * ps + gx));
      v[0] = r4.x; v[1] = r4.y; v[2] = r4.z; v[3] = r4.w;
      if (a.cg_k >= 2) {
        const float4 q4 = __ldg(reinterpret_cast<const float4*>(a.p_prev + (size_t)gy * ps + gx));
        v[0] = fmaf(beta, q4.x, v[0]); v[1] = fmaf(beta, q4.y, v[1]);
        v[2] = fmaf(beta, q4.z, v[2]); v[3] = fmaf(beta, q4.w, v[3]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool in = gy >= 0 && gy < H && gx + e >= 0 && gx + e < W;
        const size_t gi = in ? (size_t)gy * ps + gx + e : 0;
        v[e] = in ? __ldg(src1 + gi) : 0.f;
        if (in && a.cg_k >= 2) v[e] = fmaf(beta, __ldg(a.p_prev + gi), v[e]);
      }
    }
    *reinterpret_cast<float4*>(sp + py * PC + cx) = make_float4(v[0], v[1], v[2], v[3]);
    if (a.cg_k >= 1 && py >= SR && py < SR + TH && cx >= CX && cx < CX + TW && gy < H) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (gx + e < W) {
          a.p_out[(size_t)gy * ps + gx + e] = v[e];
          if (a.cg_k == 1) pi0 += (double)v[e] * v[e];
        }
    }
  }
  __syncthreads();
  for (int c = tid; c < MR * PC; c += NT) {
    const int py = c / PC, px = c - py * PC;
    const int gy = Y0 - RAD + py, gx = X0 - CX + px;
    const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
    const float mv = in ? __ldg(a.m + (size_t)gy * ps + gx) : 0.f;
    const float mm = mv * mv;
    smm[c] = mm;
    smp[c] = mm * sp[(py + SR - RAD) * PC + px];
  }
  __syncthreads();

  const int ly = warp, Y = Y0 + ly, X = X0 + 4 * lane;
  if (Y < H) {
    // ---- data part: the half stencil, M[a][a + d] = st[h][a] for d in the stored half and
    // M[a][a - d] = st[h][a - d]; row dy by row dy (own term at (Y, X..X+3), transposed term at
    // (Y - dy, X - dx..X - dx + 3): two aligned LDG.128 and a compile-time select) ----
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const float* pl = a.st + (size_t)(Y + kAsmPad) * a.psS + X + kAsmPad;   // plane 0 (centre) at (Y, X)
    auto load_row = [&](float (&pv)[20], int row) {
      const float* prow = sp + row * PC + 4 * lane;
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const float4 t = *reinterpret_cast<const float4*>(prow + 4 * j);
        pv[4 * j] = t.x; pv[4 * j + 1] = t.y; pv[4 * j + 2] = t.z; pv[4 * j + 3] = t.w;
      }
    };
    // coefficients of pixels X - dx .. X - dx + 3 of plane row `src` (dx compile time after unrolling)
    auto load_shifted = [&](const float* src, int dx, float (&o)[4]) {
      const int m = (-dx) & 3;
      const float4 t0 = __ldg(reinterpret_cast<const float4*>(src - dx - m));
      if (m == 0) {
        o[0] = t0.x; o[1] = t0.y; o[2] = t0.z; o[3] = t0.w;
        return;
      }
      const float4 t1 = __ldg(reinterpret_cast<const float4*>(src - dx - m + 4));
      const float t[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] = t[m + e];
    };
    {   // dy = 0: the centre, then dx = 1..SR both ways
      float pv[20];
      load_row(pv, ly + SR);
      const float4 c0 = __ldg(reinterpret_cast<const float4*>(pl));
      acc[0] = c0.x * pv[CX]; acc[1] = c0.y * pv[CX + 1]; acc[2] = c0.z * pv[CX + 2]; acc[3] = c0.w * pv[CX + 3];
#pragma unroll
      for (int dx = 1; dx <= SR; ++dx) {
        const float* ph = pl + (size_t)dx * a.plane;
        const float4 cf = __ldg(reinterpret_cast<const float4*>(ph));
        float ct[4];
        load_shifted(ph, dx, ct);
        acc[0] = fmaf(cf.x, pv[CX + dx + 0], acc[0]);
        acc[1] = fmaf(cf.y, pv[CX + dx + 1], acc[1]);
        acc[2] = fmaf(cf.z, pv[CX + dx + 2], acc[2]);
        acc[3] = fmaf(cf.w, pv[CX + dx + 3], acc[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = fmaf(ct[e], pv[CX - dx + e], acc[e]);
      }
    }
#pragma unroll kAsmDyUnroll
    for (int dy = 1; dy <= SR; ++dy) {
      float pvo[20], pvt[20];
      load_row(pvo, ly + dy + SR);
      load_row(pvt, ly - dy + SR);
      const float* plh = pl + (size_t)(dy * NSW - SR) * a.plane;   // plane of d = (dy, -SR)
#pragma unroll
      for (int dxi = 0; dxi < NSW; ++dxi) {
        const int dx = dxi - SR;
        const float* ph = plh + (size_t)dxi * a.plane;
        const float4 cf = __ldg(reinterpret_cast<const float4*>(ph));
        float ct[4];
        load_shifted(ph - (ptrdiff_t)dy * a.psS, dx, ct);
        acc[0] = fmaf(cf.x, pvo[CX + dx + 0], acc[0]);
        acc[1] = fmaf(cf.y, pvo[CX + dx + 1], acc[1]);
        acc[2] = fmaf(cf.z, pvo[CX + dx + 2], acc[2]);
        acc[3] = fmaf(cf.w, pvo[CX + dx + 3], acc[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = fmaf(ct[e], pvt[CX - dx + e], acc[e]);
      }
    }
    // ---- weighted NLTV part (A10): sum_d (p(z) - p(z+d)) (w_d^2 m(z)^2 + w_{-d}^2 m(z+d)^2), z + d in
    // Omega; A = sum w_d^2 p(z+d), B = sum w_{-d}^2 m^2(z+d), C = sum w_{-d}^2 m^2 p(z+d) ----
    float A_[4] = {0.f, 0.f, 0.f, 0.f}, B_[4] = {0.f, 0.f, 0.f, 0.f}, C_[4] = {0.f, 0.f, 0.f, 0.f};
    float W2z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int dyn = -RAD; dyn <= RAD; ++dyn) {
      float pv[12], mv[12], cv[12];   // columns CX + 4 lane - 4 .. + 7
      const float* pr = sp + (ly + dyn + SR) * PC + 4 * lane + 4;
      const float* mr = smm + (ly + dyn + RAD) * PC + 4 * lane + 4;
      const float* cr = smp + (ly + dyn + RAD) * PC + 4 * lane + 4;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const float4 t0 = *reinterpret_cast<const float4*>(pr + 4 * j);
        const float4 t1 = *reinterpret_cast<const float4*>(mr + 4 * j);
        const float4 t2 = *reinterpret_cast<const float4*>(cr + 4 * j);
        pv[4 * j] = t0.x; pv[4 * j + 1] = t0.y; pv[4 * j + 2] = t0.z; pv[4 * j + 3] = t0.w;
        mv[4 * j] = t1.x; mv[4 * j + 1] = t1.y; mv[4 * j + 2] = t1.z; mv[4 * j + 3] = t1.w;
        cv[4 * j] = t2.x; cv[4 * j + 1] = t2.y; cv[4 * j + 2] = t2.z; cv[4 * j + 3] = t2.w;
      }
      const bool rin = Y + dyn >= 0 && Y + dyn < H;
#pragma unroll
      for (int dxn = -RAD; dxn <= RAD; ++dxn) {
        if (dyn == 0 && dxn == 0) continue;
        const int lin = (dyn + RAD) * (2 * RAD + 1) + (dxn + RAD);
        const int d = lin > 12 ? lin - 1 : lin;   // A9 order, centre skipped
        const float w2 = G.wd[d] * G.wd[d], w2f = G.wd[23 - d] * G.wd[23 - d];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = 4 + e + dxn;   // column CX + 4 lane + e + dxn in the 12-value window
          A_[e] = fmaf(w2, pv[c], A_[e]);
          B_[e] = fmaf(w2f, mv[c], B_[e]);
          C_[e] = fmaf(w2f, cv[c], C_[e]);
          W2z[e] += (rin && X + e + dxn >= 0 && X + e + dxn < W) ? w2 : 0.f;
        }
      }
    }
    const float* pc = sp + (ly + SR) * PC + CX + 4 * lane;
    const float* mc = smm + (ly + RAD) * PC + CX + 4 * lane;
    float qz[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float pz = pc[e], mz = mc[e];
      qz[e] = acc[e] + G.cS * (pz * fmaf(mz, W2z[e], B_[e]) - fmaf(mz, A_[e], C_[e]));
      if (a.cg_k >= 1 && X + e < W) pq += (double)pz * qz[e];
    }
    float* qo = a.q + (size_t)Y * ps + X;
    if (X + 3 < W) {
      *reinterpret_cast<float4*>(qo) = make_float4(qz[0], qz[1], qz[2], qz[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (X + e < W) qo[e] = qz[e];
    }
  }
  if (a.cg_k >= 1) {
    pq = asm_warp_sum(pq);
    pi0 = asm_warp_sum(pi0);
    if (lane == 0) {
      red[warp * 2] = pq;
      red[warp * 2 + 1] = pi0;
    }
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int w = 0; w < TH; ++w) {
        s0 += red[w * 2];
        s1 += red[w * 2 + 1];
      }
      if (s0 != 0.0) atomicAdd(&ctl->cur[S_PQ + a.cg_k], s0);
      if (s1 != 0.0) atomicAdd(&ctl->cur[S_PI], s1);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------------
int asm_row_floats(int scale) {   // floats per row record
  switch (scale) {
    case 2: return AsmCfg<2>::RS;
    case 3: return AsmCfg<3>::RS;
    case 4: return AsmCfg<4>::RS;
    default: return 0;
  }
}

int asm_plane_count(int scale) {   // stored half of the stencil window (centre first)
  switch (scale) {
    case 2: return AsmCfg<2>::NH;
    case 3: return AsmCfg<3>::NH;
    case 4: return AsmCfg<4>::NH;
    default: return 0;
  }
}

template <int Z>
static cudaError_t prep_asm() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_asm_stencil<Z>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)AsmCfg<Z>::kSmemStencil)))
    return e;
  return cudaFuncSetAttribute(k_asm_normal<Z>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)AsmCfg<Z>::kSmemNormal);
}

cudaError_t prepare_asm_kernels() {
  cudaError_t e;
  if ((e = prep_asm<2>()) || (e = prep_asm<3>()) || (e = prep_asm<4>())) return e;
  return cudaSuccess;
}

template <int Z>
static void asm_build_z(const Geom& G, const Views& V, const AsmBuf& B, float om_max, cudaStream_t st) {
  using C = AsmCfg<Z>;
  dim3 gc((G.w + 31) / 32, (G.h + C::RB - 1) / C::RB, G.n_views);
  k_asm_rows<Z><<<gc, dim3(32, C::RB), 0, st>>>(G, V, B.omega, B.rows, B.count, B.list, B.pmask, B.pmw);
  k_asm_plist<<<1184, 256, 0, st>>>(G, B.pmask, B.pmw, B.count + 1, B.plist);
  dim3 gs((G.W + C::TA - 1) / C::TA, (G.H + C::TA - 1) / C::TA);
  k_asm_stencil<Z><<<gs, C::NTA, C::kSmemStencil, st>>>(G, V, B.rows, om_max, B.st, B.psS, B.plane);
}

cudaError_t launch_asm_build(const Geom& G, const Views& V, const AsmBuf& B, float om_max, cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(B.count, 0, 2 * sizeof(unsigned), st)) ||
      (e = cudaMemsetAsync(B.pmask, 0, (size_t)G.n_views * G.H * B.pmw * sizeof(unsigned), st)) ||
      (e = cudaMemsetAsync(B.tdense, 0, (size_t)G.n_views * G.h * G.w * sizeof(float), st)))
    return e;
  switch (G.scale) {
    case 2: asm_build_z<2>(G, V, B, om_max, st); break;
    case 3: asm_build_z<3>(G, V, B, om_max, st); break;
    case 4: asm_build_z<4>(G, V, B, om_max, st); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int Z>
static void asm_step_z(const Geom& G, const Views& V, const AsmStepArgs& a, bool irr, int num_sms, cudaStream_t st,
                       cudaEvent_t mid, const AsmFork& fk) {
  using C = AsmCfg<Z>;
  dim3 g((G.W + C::TW - 1) / C::TW, (G.H + C::TH - 1) / C::TH);
  if (irr && fk.side) {
    // the irregular rows' u and t (p_k formed on the fly) on the side stream, concurrent with the
    // latency-bound stencil kernel; the scatter into q after both
    AsmStepArgs af = a;
    af.p_form = 1;
    cudaEventRecord(fk.fork, st);
    cudaStreamWaitEvent(fk.side, fk.fork, 0);
    k_asm_irr_u<<<num_sms * 8, 256, 0, fk.side>>>(G, V, af);
    k_asm_irr_t<Z><<<num_sms * 4, 256, 0, fk.side>>>(G, af);
    cudaEventRecord(fk.join, fk.side);
    k_asm_normal<Z><<<g, C::TH * 32, C::kSmemNormal, st>>>(G, V, a);
    cudaStreamWaitEvent(st, fk.join, 0);
    k_asm_irr_scatter<Z><<<num_sms * 8, 256, 0, st>>>(G, V, a);
    return;
  }
  k_asm_normal<Z><<<g, C::TH * 32, C::kSmemNormal, st>>>(G, V, a);
  if (mid) cudaEventRecordWithFlags(mid, st, cudaEventRecordExternal);   // profiling split
  if (irr) {
    k_asm_irr_u<<<num_sms * 8, 256, 0, st>>>(G, V, a);
    k_asm_irr_t<Z><<<num_sms * 4, 256, 0, st>>>(G, a);
    k_asm_irr_scatter<Z><<<num_sms * 8, 256, 0, st>>>(G, V, a);
  }
}

cudaError_t launch_asm_step(const Geom& G, const Views& V, const AsmBuf& B, const AsmStep& s, bool irr, int num_sms,
                            cudaStream_t st, cudaEvent_t mid, const AsmFork& fk) {
  AsmStepArgs a{};
  a.r = s.r;
  a.p_prev = s.p_prev;
  a.p_in = s.p_in;
  a.p_out = s.p_out;
  a.m = s.m;
  a.q = s.q;
  a.ctl = s.ctl;
  a.cg_k = s.cg_k;
  a.omega = B.omega;
  a.count = B.count;
  a.list = B.list;
  a.plist = B.plist;
  a.tdense = B.tdense;
  a.udense = B.udense;
  a.st = B.st;
  a.psS = B.psS;
  a.plane = B.plane;
  a.om_max = B.om_max;
  switch (G.scale) {
    case 2: asm_step_z<2>(G, V, a, irr, num_sms, st, mid, fk); break;
    case 3: asm_step_z<3>(G, V, a, irr, num_sms, st, mid, fk); break;
    case 4: asm_step_z<4>(G, V, a, irr, num_sms, st, mid, fk); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace lfsr
