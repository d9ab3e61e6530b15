// tile_impl.cuh — the fused observation-operator tile kernel of liblfsr (v3), included by
// tile_z2.cu / tile_z3.cu / tile_z4.cu (one translation unit per zeta, compiled in parallel).
//
// One CTA owns a tile = a band of BL LR rows x a strip of LX LR columns, and a
// group of views.  Every warp of the CTA takes whole views (round robin) and
// streams the tile's "E region" (the HR positions whose blurred warped value
// reaches an own LR pixel) row by row, lane = LR column, each lane holding the
// zeta HR columns under its LR column:
//   W_k    bilinear gather at z + dtheta_k * omega(z) from the shared input tile
//          (replicate-clamped coordinate)                       P:L580-583, A12/A13
//   B, D   Gaussian blur evaluated at LR positions only: horizontal taps by warp
//          shuffles, vertical taps in a register ring (decimation is free) P:L577-579
//   epilogue per LR pixel: (WZ) e = A_k x - y_k, clamp-form prox + scaled dual
//          (Alg.1 lines 4-8, A5/A6) -> rho; (NORMAL) rho = c_A A_k p;
//          (GRAD, gd) rho = l1 sgn(e) + 2 l2 e (A30); (J, gd-ls trial) cost terms only
//   D^T B^T polyphase adjoint blur (register ring + shuffles)           A11/A14
//   W_k^T  exact bilinear scatter into a shared int32 fixed-point accumulator
//          (native ATOMS.ADD, order-independent -> deterministic per CTA)  A12
// No barrier inside the view loop.  Then the weighted NLTV term in gather form
// for the own pixels (view group g takes every G-th own row, warps
// pull rows from a shared counter), and one RED.ADD flush of accumulator + NLTV
// term (tile + halo) to global so neighbouring tiles and view groups sum.
// Arithmetic is packed FP32 (FFMA2/FADD2/FMUL2) over a lane's column pairs; the
// tiling (BL, view groups, warps) is chosen per problem by tile_kernels.cu /
// capi.cu.
// Compile-time variants: PV reads each view's own disparity map omega_k
// (A34), P2 replaces the separable Gaussian by a user blur kernel (view_pass2d, A36), PM
// stops after the epilogue and leaves the adjoint to the paper's backward warp
// (k_paper_gather, A37).
//
// Fixed-point scale: every CTA bounds |t| (the blurred adjoint value of one
// source) by tb (c_A max|p| for NORMAL; l2 (max|x| + max|y|) + (th/2) l1 3/th for
// WZ; l1 + 2 l2 (max|x| + max|y|) for GRAD; max|x| carries sum|k| with a user kernel)
// and the accumulated weight per cell by the splat density max_z sum_k
// (W_k^T 1)(z) (computed once at setup), and picks 2^s with |w t 2^s| < 2^21 and
// |acc| < 2^30: the per-contribution rounding is <= 2^-22 tb.
#pragma once
#include "tile_cfg.h"
#include <cfloat>
#include <cmath>


namespace lfsr {

#ifdef LFSR_CTA_TIMING   // development: per-CTA phase timestamps of the NORMAL launches (tools/cta_timing.py)
static __device__ unsigned long long g_cta_t[4096][4];   // per translation unit (zeta)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CTA_T(i) do { if (MODE == MODE_NORMAL && threadIdx.x == 0 && blockIdx.x < 4096) g_cta_t[blockIdx.x][i] = gtimer(); } while (0)
#else
#define CTA_T(i) do { } while (0)
#endif

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV doubles, then one atomicAdd per value into dst[slot[i]].
template <int NV>
__device__ __forceinline__ void block_reduce_add(double (&v)[NV], double* red, double* dst,
                                                 const int (&slot)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
    for (int w = 0; w < nw; ++w) s += red[w * NV + threadIdx.x];
    if (s != 0.0) atomicAdd(dst + slot[threadIdx.x], s);
  }
}

// Two-word fixed-point accumulation: v (already scaled by 2^s,
// |v| < 2^22) is split into its rounded integer part q1 and the residual
// r = v - q1 in [-1/2, 1/2], which goes to a second accumulator in units of 2^-15
// (|q2| <= 2^14, so 2^17 contributions per cell cannot overflow).  Both rounding
// steps use the 1.5*2^23 magic (FADD + IADD, no XU-pipe conversion); integer
// atomics are native (ATOMS.ADD) and associative, so the result does not depend
// on the order of the atomics.  Resolution 2^-(s+15) ~ 2^-37 of the per-CTA bound.
constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
constexpr int kMagicBits = 0x4B400000;
constexpr int kLoBits = 15;

// phase-split shared index of tile-local (py, px): columns of equal px % Z are
// contiguous, so lanes zeta columns apart hit consecutive banks.
template <int Z>
__device__ __forceinline__ int pidx(int py, int px, int PW, int PWZ) {
  const unsigned ux = (unsigned)px;
  return py * PW + (int)((ux % Z) * PWZ + ux / Z);
}

// Packed FP32 (sm_100 FFMA2/FADD2/FMUL2): two lanes of fp32 arithmetic per
// issue slot.  Each packed op rounds every component exactly like its scalar
// counterpart (x - y is computed as fma(y, -1, x), which rounds once), so the
// pairing changes the instruction count, not the results.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2s(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 sub2(float2 x, float2 y) { return __ffma2_rn(y, f2s(-1.f), x); }
// (taps[u], taps[u+1]) straight from the parameter block (u is a compile-time index)
__device__ __forceinline__ float2 tap2(const Geom& G, int u) { return (u & 1) ? G.tpo[u >> 1] : G.tpe[u >> 1]; }

// Two-word fixed-point accumulation of a pair of values into the cells i and j
// (see kLoBits): the conversions run packed, the four ATOMS.ADD stay scalar.
__device__ __forceinline__ void acc_add2(int* hi, int lo_off, int i, int j, float2 v) {
  const float2 t = __fadd2_rn(v, f2s(kMagic));
  const float2 r = sub2(v, __fadd2_rn(t, f2s(-kMagic)));
  const float2 u = __ffma2_rn(r, f2s((float)(1 << kLoBits)), f2s(kMagic));
  atomicAdd(hi + i, __float_as_int(t.x) - kMagicBits);
  atomicAdd(hi + j, __float_as_int(t.y) - kMagicBits);
  atomicAdd(hi + lo_off + i, __float_as_int(u.x) - kMagicBits);
  atomicAdd(hi + lo_off + j, __float_as_int(u.y) - kMagicBits);
}

// Tile-local arithmetic of one CTA.  INT: every E column of the tile lies inside
// the image, so no column masks are applied (samples never need clamping: the
// input tile is replicate-padded).
// A lane's zeta E columns are processed in pairs (s, s+1) with packed FP32; an
// odd zeta leaves one scalar column.
// Edge-tile routing data (TC::DUMMY): Yp = Yrow * ymul + yadd per column pair sends
// an E position outside the image to the zero rows at PHd.  Empty otherwise.
template <bool D, int NP>
struct YRoute {
  float2 ymul[NP + 1], yadd[NP + 1];
  float PHd;
};
template <int NP>
struct YRoute<false, NP> {};

template <int Z, bool INT, int RB>
struct Tile : YRoute<!INT && TCR<Z, RB>::DUMMY, Z / 2> {
  static constexpr int NP = Z / 2;     // column pairs per lane
  static constexpr bool kInt = INT;
  const float* P;
  int* ACC;
  const float* OM;
  int PW, PWZ, PY0, PX0, YE0, XE0, H, W;
  int PS;             // HR row pitch of the global disparity maps
  float tscale;
  int lo;             // offset of the residual accumulator from ACC (ints)
  unsigned koff;      // Z = 2: folded magic offsets of cells_bits()
  unsigned colmask;   // bit s: the lane's E column Z*lane+s is a real image column (used when !INT)

  bool rows_in;       // every row of the E region lies inside the image

  // row er of the E region lies inside the image (warp uniform)
  __device__ __forceinline__ bool row_in(int er) const {
    return INT || rows_in || (unsigned)(YE0 + er) < (unsigned)H;
  }

  // floor and fraction without the XU pipe: s + 1.5*2^23 rounded toward -inf is
  // 1.5*2^23 + floor(s) exactly (|s| < 2^22), so its bit pattern is the integer.
  // The coordinates are tile-local (origin PY0/PX0, |s| < ~300), so the fraction
  // keeps ~2^-15 absolute precision whatever the image size (an absolute HR
  // coordinate near 2048 would leave only 2^-12).
  // axis2 returns the raw bit patterns kMagicBits + floor(s).
  __device__ __forceinline__ static void axis2(float2 s, int& n0, int& n1, float2& f) {
    const float2 r = __fadd2_rd(s, f2s(kMagic));
    n0 = __float_as_int(r.x);
    n1 = __float_as_int(r.y);
    f = sub2(s, __fadd2_rn(r, f2s(-kMagic)));
  }
  __device__ __forceinline__ static void axis(float s, int& n, float& f) {
    const float r = __fadd_rd(s, kMagic);
    n = __float_as_int(r) - kMagicBits;
    f = s - (r - kMagic);
  }
  // phase-split indices of the top-left / top-right source cells of tile cell (iy, ix)
  __device__ __forceinline__ void cells(int iy, int ix, int& i00, int& i01) const {
    const unsigned ux = (unsigned)ix, ph = ux % Z, q = ux / Z;
    i00 = iy * PW + (int)(ph * PWZ + q);
    i01 = (ph == Z - 1) ? i00 - (Z - 1) * PWZ + 1 : i00 + PWZ;
  }
  // The same from the raw bits b = kMagicBits + n.  kMagicBits is even, so for
  // zeta = 2 the phase is b % 2 and the offsets fold into koff (mod 2^32); zeta = 4
  // would fold the same way but measured longer code, zeta = 3 cannot.
  __device__ __forceinline__ void cells_bits(int by, int bx, int& i00, int& i01) const {
    if constexpr (Z == 2) {
      const unsigned ux = (unsigned)bx, ph = ux % Z, q = ux / Z;
      i00 = (int)((unsigned)by * (unsigned)PW + ph * (unsigned)PWZ + q + koff);
      i01 = (ph == Z - 1) ? i00 - (Z - 1) * PWZ + 1 : i00 + PWZ;
    } else {
      cells(by - kMagicBits, bx - kMagicBits, i00, i01);
    }
  }

  // Source cells and bilinear fractions of the E positions (Yf, Xf) and
  // (Yf, Xf + 1) (A12/A13).  No clamping: the input tile holds the
  // image replicate-padded, and a bilinear sample of the replicate-padded image
  // equals the sample at the clamped coordinate; the adjoint scatters into the
  // padding and phase 4 folds it back onto the edge cells (the transpose of the
  // padding).
  __device__ __forceinline__ void sample2(float2 Yp, float Xf, float2 om, float drho, float dtau,
                                          int (&i00)[2], int (&i01)[2], float2& a, float2& b) const {
    const float2 sy = __ffma2_rn(f2s(dtau), om, Yp);
    const float2 sx = __ffma2_rn(f2s(drho), om, f2(Xf, Xf + 1.f));
    int by0, by1, bx0, bx1;
    axis2(sy, by0, by1, a);
    axis2(sx, bx0, bx1, b);
    cells_bits(by0, bx0, i00[0], i01[0]);
    cells_bits(by1, bx1, i00[1], i01[1]);
  }
  __device__ __forceinline__ void sample(float Yf, float Xf, float om, float drho, float dtau,
                                         int& i00, int& i01, float& a, float& b) const {
    int iy, ix;
    axis(fmaf(dtau, om, Yf), iy, a);
    axis(fmaf(drho, om, Xf), ix, b);
    cells(iy, ix, i00, i01);
  }

  // E positions outside the image carry zero (blur zero padding, A11): rows by a
  // warp-uniform test (row_in), columns by the per-lane mask (col_in).
  __device__ __forceinline__ bool col_in(int s) const { return INT || TCR<Z, RB>::DUMMY || ((colmask >> s) & 1u); }
  __device__ __forceinline__ float2 colsel(float2 v, int s) const {
    return (INT || TCR<Z, RB>::DUMMY) ? v : f2(col_in(s) ? v.x : 0.f, col_in(s + 1) ? v.y : 0.f);
  }
  static constexpr bool kDummy = !INT && TCR<Z, RB>::DUMMY;
  // E row of the samples: the row itself, or the dummy zero rows when it is outside the image
  __device__ __forceinline__ float yrow(int er) const {
    const float Yf = (float)(YE0 - PY0 + er);
    if constexpr (kDummy) return (unsigned)(YE0 + er) >= (unsigned)H ? this->PHd : Yf;
    return Yf;
  }
  __device__ __forceinline__ float yone(float Yrow) const {   // the odd column of an odd zeta
    if constexpr (kDummy) return fmaf(Yrow, this->ymul[NP].x, this->yadd[NP].x);
    return Yrow;
  }
  __device__ __forceinline__ float2 ypair(float Yrow, int k) const {
    if constexpr (kDummy) return __ffma2_rn(f2s(Yrow), this->ymul[k], this->yadd[k]);
    return f2s(Yrow);
  }

  // Disparity of the lane's zeta E positions on E row er: the shared map staged in
  // shared memory (omk == nullptr), or view k's own map omega_k read from global memory
  // (per-view mode, A34; zero outside the image like the staged map).
  __device__ __forceinline__ void load_om(int er, int lane, float (&om)[Z], const float* omk) const {
    if (omk) {
      const int Yg = YE0 + er, X0g = XE0 + Z * lane;
      const bool rin = (unsigned)Yg < (unsigned)H;
      const float* src = omk + (size_t)(rin ? Yg : 0) * PS;
#pragma unroll
      for (int s = 0; s < Z; ++s) om[s] = (rin && (unsigned)(X0g + s) < (unsigned)W) ? __ldg(src + X0g + s) : 0.f;
      return;
    }
    const float* src = OM + er * TCR<Z, RB>::ECOL + Z * lane;
    if constexpr (Z == 2) {
      float2 v = *reinterpret_cast<const float2*>(src);
      om[0] = v.x; om[1] = v.y;
    } else if constexpr (Z == 4) {
      float4 v = *reinterpret_cast<const float4*>(src);
      om[0] = v.x; om[1] = v.y; om[2] = v.z; om[3] = v.w;
    } else {
#pragma unroll
      for (int s = 0; s < Z; ++s) om[s] = src[s];
    }
  }

  // W_k at the lane's zeta E positions of row er, then the row's values at E columns
  // zeta*lane + v, v < NTAP (the horizontal blur window of the lane's LR column):
  // own positions, the rest from the next lanes by shuffles.
  // omr: the row's disparities already in registers (per-view ring of view_pass), or nullptr.
  __device__ __forceinline__ void fwd_vals(int er, int lane, float drho, float dtau, const float* omk,
                                           float (&val)[TCR<Z, RB>::NTAP], const float* omr = nullptr) const {
    constexpr int NTAP = TCR<Z, RB>::NTAP;
    float om[Z], wp[Z];
    if (omr) {
#pragma unroll
      for (int s = 0; s < Z; ++s) om[s] = omr[s];
    } else {
      load_om(er, lane, om, omk);
    }
    const float Yf = yrow(er);
    const float X0 = (float)(XE0 - PX0 + Z * lane);
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int s = 2 * k;
      int i00[2], i01[2];
      float2 a, b;
      sample2(ypair(Yf, k), X0 + (float)s, f2(om[s], om[s + 1]), drho, dtau, i00, i01, a, b);
      const float2 p00 = f2(P[i00[0]], P[i00[1]]), p01 = f2(P[i01[0]], P[i01[1]]);
      const float2 p10 = f2(P[i00[0] + PW], P[i00[1] + PW]), p11 = f2(P[i01[0] + PW], P[i01[1] + PW]);
      const float2 top = __ffma2_rn(b, sub2(p01, p00), p00), bot = __ffma2_rn(b, sub2(p11, p10), p10);
      const float2 v = colsel(__ffma2_rn(a, sub2(bot, top), top), s);
      wp[s] = v.x;
      wp[s + 1] = v.y;
    }
    if constexpr (Z & 1) {
      constexpr int s = Z - 1;
      int i00, i01;
      float a, b;
      sample(yone(Yf), X0 + (float)s, om[s], drho, dtau, i00, i01, a, b);
      const float p00 = P[i00], p01 = P[i01], p10 = P[i00 + PW], p11 = P[i01 + PW];
      const float top = fmaf(b, p01 - p00, p00), bot = fmaf(b, p11 - p10, p10);
      wp[s] = col_in(s) ? fmaf(a, bot - top, top) : 0.f;
    }
#pragma unroll
    for (int v = 0; v < NTAP; ++v)
      val[v] = (v < Z) ? wp[v % Z] : __shfl_down_sync(0xffffffffu, wp[v % Z], v / Z);
  }

  // W_k then the horizontal blur taps at this lane's LR column, for E row er.
  __device__ __forceinline__ float fwd_row(int er, int lane, float drho, float dtau, const float* omk,
                                          const Geom& G, const float* omr = nullptr) const {
    constexpr int NTAP = TCR<Z, RB>::NTAP;
    if (!kDummy && !row_in(er)) return 0.f;    // blur zero padding (A11), warp uniform
    float val[NTAP];
    fwd_vals(er, lane, drho, dtau, omk, val, omr);
    float2 h2 = f2s(0.f);
#pragma unroll
    for (int v = 0; v + 1 < NTAP; v += 2) h2 = __ffma2_rn(tap2(G, v), f2(val[v], val[v + 1]), h2);
    float h = h2.x + h2.y;
    if constexpr (NTAP & 1) h = fmaf(G.taps[NTAP - 1], val[NTAP - 1], h);
    return h;
  }

  // Horizontal adjoint blur of the row's LR-column values t1b and the exact bilinear
  // scatter (W_k^T) of the lane's zeta positions into the fixed-point accumulator.
  // A position's four weights go out as two (row, row + 1) pairs; adjacent positions
  // whose source columns coincide (smooth disparity) are merged first: zeta + 1 pairs
  // instead of 2 zeta (per lane and boundary; the all-or-nothing warp test it replaces
  // cost 4 % at C4/C5).
  __device__ __forceinline__ void adj_row(int er, int lane, float t1b, float drho, float dtau, const float* omk,
                                          const Geom& G, const float* omr = nullptr) const {
    constexpr int NJ = 2 * TCR<Z, RB>::R / Z + 1;
    constexpr int R2 = 2 * TCR<Z, RB>::R;
    if (!kDummy && !row_in(er)) return;        // E positions outside the image carry no adjoint (A11)
    float tv[NJ];
    tv[0] = t1b;
#pragma unroll
    for (int j = 1; j < NJ; ++j) {
      const float v = __shfl_up_sync(0xffffffffu, t1b, j);
      tv[j] = lane >= j ? v : 0.f;
    }
    float tt[Z];   // the adjoint blur value of each of the lane's zeta positions
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int s = 2 * k;
      float2 t = f2s(0.f);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        if (Z * j + s + 1 <= R2) t = __ffma2_rn(tap2(G, Z * j + s), f2s(tv[j]), t);
        else if (Z * j + s <= R2) t.x = fmaf(G.taps[Z * j + s], tv[j], t.x);
      }
      tt[s] = t.x;
      tt[s + 1] = t.y;
    }
    if constexpr (Z & 1) {
      constexpr int s = Z - 1;
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (Z * j + s <= R2) t = fmaf(G.taps[Z * j + s], tv[j], t);
      tt[s] = t;
    }
    scatter(er, lane, tt, drho, dtau, omk, omr);
  }

  // The exact bilinear scatter (W_k^T) of the adjoint blur values tt of the lane's zeta
  // positions of E row er into the fixed-point accumulator (the row must be inside the
  // image or a routed dummy row).
  __device__ __forceinline__ void scatter(int er, int lane, const float (&tt)[Z], float drho, float dtau,
                                          const float* omk, const float* omr = nullptr) const {
    float om[Z];
    if (omr) {
#pragma unroll
      for (int s = 0; s < Z; ++s) om[s] = omr[s];
    } else {
      load_om(er, lane, om, omk);
    }
    const float Yf = yrow(er);
    const float X0 = (float)(XE0 - PX0 + Z * lane);
    int i00[Z], i01[Z];
    float2 w0[Z], w1[Z];   // (row, row + 1) weights times t on the left / right source column
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int s = 2 * k;
      const float2 t = f2(tt[s], tt[s + 1]);
      int c0[2], c1[2];
      float2 a, b;
      sample2(ypair(Yf, k), X0 + (float)s, f2(om[s], om[s + 1]), drho, dtau, c0, c1, a, b);
      i00[s] = c0[0]; i01[s] = c1[0]; i00[s + 1] = c0[1]; i01[s + 1] = c1[1];
      const float2 ts = __fmul2_rn(colsel(t, s), f2s(tscale));
      // per position: (ts (1 - a), ts a) = the two source rows' shares, split by b into
      // columns (scalar here: the packed form would need the pairs transposed)
      const float ta0 = ts.x * a.x, ta1 = ts.y * a.y;
      const float2 q0 = f2(ts.x - ta0, ta0), q1 = f2(ts.y - ta1, ta1);
      w1[s] = __fmul2_rn(q0, f2s(b.x));
      w0[s] = sub2(q0, w1[s]);
      w1[s + 1] = __fmul2_rn(q1, f2s(b.y));
      w0[s + 1] = sub2(q1, w1[s + 1]);
    }
    if constexpr (Z & 1) {
      constexpr int s = Z - 1;
      const float t = tt[s];
      float a, b;
      sample(yone(Yf), X0 + (float)s, om[s], drho, dtau, i00[s], i01[s], a, b);
      const float ts = col_in(s) ? t * tscale : 0.f;
      const float ta = ts * a;
      const float2 q = f2(ts - ta, ta);
      w1[s] = __fmul2_rn(q, f2s(b));
      w0[s] = sub2(q, w1[s]);
    }
    // per lane and per column boundary: merge when the two positions share the column
    // (i00[s] == i01[s-1]); the lanes that do not, add the left position's right column
    // separately (a warp-uniform skip when no lane needs it)
    acc_add2(ACC, lo, i00[0], i00[0] + PW, w0[0]);
#pragma unroll
    for (int s = 1; s < Z; ++s) {
      const bool adj = i00[s] == i01[s - 1];
      acc_add2(ACC, lo, i00[s], i00[s] + PW, adj ? __fadd2_rn(w0[s], w1[s - 1]) : w0[s]);
      if (__any_sync(0xffffffffu, !adj) && !adj) acc_add2(ACC, lo, i01[s - 1], i01[s - 1] + PW, w1[s - 1]);
    }
    acc_add2(ACC, lo, i01[Z - 1], i01[Z - 1] + PW, w1[Z - 1]);
  }
};

// Weighted NLTV term of one own pixel z (readings A9/A10):
//   NORMAL: sum_d Delta_d^T (W_d^2 Delta_d p)(z) and its <p, .> share (W_d = w_d m)
//   WZ:     z/w steps of the NLTV rows (Alg.1 lines 5-8, clamp form A5/A6) for the
//           pairs (z, z+d), written to the other w_S buffer, and
//           sum_d Delta_d^T (W_d f_d)(z) with the backward neighbour's f_d
//           recomputed from the old duals (gather form: no atomics, no race).
// RAD > 0: offsets unrolled at compile time (paper's 5x5 window: RAD = 2).
__device__ __forceinline__ float sgnf(float v) { return v > 0.f ? 1.f : (v < 0.f ? -1.f : 0.f); }   // A30

struct NltvCtx {
  const float* P;
  const float* M;
  const float* __restrict__ wSr;
  float* __restrict__ wSw;
  size_t plane;
  int PW, PWZ, MW, H, W, ps;
  float ith;
};

template <int Z, int MODE, bool CHECK, int RAD, int RB>
__device__ __forceinline__ float nltv_pixel(const NltvCtx& c, const Geom& G, int Y, int X, int py, int px, int mi,
                                            size_t gi, double& pq, double& reg, double& res) {
  const float xz = c.P[pidx<Z>(py, px, c.PW, c.PWZ)];
  const float mz = c.M[mi];
  float acc = 0.f;
  float fpq = 0.f, freg = 0.f, fres = 0.f;   // this pixel's reduction terms (<= s_d each), fp32
  // the m tile pitch is a compile-time constant on the unrolled (RAD > 0) path
  const int MW = RAD > 0 ? TCR<Z, RB>::TX + 2 * RAD : c.MW;
  auto one = [&](int d, int dy, int dx) {
    const float wd = G.wd[d];
    const bool fin = !CHECK || ((Y + dy >= 0) && (Y + dy < c.H) && (X + dx >= 0) && (X + dx < c.W));
    const bool bin = !CHECK || ((Y - dy >= 0) && (Y - dy < c.H) && (X - dx >= 0) && (X - dx < c.W));
    const float xf = c.P[pidx<Z>(py + dy, px + dx, c.PW, c.PWZ)];   // in the tile even when outside Omega
    const float xb = c.P[pidx<Z>(py - dy, px - dx, c.PW, c.PWZ)];
    const float mb = c.M[mi - dy * MW - dx];
    if (MODE == MODE_GRAD || MODE == MODE_J) {
      // G_d = W_d (.) Delta_d x and the subgradient S_w^T sgn(G) in gather form (A30)
      const float wz = wd * mz;
      const float g = fin ? wz * (xz - xf) : 0.f;
      freg += fabsf(g);
      if (MODE == MODE_GRAD) {
        acc = fmaf(wz, sgnf(g), acc);
        if (bin) {
          const float wb = wd * mb;
          acc = fmaf(-wb, sgnf(wb * (xb - xz)), acc);
        }
      }
    } else if (MODE == MODE_NORMAL) {
      const float wz = wd * mz, wb = wd * mb;
      const float dp = xz - xf;
      const float f2 = fin ? wz * wz : 0.f;
      acc = fmaf(f2, dp, acc);
      fpq = fmaf(f2 * dp, dp, fpq);
      const float b2 = bin ? wb * wb : 0.f;
      acc = fmaf(-b2, xb - xz, acc);
    } else {
      const size_t pl = (size_t)d * c.plane;
      const float wz = wd * mz;
      const float g = fin ? wz * (xz - xf) : 0.f;             // W_d (.) Delta_d x
      const float wso = __ldg(c.wSr + pl + gi);
      const float wn = fminf(fmaxf(g + wso, -c.ith), c.ith);
      c.wSw[pl + gi] = wn;
      freg += fabsf(g);
      fres = fmaf(wn - wso, wn - wso, fres);
      if (fin) acc = fmaf(wz, 2.f * wn - wso, acc);
      if (bin) {
        const float wb = wd * mb;
        const float wsb = __ldg(c.wSr + pl + gi - (size_t)dy * c.ps - dx);
        const float wnb = fminf(fmaxf(fmaf(wb, xb - xz, wsb), -c.ith), c.ith);
        acc = fmaf(-wb, 2.f * wnb - wsb, acc);
      }
    }
  };
  if constexpr (RAD > 0) {
#pragma unroll
    for (int dy = -RAD; dy <= RAD; ++dy) {
#pragma unroll
      for (int dx = -RAD; dx <= RAD; ++dx) {
        if (dy == 0 && dx == 0) continue;
        const int lin = (dy + RAD) * (2 * RAD + 1) + (dx + RAD);
        const int d = lin > (2 * RAD + 1) * RAD + RAD ? lin - 1 : lin;   // row-major order, centre skipped (A9)
        one(d, dy, dx);
      }
    }
  } else {
    for (int d = 0; d < G.s_d; ++d) one(d, G.ody[d], G.odx[d]);
  }
  if (MODE == MODE_NORMAL) pq += (double)fpq;
  if (MODE == MODE_WZ) {
    reg += (double)freg;
    res += (double)fres;
  }
  if (MODE == MODE_GRAD || MODE == MODE_J) reg += (double)freg;
  return acc;
}

// Phase 2 of k_tile: every warp streams whole views through the tile (see header).
// NV views are processed interleaved row by row (independent dependency chains
// for the scheduler); the last odd view of a warp takes the NV = 1 path.
// Per-LR-pixel step after the forward operator value a = A_k x (i, j), returning the
// value rho whose adjoint the pass accumulates (own LR pixels only).
template <int MODE>
__device__ __forceinline__ float lr_epilogue(float a, float y_cur, float wa_cur, size_t lg, const Geom& G,
                                             const TileIO& io, float& fa, float& fb, float& fc) {
  const float lam1 = G.lambda1, lam2 = G.lambda2, ith = G.inv_theta;
  float rho = 0.f;
  if (MODE == MODE_A) {
    io.out_lr[lg] = a;
  } else if (MODE == MODE_NORMAL) {
    rho = G.cA * a;
    fa = fmaf(a, a, fa);                                // <p, c_A A^T A p> = c_A |A p|^2
  } else if (MODE == MODE_WZ) {
    const float e_ = a - y_cur;                         // e = A_k x - y_k (Alg.1 line 4)
    const float wa = wa_cur;
    const float u = lam1 * e_ + wa;                     // u = F x - b' + w (line 5)
    const float wn = fminf(fmaxf(u, -ith), ith);        // w+ = u - prox(u) = clamp (A5/A6)
    const float f = 2.f * wn - wa;                      // f = 2w^n - w^{n-1} (line 8)
    rho = lam2 * e_ + G.cS * lam1 * f;                  // A^T a + (th/2) F^T f, data rows
    io.wA[lg] = wn;
    fa += fabsf(e_);
    fb = fmaf(e_, e_, fb);
    fc = fmaf(wn - wa, wn - wa, fc);
  } else if (MODE == MODE_GRAD || MODE == MODE_J) {
    const float e_ = a - y_cur;                         // e = A_k x - y_k
    if (MODE == MODE_GRAD) rho = fmaf(2.f * lam2, e_, lam1 * sgnf(e_));   // l1 sgn(e) + 2 l2 e (A30)
    fa += fabsf(e_);
    fb = fmaf(e_, e_, fb);
  }
  return rho;
}

template <int MODE>
__device__ __forceinline__ void pass_reductions(const Geom& G, float fa, float fb, float fc, double& red_a,
                                                double& red_b, double& red_c) {
  if (MODE == MODE_NORMAL) red_a += (double)G.cA * (double)fa;
  if (MODE == MODE_GRAD || MODE == MODE_J) {
    red_a += (double)fa;
    red_b += (double)fb;
  }
  if (MODE == MODE_WZ) {
    red_a += (double)fa;
    red_b += (double)fb;
    red_c += (double)fc;
  }
}

// PM (paper-mode adjoint, A37): the pass stops after the epilogue and writes rho to
// io.rho_out; k_paper_gather applies the backward warp afterwards.
template <int Z, int MODE, bool INT, int NV, bool PV, bool PM, int RB>
__device__ __forceinline__ void view_pass(const Tile<Z, INT, RB>& t, const Geom& G, const Views& V, const TileIO& io,
                                          const int (&ks)[NV], int lane, int i0, int j0, int BL, double& red_a,
                                          double& red_b, double& red_c) {
  using C = TCR<Z, RB>;
  constexpr int LX = C::LX, NTAP = C::NTAP, KEEP = C::KEEP;
  constexpr bool kFwd = (MODE != MODE_AT);
  constexpr bool kAdj = (MODE != MODE_A && MODE != MODE_J);
  constexpr bool kY = (MODE == MODE_WZ || MODE == MODE_GRAD || MODE == MODE_J);   // reads y_k
  const int j = j0 + lane;
  const bool col_ok = lane < LX && j < G.w;
  constexpr bool kAdjW = kAdj && !PM;   // the exact adjoint scatter of this pass
  float drho[NV], dtau[NV], fr[NV][NTAP], br[NV][NTAP], y_nx[NV], wa_nx[NV];
  const float* omk[NV];   // per-view disparity map omega_k (A34), nullptr: the shared map in shared memory
  // PV: each E row's omega_k values are read from global memory once, when the forward pass
  // reaches the row, and kept (ring position u = E row zeta*li + u, like fr) until its adjoint
  constexpr int NOR = PV ? NTAP : 1;
  float omr[NV][NOR][Z];
  size_t lrow0[NV];
  float fa = 0.f, fb = 0.f, fc = 0.f;   // this pass's partial sums (<= BL * NV terms per lane), fp32
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    drho[v] = V.off[ks[v]].x;
    dtau[v] = V.off[ks[v]].y;
    omk[v] = PV ? io.omega + (size_t)ks[v] * G.H * G.ps : nullptr;   // compile-time nullptr: shared map
#pragma unroll
    for (int u = 0; u < NTAP; ++u) { fr[v][u] = 0.f; br[v][u] = 0.f; }
    lrow0[v] = ((size_t)ks[v] * G.h) * G.lps + j;
    y_nx[v] = 0.f;
    wa_nx[v] = 0.f;
    // software prefetch of the next LR row's observation and dual (WZ)
    if (kY && col_ok && i0 < G.h) {
      y_nx[v] = io.y[lrow0[v] + (size_t)i0 * G.lps];
      if (MODE == MODE_WZ) wa_nx[v] = io.wA[lrow0[v] + (size_t)i0 * G.lps];
    }
  }
  if (kFwd) {
#pragma unroll
    for (int u = 0; u < KEEP; ++u)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if constexpr (PV) {
          t.load_om(u, lane, omr[v][u], omk[v]);
          fr[v][u] = t.fwd_row(u, lane, drho[v], dtau[v], omk[v], G, omr[v][u]);
        } else {
          fr[v][u] = t.fwd_row(u, lane, drho[v], dtau[v], omk[v], G);
        }
      }
  }
  for (int li = 0; li < BL; ++li) {
    const int i = i0 + li;
    const bool ok = col_ok && i < G.h;
    float rho[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const size_t lg = lrow0[v] + (size_t)i * G.lps;
      const float y_cur = y_nx[v], wa_cur = wa_nx[v];
      if (kY && col_ok && li + 1 < BL && i + 1 < G.h) {
        y_nx[v] = io.y[lg + G.lps];
        if (MODE == MODE_WZ) wa_nx[v] = io.wA[lg + G.lps];
      }
      rho[v] = 0.f;
      if (kFwd) {
#pragma unroll
        for (int u = 0; u < Z; ++u) {
          if constexpr (PV) {
            t.load_om(Z * li + KEEP + u, lane, omr[v][KEEP + u], omk[v]);
            fr[v][KEEP + u] = t.fwd_row(Z * li + KEEP + u, lane, drho[v], dtau[v], omk[v], G, omr[v][KEEP + u]);
          } else {
            fr[v][KEEP + u] = t.fwd_row(Z * li + KEEP + u, lane, drho[v], dtau[v], omk[v], G);
          }
        }
        float2 a2 = f2s(0.f);                                            // A_k x at LR pixel (i, j)
#pragma unroll
        for (int u = 0; u + 1 < NTAP; u += 2) a2 = __ffma2_rn(tap2(G, u), f2(fr[v][u], fr[v][u + 1]), a2);
        float a = a2.x + a2.y;
        if constexpr (NTAP & 1) a = fmaf(G.taps[NTAP - 1], fr[v][NTAP - 1], a);
        if (ok) rho[v] = lr_epilogue<MODE>(a, y_cur, wa_cur, lg, G, io, fa, fb, fc);
        if (PM && ok) io.rho_out[lg] = rho[v];
#pragma unroll
        for (int u = 0; u < KEEP; ++u) fr[v][u] = fr[v][u + Z];
      } else {
        rho[v] = ok ? io.in_lr[lg] : 0.f;
      }
    }
    if (kAdjW) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
#pragma unroll
        for (int u = 0; u + 1 < NTAP; u += 2) {                                          // vertical adjoint
          const float2 b2 = __ffma2_rn(tap2(G, u), f2s(rho[v]), f2(br[v][u], br[v][u + 1]));
          br[v][u] = b2.x;
          br[v][u + 1] = b2.y;
        }
        if constexpr (NTAP & 1) br[v][NTAP - 1] = fmaf(G.taps[NTAP - 1], rho[v], br[v][NTAP - 1]);
#pragma unroll
        for (int u = 0; u < Z; ++u)
          t.adj_row(Z * li + u, lane, br[v][u], drho[v], dtau[v], omk[v], G, (PV && kFwd) ? omr[v][u] : nullptr);
        if constexpr (PV && kFwd) {
#pragma unroll
          for (int u = 0; u < KEEP; ++u)
#pragma unroll
            for (int s = 0; s < Z; ++s) omr[v][u][s] = omr[v][u + Z][s];
        }
#pragma unroll
        for (int u = 0; u < NTAP; ++u) br[v][u] = (u < KEEP) ? br[v][u + Z] : 0.f;
      }
    }
  }
  if (kAdjW) {
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int u = 0; u < KEEP; ++u)
        t.adj_row(Z * BL + u, lane, br[v][u], drho[v], dtau[v], omk[v], G, (PV && kFwd) ? omr[v][u] : nullptr);
  }
  pass_reductions<MODE>(G, fa, fb, fc, red_a, red_b, red_c);
}

// The same pass with a user (non-separable) blur kernel (A36), kernel
// psf2[a][b] in E-offset order.  Forward: every E row's window values (fwd_vals) feed the
// Q pending LR rows it lies under with that kernel row (sliding accumulators instead of
// the separable code's ring of horizontally filtered rows).  Adjoint: each lane keeps the
// rho of its own LR column for the last Q LR rows; a finished E row forms, per kernel
// column b, the vertical partial sum over those rows, and the partials of the LR columns to
// the left (the Q columns an E column receives from) arrive by warp shuffles -- Q registers
// of history instead of Q x Q (kernels up to 15 x 15 without spills).
template <int Z, int MODE, bool INT, int RB>
__device__ __forceinline__ void view_pass2d(const Tile<Z, INT, RB>& t, const Geom& G, const Views& V, const TileIO& io,
                                            int k, int lane, int i0, int j0, int BL, double& red_a, double& red_b,
                                            double& red_c) {
  using C = TCR<Z, RB>;
  constexpr int LX = C::LX, NTAP = C::NTAP, KEEP = C::KEEP, R2 = 2 * C::R;
  constexpr int Q = R2 / Z + 1;      // LR rows one E row lies under (and LR columns one E column)
  constexpr bool kFwd = (MODE != MODE_AT);
  constexpr bool kAdj = (MODE != MODE_A && MODE != MODE_J);
  constexpr bool kY = (MODE == MODE_WZ || MODE == MODE_GRAD || MODE == MODE_J);
  const int j = j0 + lane;
  const bool col_ok = lane < LX && j < G.w;
  const float drho = V.off[k].x, dtau = V.off[k].y;
  const size_t lrow0 = ((size_t)k * G.h) * G.lps + j;
  float acc[Q], rh[Q];
#pragma unroll
  for (int d = 0; d < Q; ++d) {
    acc[d] = 0.f;
    rh[d] = 0.f;
  }
  float fa = 0.f, fb = 0.f, fc = 0.f;
  float y_nx = 0.f, wa_nx = 0.f;
  if (kY && col_ok && i0 < G.h) {
    y_nx = io.y[lrow0 + (size_t)i0 * G.lps];
    if (MODE == MODE_WZ) wa_nx = io.wA[lrow0 + (size_t)i0 * G.lps];
  }
  // E row er sits at offset p below the top of the current LR row's window
  auto feed = [&](int er, int p) {
    if (!t.kDummy && !t.row_in(er)) return;          // zero padding (A36)
    float val[NTAP];
    t.fwd_vals(er, lane, drho, dtau, nullptr, val);
#pragma unroll
    for (int d = 0; d < Q; ++d) {
      const int a = p - Z * d;
      if (a < 0 || a > R2) continue;
      float h = acc[d];
#pragma unroll
      for (int b = 0; b < NTAP; ++b) h = fmaf(G.psf2[a][b], val[b], h);
      acc[d] = h;
    }
  };
  // finished E row er at offset uu below the top of the newest LR row in the history
  auto emit = [&](int er, int uu) {
    if (!t.kDummy && !t.row_in(er)) return;
    float tt[Z];
#pragma unroll
    for (int s = 0; s < Z; ++s) tt[s] = 0.f;
#pragma unroll
    for (int jj = 0; jj < Q; ++jj) {
#pragma unroll
      for (int s = 0; s < Z; ++s) {
        const int b = Z * jj + s;
        if (b > R2) continue;
        float h = 0.f;   // column (lane - jj)'s vertical partial for kernel column b
#pragma unroll
        for (int d = 0; d < Q; ++d) {
          const int a = Z * d + uu;
          if (a <= R2) h = fmaf(G.psf2[a][b], rh[d], h);
        }
        if (jj == 0) {
          tt[s] += h;
        } else {
          const float v = __shfl_up_sync(0xffffffffu, h, jj);
          tt[s] += lane >= jj ? v : 0.f;
        }
      }
    }
    t.scatter(er, lane, tt, drho, dtau, nullptr);
  };
  if (kFwd) {
#pragma unroll
    for (int u = 0; u < KEEP; ++u) feed(u, u);
  }
  for (int li = 0; li < BL; ++li) {
    const int i = i0 + li;
    const bool ok = col_ok && i < G.h;
    const size_t lg = lrow0 + (size_t)i * G.lps;
    const float y_cur = y_nx, wa_cur = wa_nx;
    if (kY && col_ok && li + 1 < BL && i + 1 < G.h) {
      y_nx = io.y[lg + G.lps];
      if (MODE == MODE_WZ) wa_nx = io.wA[lg + G.lps];
    }
    float rho = 0.f;
    if (kFwd) {
#pragma unroll
      for (int u = 0; u < Z; ++u) feed(Z * li + KEEP + u, KEEP + u);
      const float a = acc[0];                                   // A_k x at LR pixel (i, j)
#pragma unroll
      for (int d = 0; d + 1 < Q; ++d) acc[d] = acc[d + 1];
      acc[Q - 1] = 0.f;
      if (ok) rho = lr_epilogue<MODE>(a, y_cur, wa_cur, lg, G, io, fa, fb, fc);
    } else {
      rho = ok ? io.in_lr[lg] : 0.f;
    }
    if (kAdj) {
#pragma unroll
      for (int d = Q - 1; d > 0; --d) rh[d] = rh[d - 1];
      rh[0] = rho;
#pragma unroll
      for (int u = 0; u < Z; ++u) emit(Z * li + u, u);
    }
  }
  if (kAdj) {
#pragma unroll
    for (int u = 0; u < KEEP; ++u) emit(Z * BL + u, Z + u);
  }
  pass_reductions<MODE>(G, fa, fb, fc, red_a, red_b, red_c);
}

template <int Z, int MODE, bool INT, bool PV, bool P2, bool PM, int RB>
__device__ __forceinline__ void views(const Tile<Z, INT, RB>& t, const Geom& G, const Views& V, const TileGeom& T,
                                      const TileIO& io, int grp, int lane, int warp, int NW, int i0, int j0, int BL,
                                      double& red_a, double& red_b, double& red_c) {
  const int kbeg = grp * T.vpg;
  const int kend = min(G.n_views, kbeg + T.vpg);
  for (int k = kbeg + warp; k < kend; k += NW) {
    const int ks[1] = {k};
    if constexpr (P2) view_pass2d<Z, MODE, INT, RB>(t, G, V, io, k, lane, i0, j0, BL, red_a, red_b, red_c);
    else view_pass<Z, MODE, INT, 1, PV, PM, RB>(t, G, V, io, ks, lane, i0, j0, BL, red_a, red_b, red_c);
  }
}

// FIXBL: the tile height is the compile-time default TCR<Z, RB>::BL (the launcher picks this
// instantiation whenever T.BL equals it: constant loop bounds, ~1.5 % faster at C3).
// PV: per-view disparity maps omega_k read from global memory (A34); a compile-time
// switch because even a warp-uniform runtime test cost the shared-map path ~12 %.
// P2: user (non-separable) blur kernel (A36, view_pass2d).
// PM: paper-mode adjoint (A37): no scatter, rho to io.rho_out (k_paper_gather follows).
// RB: blur radius of the instance (the Gaussian's R(zeta), or kPsfBigR for large user kernels).
template <int Z, int MODE, bool FIXBL, bool PV, bool P2, bool PM, int RB = TileCfg<Z>::R>
__global__ void __launch_bounds__(LaunchCfgR<Z, MODE, RB>::MAXW * 32, LaunchCfgR<Z, MODE, RB>::MINB)
k_tile(const Geom G, const Views V, const TileGeom T, const TileIO io) {
  using C = TCR<Z, RB>;
  constexpr int R = C::R, LX = C::LX, TX = C::TX, ECOL = C::ECOL;
  const int BL = FIXBL ? C::BL : T.BL, TY = Z * BL, EY = Z * BL + C::KEEP;
  constexpr bool kFwd = (MODE != MODE_AT);
  constexpr bool kAdj = (MODE != MODE_A && MODE != MODE_J);
  constexpr bool kWeights = (MODE == MODE_WZ || MODE == MODE_GRAD);   // m from x in the tile (A16, A31)

  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  const int ntiles = T.ntl ? T.ntl : T.ntYl * T.ntX;  // tiles of this strip (all tiles with one rank),
  const int tile = T.ntl ? T.tlist[blockIdx.x % ntiles] : blockIdx.x % ntiles;   // or the MISR border tiles
  const int grp = blockIdx.x / ntiles;
  const int ti = T.tY0 + tile / T.ntX, tj = tile % T.ntX;
  const int i0 = ti * BL, j0 = tj * LX;          // LR origin of the tile
  const int Y0 = i0 * Z, X0 = j0 * Z;             // HR origin of the own pixels
  const int YE0 = Y0 - R, XE0 = X0 - R;           // E-region origin
  const int PY0 = YE0 - T.SYe - 1, PX0 = XE0 - T.SXe - 1;  // input-tile origin (+1 spare, see axis())
  const int PH = T.PH, PW = T.PW, PWn = ECOL + 2 * T.SXe + 2;
  const int H = G.H, W = G.W, ps = G.ps;
  Control* ctl = io.ctl;
  if (MODE == MODE_NORMAL && (io.cg_k >= 2 || io.cgcg_step >= 1) && ctl->cur[S_STOP] != 0.0) return;  // CG stopped
  CTA_T(0);
  // gd-ls trial t runs only while no earlier trial met the Armijo condition (A32); every
  // CTA reads the same fp64 sums, so all take the same decision
  float ls_beta = 0.f;
  if (MODE == MODE_J) {
    const double* cur = ctl->cur;
    const double J0 = (double)G.lambda1 * cur[S_L1] + (double)G.lambda2 * cur[S_L2] + cur[S_REG];
    for (int t = 0; t < io.ls_t; ++t) {
      const double et = ldexp((double)io.eta0, -t);
      const double* jt = cur + S_TJ + 3 * t;
      const double Jt = (double)G.lambda1 * jt[0] + (double)G.lambda2 * jt[1] + jt[2];
      if (Jt <= J0 - (double)io.armijo_c * et * cur[S_GN]) return;
    }
    ls_beta = -ldexpf(io.eta0, -io.ls_t);
  }

  float* P = smem;                                           // PH*PW  input tile (phase split)
  const int PHA = PH + (C::DUMMY ? 2 : 0);                   // + 2 zero rows (TC::DUMMY, Tile::yrow)
  int* ACC = reinterpret_cast<int*>(P + PHA * PW);           // 2*PHA*PW fixed-point accumulator (hi, lo)
  const int LO = PHA * PW;
  float* OM = P + 3 * PHA * PW;                              // EY*ECOL disparity on the E region
  float* M = OM + EY * ECOL;                                 // MH*MW  weight map, own + radius
  float* NL = M + T.MH * T.MW;                               // TY*TX  NLTV term of the own pixels
  const size_t red_off = ((size_t)(NL - smem) + (size_t)TY * TX + 1) & ~(size_t)1;   // 8-byte aligned
  double* RED = reinterpret_cast<double*>(smem + red_off);
  __shared__ float s_max;
  __shared__ float s_scale[2];
  __shared__ int s_nl_next;

  const int PWZ = T.PWZ;

  // ---- phase 1: input tile (+ CG direction update), disparity, m -----------
  double pi0_part = 0.0;
  float beta = 0.f, pmax = 0.f;
  if (MODE == MODE_NORMAL && io.cg_k >= 2) {
    double pim1 = ctl->cur[S_PI + io.cg_k - 1], pim2 = ctl->cur[S_PI + io.cg_k - 2];
    beta = (float)(pim1 / pim2);    // Alg.2 line 10 (reading A2): p_k = r_k + beta p_{k-1}
  }
  if (MODE == MODE_J) beta = ls_beta;   // trial point x - eta_t g
  const bool two_in = (MODE == MODE_NORMAL && io.cg_k >= 2) || MODE == MODE_J;
  if (tid == 0) {
    s_max = 0.f;
    s_nl_next = 0;
  }
  {
    // 4 independent loads in flight per thread (the tile load is latency bound)
    constexpr int U = 4;
    const int n = PH * PWn;
    for (int e0 = tid; e0 < n; e0 += U * NT) {
      float v[U], v2[U];
      size_t gi[U];
      bool own[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * NT;
        const int py = e / PWn, px = e - py * PWn;
        const int gy = PY0 + py, gx = PX0 + px;
        // replicate padding outside the image (see Tile::sample)
        const int cy = min(max(gy, 0), H - 1), cx = min(max(gx, 0), W - 1);
        gi[u] = (size_t)cy * ps + cx;
        own[u] = e < n && gy == cy && gx == cx && gy >= Y0 && gy < Y0 + TY && gx >= X0 && gx < X0 + TX;
        v[u] = (kFwd && e < n) ? __ldg(io.in_hr + gi[u]) : 0.f;
        v2[u] = (two_in && e < n) ? __ldg(io.in_hr2 + gi[u]) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * NT;
        if (e >= n) break;
        float val = v[u];
        if (MODE == MODE_NORMAL && io.cg_k >= 1) {
          if (io.cg_k == 1) {
            if (own[u] && grp == 0) pi0_part += (double)val * val;   // pi_0 = <r_0, r_0> (Alg.2 line 3)
          } else {
            val = val + beta * v2[u];
          }
          if (own[u] && grp == 0 && io.p_out) io.p_out[gi[u]] = val;
        }
        if (MODE == MODE_J) val = fmaf(beta, v2[u], val);   // the same rounding as k_gd_update
        pmax = fmaxf(pmax, fabsf(val));
        const int py = e / PWn, px = e - py * PWn;
        const int i = pidx<Z>(py, px, PW, PWZ);
        if (kFwd) P[i] = val;
        if (kAdj) { ACC[i] = 0; ACC[LO + i] = 0; }
      }
    }
  }
  if (kAdj && PW > PWn) {  // phase-split padding cells of the accumulator
    for (int e = tid; e < PH * (PW - PWn); e += NT) {
      const int py = e / (PW - PWn), px = PWn + e - py * (PW - PWn);
      const int i = pidx<Z>(py, px, PW, PWZ);
      ACC[i] = 0;
      ACC[LO + i] = 0;
    }
  }
  if (!PV)
  for (int e = tid; e < EY * ECOL; e += NT) {   // 0 outside the image (the dummy rows rely on it)
    const int er = e / ECOL, c = e - er * ECOL;
    const int Y = YE0 + er, X = XE0 + c;
    OM[e] = (Y >= 0 && Y < H && X >= 0 && X < W) ? io.omega[(size_t)Y * ps + X] : 0.f;
  }
  if (C::DUMMY)   // the two zero rows past the input tile (and their accumulator cells)
    for (int e = tid; e < 2 * PW; e += NT) {
      P[PH * PW + e] = 0.f;
      ACC[PH * PW + e] = 0;
      ACC[LO + PH * PW + e] = 0;
    }
  const int rr = G.radius, MW = T.MW;
  if ((MODE == MODE_NORMAL && io.do_nltv) || MODE == MODE_J) {   // frozen m (J: of this gd iteration)
    for (int e = tid; e < T.MH * MW; e += NT) {
      const int my = e / MW, mx = e - my * MW;
      const int gy = Y0 - rr + my, gx = X0 - rr + mx;
      M[e] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? io.m[(size_t)gy * ps + gx] : 0.f;
    }
  }
  // block max of |input| -> fixed-point scale
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
  __syncthreads();
  if (lane == 0 && pmax > 0.f) atomicMax(reinterpret_cast<unsigned*>(&s_max), __float_as_uint(pmax));
  __syncthreads();
  if (tid == 0) {
    float tb = 0.f;
    if (MODE == MODE_NORMAL) tb = G.cA * (P2 ? G.ksum * s_max : s_max);
    if (MODE == MODE_WZ) tb = G.lambda2 * ((P2 ? G.ksum * s_max : s_max) + G.ymax) + G.cS * G.lambda1 * 3.f * G.inv_theta;
    if (MODE == MODE_AT) tb = io.tmax_in;
    if (MODE == MODE_GRAD) tb = G.lambda1 + 2.f * G.lambda2 * ((P2 ? G.ksum * s_max : s_max) + G.ymax);   // |l1 sgn(e) + 2 l2 e|
    tb *= G.gpoly2;   // the polyphase adjoint blur shrinks max|rho|
    float sc = 0.f, isc = 0.f;
    if (tb > 0.f && isfinite(tb)) {
      int e1, e2;
      frexpf(tb, &e1);
      frexpf(tb * fmaxf(G.dmax, 1.f) * 1.02f, &e2);
      const int s = min(21 - e1, 30 - e2);
      sc = ldexpf(1.f, s);
      isc = ldexpf(1.f, -s);
    }
    s_scale[0] = sc;
    s_scale[1] = isc;
  }
  if (kWeights) {  // m over own + radius from x (A8/A17/A19)
    __syncthreads();      // P complete
    for (int e = tid; e < T.MH * MW; e += NT) {
      const int my = e / MW, mx = e - my * MW;
      const int gy = Y0 - rr + my, gx = X0 - rr + mx;
      float mz = 0.f;
      if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
        const size_t gi = (size_t)gy * ps + gx;
        if (io.reweight) {
          const int py = gy - PY0, px = gx - PX0;
          const float xr = P[pidx<Z>(py, min(gx + 1, W - 1) - PX0, PW, PWZ)], xl = P[pidx<Z>(py, max(gx - 1, 0) - PX0, PW, PWZ)];
          const float xd = P[pidx<Z>(min(gy + 1, H - 1) - PY0, px, PW, PWZ)], xu = P[pidx<Z>(max(gy - 1, 0) - PY0, px, PW, PWZ)];
          const float gxv = 0.5f * (xr - xl), gyv = 0.5f * (xd - xu);
          mz = G.lambda_reg * io.wo[gi] * expf(-(gxv * gxv + gyv * gyv) * G.inv_sigma_e);
          const bool own = gy >= Y0 && gy < Y0 + TY && gx >= X0 && gx < X0 + TX;
          if (own && grp == 0) io.m[gi] = mz;
        } else {
          mz = io.m[gi];
        }
      }
      M[e] = mz;
    }
  }
  __syncthreads();

  // ---- phase 2: views (no barriers) ----------------------------------------
  double red_a = 0.0, red_b = 0.0, red_c = 0.0;
  {
    // Column mask of this lane's E positions (bit s = a real image column); rows are
    // tested per row (Tile::row_in) unless the whole E region is inside the image.
    unsigned colmask = 0;
#pragma unroll
    for (int s2 = 0; s2 < Z; ++s2) {
      const int c = Z * lane + s2, X = XE0 + c;
      // (E columns past EXv feed no own LR column and receive a zero adjoint: left as they are,
      // so their real disparity keeps the warp's adjacency test of adj_row true)
      if (X >= 0 && X < W) colmask |= 1u << s2;
    }
    const bool rows_in = (YE0 >= 0) && (YE0 + EY <= H);
    const bool cols_in = (XE0 >= 0) && (XE0 + C::EXv <= W);
    const unsigned koff = 0u - ((unsigned)kMagicBits * (unsigned)PW + (unsigned)kMagicBits / Z);
    auto run = [&](auto tile) {
      tile.colmask = colmask;
      if constexpr (decltype(tile)::kDummy) {
        tile.PHd = (float)PH;
#pragma unroll
        for (int k = 0; k <= decltype(tile)::NP; ++k) {
          const float m0 = ((colmask >> (2 * k)) & 1u) ? 1.f : 0.f;
          const float m1 = (2 * k + 1 < Z && ((colmask >> (2 * k + 1)) & 1u)) ? 1.f : 0.f;
          tile.ymul[k] = f2(m0, m1);
          tile.yadd[k] = f2((1.f - m0) * (float)PH, (1.f - m1) * (float)PH);
        }
      }
      tile.P = P; tile.ACC = ACC; tile.OM = OM; tile.PW = PW; tile.PWZ = PWZ; tile.PY0 = PY0; tile.PX0 = PX0;
      tile.YE0 = YE0; tile.XE0 = XE0; tile.H = H; tile.W = W; tile.PS = ps; tile.tscale = s_scale[0]; tile.lo = LO;
      tile.koff = koff; tile.rows_in = rows_in;
      views<Z, MODE, decltype(tile)::kInt, PV, P2, PM, RB>(tile, G, V, T, io, grp, lane, warp, NW, i0, j0, BL, red_a, red_b, red_c);
    };
    if (cols_in && rows_in) run(Tile<Z, true, RB>{});   // (columns-only interior: measured slower)
    else run(Tile<Z, false, RB>{});
  }
  if (MODE == MODE_A) return;
  CTA_T(1);

  // ---- phase 3: NLTV term of the own pixels (view group g takes own rows g, g+G, ...);
  // warps that finish their views early pull rows from a shared counter, so the NLTV
  // work (the w_S stream in WZ) fills the wait for the slowest warp.
  double red_reg = 0.0;
  const int ng = T.groups;
  const bool nltv = (MODE == MODE_WZ && !io.wz_no_nltv) || MODE == MODE_GRAD || MODE == MODE_J ||
                    (MODE == MODE_NORMAL && io.do_nltv);
  if (nltv) {
    NltvCtx c;
    c.P = P; c.M = M; c.PW = PW; c.PWZ = PWZ; c.MW = MW; c.H = H; c.W = W; c.ps = ps;
    c.ith = G.inv_theta;
    const int rd = ctl->iter & 1;
    c.wSr = rd ? io.wS1 : io.wS0;
    c.wSw = rd ? io.wS0 : io.wS1;
    c.plane = (size_t)H * ps;
    const int my_rows = TY > grp ? (TY - grp + ng - 1) / ng : 0;
    for (;;) {
      int row = 0;
      if (lane == 0) row = atomicAdd(&s_nl_next, 1);
      row = __shfl_sync(0xffffffffu, row, 0);
      if (row >= my_rows) break;
      const int oy = grp + ng * row;
      for (int ox = lane; ox < TX; ox += 32) {
        const int Y = Y0 + oy, X = X0 + ox;
        float acc = 0.f;
        if (Y < H && X < W) {
          const int py = Y - PY0, px = X - PX0;
          const int mi = (oy + rr) * MW + (ox + rr);
          const size_t gi = (size_t)Y * ps + X;
          double pq = 0.0;
          const bool inner = Y >= rr && Y < H - rr && X >= rr && X < W - rr;
          if (rr == 2) {
            acc = inner ? nltv_pixel<Z, MODE, false, 2, RB>(c, G, Y, X, py, px, mi, gi, pq, red_reg, red_c)
                        : nltv_pixel<Z, MODE, true, 2, RB>(c, G, Y, X, py, px, mi, gi, pq, red_reg, red_c);
          } else {
            acc = nltv_pixel<Z, MODE, true, 0, RB>(c, G, Y, X, py, px, mi, gi, pq, red_reg, red_c);
          }
          if (MODE == MODE_WZ || MODE == MODE_NORMAL) acc *= G.cS;
          red_b += (double)G.cS * pq;
        }
        NL[oy * TX + ox] = acc;
      }
    }
  }
  if (MODE == MODE_J) {   // cost terms of trial t only (no output image)
    double v[3] = {red_a, red_b, red_reg};
    const int slot[3] = {S_TJ + 3 * io.ls_t, S_TJ + 3 * io.ls_t + 1, S_TJ + 3 * io.ls_t + 2};
    block_reduce_add<3>(v, RED, ctl->cur, slot);
    return;
  }
  __syncthreads();   // views and NLTV done: ACC and NL complete
  CTA_T(2);

  // ---- phase 4: flush accumulator + NLTV (tile + halo) with RED.ADD ----------
  {
    const float isc = s_scale[1];
    const float sign = (MODE == MODE_WZ) ? -1.f : 1.f;   // WZ writes r = -v (reading A3)
    for (int e = tid; e < PH * PWn; e += NT) {
      const int py = e / PWn, px = e - py * PWn;
      const int gy = PY0 + py, gx = PX0 + px;
      const int ia = pidx<Z>(py, px, PW, PWZ);
      float v = fmaf((float)ACC[LO + ia], 1.f / (float)(1 << kLoBits), (float)ACC[ia]) * isc;
      const int oy = gy - Y0, ox = gx - X0;
      if (nltv && gy < H && gx < W && oy >= 0 && oy < TY && ox >= 0 && ox < TX && (oy % ng) == grp)
        v += NL[oy * TX + ox];
      // padding cells fold onto their replicate source (transpose of the padding)
      const int cy = min(max(gy, 0), H - 1), cx = min(max(gx, 0), W - 1);
      // MISR fast path: k_misr_normal owns the outputs inside the stencil rectangle Z_s
      if (io.zs_on && cy >= io.zs_y0 && cy < io.zs_y1 && cx >= io.zs_x0 && cx < io.zs_x1) continue;
      if (v != 0.f) atomicAdd(&io.out_hr[(size_t)cy * ps + cx], sign * v);
    }
  }
  // ---- reductions ----------------------------------------------------------------
  if (MODE == MODE_WZ) {
    double v[4] = {red_a, red_b, red_reg, red_c};
    const int slot[4] = {S_L1, S_L2, S_REG, S_RES2};
    block_reduce_add<4>(v, RED, ctl->cur, slot);
  } else if (MODE == MODE_GRAD) {
    double v[3] = {red_a, red_b, red_reg};
    const int slot[3] = {S_L1, S_L2, S_REG};
    block_reduce_add<3>(v, RED, ctl->cur, slot);
  } else if (MODE == MODE_NORMAL && io.cg_k >= 1) {
    // PM: the data part comes from the gather; MISR fast path: k_misr_normal forms <p, q>
    double v[2] = {io.no_pq ? 0.0 : (PM ? 0.0 : red_a) + red_b, pi0_part};
    // Chronopoulos-Gear (strips): delta = <r, M r> and gamma = <r, r> side by side (one all-reduce)
    const int slot[2] = {io.cgcg_slot > 0 ? io.cgcg_slot + 1 : S_PQ + io.cg_k, io.cgcg_slot > 0 ? io.cgcg_slot : S_PI + 0};
    block_reduce_add<2>(v, RED, ctl->cur, slot);
  }
  CTA_T(3);
}

// Per-zeta host entry points (instantiated once per zeta in tile_z<zeta>.cu).
// Instances: (fixed-height | runtime height) x shared map for every mode; runtime height
// only for per-view maps (PV) and for a user blur kernel (P2).
template <int Z>
struct TileZ {
  template <int MODE, bool F, bool PV, bool P2, bool PM = false, int RB = TileCfg<Z>::R>
  static cudaError_t launch1(const Geom& G, const Views& V, const TileGeom& T, const TileIO& io, cudaStream_t st) {
    const int nw = MODE == MODE_NORMAL ? T.nwarps_n : T.nwarps;
    const size_t sm = MODE == MODE_NORMAL ? T.smem_normal : T.smem;
    k_tile<Z, MODE, F, PV, P2, PM, RB><<<(T.ntl ? T.ntl : T.ntYl * T.ntX) * T.groups, nw * 32, sm, st>>>(G, V, T, io);
    return cudaGetLastError();
  }
  template <int MODE>
  static cudaError_t launchm(const Geom& G, const Views& V, const TileGeom& T, const TileIO& io, cudaStream_t st) {
    constexpr bool kHasAdj = (MODE == MODE_WZ || MODE == MODE_NORMAL || MODE == MODE_GRAD);
    if constexpr (kHasAdj)
      if (G.paper) return launch1<MODE, false, false, false, true>(G, V, T, io, st);
    if (G.psf2d)
      return G.psf_rb == kPsfBigR ? launch1<MODE, false, false, true, false, kPsfBigR>(G, V, T, io, st)
                                  : launch1<MODE, false, false, true>(G, V, T, io, st);
    if (G.per_view) return launch1<MODE, false, true, false>(G, V, T, io, st);
    if (MODE == MODE_GRAD || MODE == MODE_J) return launch1<MODE, false, false, false>(G, V, T, io, st);
    return T.BL == TC<Z>::BL ? launch1<MODE, true, false, false>(G, V, T, io, st)
                             : launch1<MODE, false, false, false>(G, V, T, io, st);
  }
  static cudaError_t launch(int mode, const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                           cudaStream_t st) {
    switch (mode) {
      case MODE_WZ: return launchm<MODE_WZ>(G, V, T, io, st);
      case MODE_NORMAL: return launchm<MODE_NORMAL>(G, V, T, io, st);
      case MODE_A: return launchm<MODE_A>(G, V, T, io, st);
      case MODE_AT: return launchm<MODE_AT>(G, V, T, io, st);
      case MODE_GRAD: return launchm<MODE_GRAD>(G, V, T, io, st);
      case MODE_J: return launchm<MODE_J>(G, V, T, io, st);
    }
    return cudaErrorInvalidValue;
  }
  template <int MODE, bool F, bool PV, bool P2, bool PM = false, int RB = TileCfg<Z>::R>
  static cudaError_t prep1(size_t smem) {
    return cudaFuncSetAttribute(k_tile<Z, MODE, F, PV, P2, PM, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
  }
  template <int MODE>
  static cudaError_t prepm(size_t smem) {
    cudaError_t e;
    if (MODE != MODE_GRAD && MODE != MODE_J)
      if ((e = prep1<MODE, true, false, false>(smem)) != cudaSuccess) return e;
    if ((e = prep1<MODE, false, false, false>(smem)) != cudaSuccess) return e;
    if ((e = prep1<MODE, false, true, false>(smem)) != cudaSuccess) return e;
    if constexpr (MODE == MODE_WZ || MODE == MODE_NORMAL || MODE == MODE_GRAD)
      if ((e = prep1<MODE, false, false, false, true>(smem)) != cudaSuccess) return e;
    if ((e = prep1<MODE, false, false, true, false, kPsfBigR>(smem)) != cudaSuccess) return e;
    return prep1<MODE, false, false, true>(smem);
  }
  static cudaError_t prepare(size_t smem) {
    cudaError_t e;
    if ((e = prepm<MODE_WZ>(smem)) != cudaSuccess) return e;
    if ((e = prepm<MODE_NORMAL>(smem)) != cudaSuccess) return e;
    if ((e = prepm<MODE_A>(smem)) != cudaSuccess) return e;
    if ((e = prepm<MODE_AT>(smem)) != cudaSuccess) return e;
    if ((e = prepm<MODE_GRAD>(smem)) != cudaSuccess) return e;
    return prepm<MODE_J>(smem);
  }
  static int occupancy(int threads, size_t smem) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_tile<Z, MODE_NORMAL, false, false, false, false>, threads,
                                                      smem) != cudaSuccess) {
      cudaGetLastError();
      return 1;
    }
    return n > 0 ? n : 1;
  }
};

}  // namespace lfsr
