// internal.h — device-side data structures shared by the liblfsr kernels and
// the C-ABI host code.  Nothing here is visible through include/lfsr.h.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lfsr {

constexpr int kMaxViews = 1024;  // view offsets travel in the kernel parameter block
constexpr int kMaxTaps = 8;      // blur radius R <= 3 for zeta <= 4 (Appendix B of DESIGN.md)
constexpr int kMaxOffsets = 80;  // s_d for r <= 4
constexpr int kMaxK = 64;        // CG steps per ADMM iteration
constexpr int kThreads = 256;    // threads per tile CTA
constexpr int kMaxLs = 32;       // gd-ls: Armijo trials per iteration (reading A32)
constexpr int kPsfBigR = 7;      // blur radius of the large user-kernel tile instances (A36: up to 15x15)

// Scalar slots of the current ADMM iteration (doubles in Control::cur).
enum Slot : int {
  S_L1 = 0,     // sum |e|
  S_L2 = 1,     // sum e^2
  S_REG = 2,    // sum_d sum_z |W_d Delta_d x|
  S_RES2 = 3,   // |w^n - w^{n-1}|^2
  S_NF = 4,     // non-finite count
  S_CGIT = 5,   // CG steps taken
  S_BREAK = 6,  // CG breakdown flag
  S_STOP = 7,   // CG stopped flag (pi < tau, pi == 0 or breakdown)
  S_PI = 8,     // pi_k = <r_k, r_k>, k = 0..K      at S_PI + k
  S_PQ = S_PI + kMaxK + 1,  // <p_k, M p_k>, k = 1..K at S_PQ + k
  S_GN = S_PQ + kMaxK + 1,  // gd: |g|^2
  S_TJ = S_GN + 1,          // gd-ls: cost terms (sum|e|, sum e^2, sum|G|) of trial t at S_TJ + 3t
  S_CG = S_TJ + 3 * kMaxLs, // strips, Chronopoulos-Gear CG: (gamma_j, delta_j) of step j at S_CG + 2j
  S_ALPHA = S_CG + 2 * (kMaxK + 1),   // ... and the previous step's alpha
  S_COUNT = S_ALPHA + 1
};

// Stats record layout in the ring (doubles).
enum StatSlot : int {
  T_ITER = 0, T_CGIT, T_BREAK, T_NF, T_J, T_L1, T_L2, T_REG, T_RES, T_PI0, T_PILAST, T_COUNT
};

struct Control {
  double cur[S_COUNT];
  double* ring;       // [cap][T_COUNT]
  int32_t cap;
  int32_t iter;       // ADMM iterations completed since set_observations
  uint32_t done;      // last-block counter for the closing kernel
  int32_t pad;
};

// Geometry + solver constants, passed by value to every kernel.
struct Geom {
  int32_t H, W, h, w;         // HR / LR sizes
  int32_t ps, lps;            // HR row pitch, LR row pitch (floats, multiples of 32)
  int32_t scale, R;           // zeta, blur radius
  int32_t n_views, ref_view;
  int32_t radius, s_d;        // NLTV window radius and offset count
  int32_t SY, SX;             // ceil(max |dtau * omega|), ceil(max |drho * omega|)
  int32_t K;                  // CG max steps
  float lambda1, lambda2, lambda_reg, theta, inv_theta;
  float inv_sigma_e, inv_2s1sq, inv_2s2sq;  // 0 when the factor is disabled (sigma = inf)
  float cg_tol;
  float cA;                   // lambda2 + (theta/2) lambda1^2   (A7)
  float dmax;                 // max_z sum_k (W_k^T 1)(z) (set at set_observations)
  float ymax;                 // max |y|
  float gpoly2;               // (max polyphase tap sum)^2: |B^T D^T rho| <= gpoly2 max|rho|
  float cS;                   // theta / 2
  int32_t tile_bl;            // LR rows per tile (host-chosen, 0 = the zeta default; see make_tile_geom)
  int32_t tile_g, tile_nw;    // view groups and warps per CTA (host-chosen, 0 = the cost model's choice)
  int32_t tile_nwn;           // warps per CTA of the NORMAL launches (host-chosen, 0 = tile_nw)
  int32_t per_view;           // 1: omega is [n_views][H][ps], view k warped with omega_k (A34)
  int32_t psf2d;              // 1: user blur kernel (A36) in psf2 instead of the separable taps
  int32_t paper;              // 1: the paper's backward-warp adjoint W_k^* with omega_0 (A37)
  float ksum;                 // sum |k| of the blur kernel (1 for the normalised Gaussian): |B w| <= ksum max|w|
  int32_t psf_rb;             // blur radius of the psf2 layout: R (kernel radius <= R) or 7 (larger kernels)
  float psf2[2 * 7 + 1][2 * 7 + 1];   // psf2[a][b] = k[rb-a][rb-b]: E-offset (correlation) order, zero padded to 2 rb + 1
  float taps[kMaxTaps * 2 + 1];
  float2 tpe[kMaxTaps + 1];   // tap pairs (taps[2v], taps[2v+1]), zero past 2R (packed FP32 operands)
  float2 tpo[kMaxTaps + 1];   // tap pairs (taps[2v+1], taps[2v+2])
  float wd[kMaxOffsets];      // spatial weights w_d
  int8_t ody[kMaxOffsets], odx[kMaxOffsets];
};

struct Views {
  float2 off[kMaxViews];      // (drho, dtau)
};

// Tile decomposition of the HR grid; every field is derived on the host.
// A tile = a band of BL LR rows x a strip of LX LR columns (one warp column of
// 32 lanes, lane = LR column); its "E region" is the set of HR positions whose
// blurred warped value reaches an own LR pixel: EY rows x ECOL (= 32 zeta)
// columns, of which EXv are real.
struct TileGeom {
  int32_t BL, LX;             // LR rows / columns per tile
  int32_t TY, TX;             // own HR pixels per tile (= zeta * BL, zeta * LX)
  int32_t EY, ECOL, EXv;      // E region rows, allocated columns, valid columns
  int32_t SYe, SXe;           // halo of the input tile around the E region (>= radius)
  int32_t PH, PW, PWZ;        // input tile rows, row pitch (= zeta * PWZ), phase pitch
  int32_t MH, MW;             // m tile (own + radius halo)
  int32_t ntY, ntX;           // tiles per axis (whole image)
  int32_t tY0, ntYl;          // this strip's tile rows [tY0, tY0 + ntYl)
  int32_t groups;             // view groups (CTAs per tile)
  int32_t vpg;                // views per group
  int32_t nwarps;             // warps per CTA (views of a group are dealt round-robin)
  int32_t nwarps_n;           // warps per CTA of the NORMAL (CG operator) launches (may exceed nwarps)
  const int* tlist;           // MISR fast path: the border tiles only (indices into the ntYl x ntX grid), or null
  int32_t ntl;                // entries of tlist (0: every tile)
  size_t smem;                // dynamic shared memory bytes (largest mode)
  size_t smem_normal;         // ... of the NORMAL mode
};

// Pointers of one tile-kernel launch (see tile_kernels.cu).
struct TileIO {
  const float* in_hr;    // x (WZ) | r (NORMAL-CG) | p (NORMAL-op, A)
  const float* in_hr2;   // p_{k-1} (NORMAL-CG) or nullptr
  float* p_out;          // p_k written for own pixels (NORMAL-CG) or nullptr
  const float* omega;
  const float* y;        // WZ
  float* wA;             // WZ (in/out)
  float* wS0;            // WZ: w_S ping-pong buffers; read wS[iter&1], write wS[(iter&1)^1]
  float* wS1;
  const float* wo;       // WZ (weights)
  float* m;              // WZ: written (if reweight) / read; NORMAL: read
  const float* in_lr;    // AT
  float* out_lr;         // A
  float* out_hr;         // accumulated (RED.ADD) output: r (WZ, sign -1) | q (NORMAL) | AT
  Control* ctl;
  float tmax_in;         // AT: max |in_lr| (bound for the fixed-point scale)
  int32_t cg_k;          // NORMAL-CG: step index k >= 1; 0 = plain operator
  int32_t reweight;      // WZ: recompute m from x
  int32_t do_nltv;       // NORMAL: include the (th/2) S^T S term
  int32_t ls_t;          // J: line-search trial index t (input tile = x - eta0 2^-t g, in_hr2 = g)
  float* rho_out;        // paper mode (A37): rho of every LR pixel [n_views][h][lps] for k_paper_gather
  float eta0;            // J: initial step of the line search
  float armijo_c;        // J: Armijo constant c (reading A32)
  int32_t zs_on;         // MISR fast path: flush only outside the stencil rectangle Z_s ...
  int32_t zs_y0, zs_y1, zs_x0, zs_x1;
  int32_t no_pq;         // ... and leave <p, Mp> to k_misr_normal
  int32_t wz_no_nltv;    // WZ: the NLTV rows run in k_wz_nltv (nltv.cu) instead of phase 3
  int32_t cgcg_slot;     // NORMAL, strips (Chronopoulos-Gear): > 0: w = M r with gamma = <r, r> -> cur[slot],
  int32_t cgcg_step;     //   delta = <r, M r> -> cur[slot + 1]; step index j (j >= 1: skip once CG stopped)
};

// WZ: ADMM wz-step; NORMAL: CG normal operator; A / AT: test operators;
// GRAD: cost terms and subgradient of J for gd (A30); J: cost terms of one gd-ls trial.
enum TileMode : int { MODE_WZ = 0, MODE_NORMAL = 1, MODE_A = 2, MODE_AT = 3, MODE_GRAD = 4, MODE_J = 5 };

// MISR fast path (misr.cu): the zeta^2-phase stencil of the data normal operator for constant
// shifts, the NLTV weights, and the launch arguments.
constexpr int kMisrMaxCoef = 16 * 15 * 15;   // zeta^2 phases x (4R+3)^2 taps, zeta <= 4 (R <= 3)

struct MisrStencil {
  float s[kMisrMaxCoef];   // [phase py*zeta+px][dy + WR][dx + WR], WR = 2R + 1; c_A folded in
  float w2[24], w2f[24];   // w_d^2 and w_{-d}^2 in the offset order of A9 (5x5 window)
  float W2;                // sum_d w_d^2
  // separable form (sep = 1; views on a Cartesian grid of shifts, symmetric separable NLTV
  // weights w_d^2 = u[dy] u[dx], d != 0): M_data = T_y (x) T_x exactly, border included, with the
  // banded 1-D matrices in MisrArgs::tyt / txt -- no border kernel
  int32_t sep;
  float u[5];
};

struct MisrArgs {
  const float* r;       // CG residual (k >= 1) ...
  const float* p_prev;  // ... and the previous direction (k >= 2)
  const float* p_in;    // k = 0 (plain operator): the input
  float* p_out;         // k >= 1: p_k on the owned rectangle
  const float* m;       // weight map (NLTV)
  const float* tyt;     // sep: T_y [H][2WR+1] (c_A folded in), T_x [W][2WR+1]; row z holds the taps to z + D
  const float* txt;
  float* q;             // output (stored on Z_s; the band is the border kernel's)
  Control* ctl;
  int cg_k, do_nltv;
  int zs_y0, zs_y1, zs_x0, zs_x1;   // stencil-exact rectangle Z_s
  int o_y0, o_y1, o_x0, o_x1;       // pixels not owned by a border tile (p_out, pi_0)
};

// Assembled data normal operator (asm.cu): the stencil planes of the regular
// rows of the stacked A_k, the irregular rows as a compact list with per-tile CSR lists, per-row t.
constexpr int kAsmPad = 8;   // zero rows / columns around every stencil plane (>= the stencil radius)

struct AsmBuf {
  const float* omega;   // disparity (shared [H][ps] or per view)
  float* st;            // [NH][H + 2 pad][psS] stencil planes (c_A folded in)
  int psS;              // plane row pitch (floats)
  size_t plane;         // floats per plane
  float* rows;          // [n_views][h][w][RS] row records: (2R+2)^2 window weights, base (y << 16 | x) or INT_MIN
  unsigned* count;      // [0] irregular rows, [1] positions in their windows (device)
  int2* list;           // [n_views h w] irregular rows (k, iy << 16 | ix), first count[0] valid
  unsigned* pmask;      // [n_views][H][pmw] positions in an irregular row's blur window
  int pmw;
  uint2* plist;         // [n_views H W] those positions (k, Y << 16 | X), first count[1] valid
  float* tdense;        // [n_views][h][w] t = c_A a . p of the irregular rows (0 at regular rows)
  float* udense;        // [n_views][H][W] u = W_k p at the positions (per CG step)
  float om_max;         // max |omega| (footprints)
};

struct AsmFork {          // side stream + events for the concurrent irregular-row kernels (null: serial)
  cudaStream_t side;
  cudaEvent_t fork, join;
};

struct AsmStep {
  const float* r;       // CG residual (k >= 1)
  const float* p_prev;  // p_{k-1} (k >= 2)
  const float* p_in;    // k = 0: the operator input
  float* p_out;         // k >= 1: p_k
  const float* m;       // NLTV weight map
  float* q;             // output (stored)
  Control* ctl;
  int cg_k;
};

// gd / gd-ls configuration of one iteration graph (readings A30-A33).
struct GdCfg {
  float eta0;        // (initial) step
  float armijo_c;    // Armijo constant
  int32_t ls;        // 1: Armijo backtracking over L trials
  int32_t L;         // trials (<= kMaxLs)
};

struct State {
  // persistent solver state (pitched)
  float* x;      // [H][ps]
  float* y;      // [n_views][h][lps]
  float* wA;     // [n_views][h][lps]
  float* wS[2];  // [s_d][H][ps] ping-pong (read iter&1, write the other)
  float* density;  // [H][ps] splat density sum_k W_k^T 1 (fixed-point bound)
  float* omega;  // [H][ps], or [n_views][H][ps] with per-view disparity (A34)
  float* wo;     // [H][ps]
  float* m;      // [H][ps]
  // CG vectors
  float* r;      // [H][ps]
  float* p[2];   // ping-pong
  float* q;      // [H][ps]
  // scratch for ops
  float* tmp_hr;   // [H][ps]
  float* tmp_lr;   // [n_views][h][lps]
  float* rho;      // [n_views][h][lps] paper mode (A37) only
  Control* ctl;
};

}  // namespace lfsr
