/*
 * lfsr.h — C ABI of the B200-native ADMM light-field super-resolution library
 * (liblfsr.so), the data-parallel hot path of arXiv 2206.05047:
 * "A GPU-Accelerated Light-field Super-resolution Framework Based on Mixed
 * Noise Model and Weighted Regularization" (Tran, Sun, Simon).
 *
 * Citation key: P:Lnnn = line nnn of the paper's LaTeX source;
 * S:Lnnn = SPEC.md; readings A1..A27 = DESIGN.md §3.
 *
 * The library minimises (Eq. sr_fin)
 *     J(x) = l1 sum_k |A_k x - y_k|_1 + l2 sum_k |A_k x - y_k|_2^2
 *          + sum_d |W_d (.) (S_d - I) x|_1 ,      A_k = D B W_k
 * with the restructured scaled-dual ADMM of Algorithm 1 and the
 * conjugate-gradient x-step of Algorithm 2 (textbook readings
 * A1-A4).  Every step runs in hand-written sm_100a CUDA kernels; there is no
 * CPU fallback: without a usable CUDA device every call that needs one
 * returns LFSR_ERR_CUDA.
 *
 * Conventions (all calls):
 *   - All arrays are dense, row-major, fp32 (float) unless stated.
 *   - HR size H x W = (scale*lr_height) x (scale*lr_width); p = H*W, q = h*w.
 *   - `mem` says whether every pointer of that call is host (LFSR_MEM_HOST) or
 *     device (LFSR_MEM_DEVICE, same CUDA device as the ctx) memory.
 *   - The caller owns every pointer it passes; the library copies inputs and
 *     never keeps a caller pointer.  Host inputs are fully consumed before the
 *     call returns; device inputs are read in the order of the ctx stream.
 *   - Calls never throw; C++ exceptions never cross this boundary.
 *   - A ctx is single-threaded; different ctxs are independent.
 *   - After LFSR_ERR_CUDA / LFSR_ERR_NCCL the ctx is poisoned: every later call
 *     except lfsr_destroy / lfsr_last_error returns LFSR_ERR_STATE.
 */
#ifndef LFSR_H_
#define LFSR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFSR_ABI_VERSION 3

#if defined(__GNUC__)
#define LFSR_API __attribute__((visibility("default")))
#else
#define LFSR_API
#endif

typedef struct lfsr_ctx lfsr_ctx; /* opaque; owns all device state */

typedef enum {
  LFSR_OK = 0,
  LFSR_ERR_INVALID_ARG = 1, /* validation failed; no side effects              */
  LFSR_ERR_STATE = 2,       /* wrong call order or poisoned ctx                */
  LFSR_ERR_OOM = 3,         /* device allocation failed                        */
  LFSR_ERR_CUDA = 4,        /* CUDA error (incl. no device); ctx poisoned      */
  LFSR_ERR_NCCL = 5,        /* NCCL error; ctx poisoned                        */
  LFSR_ERR_DIVERGED = 6,    /* non-finite x or cost; see stats[].nonfinite     */
  LFSR_ERR_UNSUPPORTED = 7  /* valid but not supported by this build           */
} lfsr_status;

typedef enum { LFSR_MEM_HOST = 0, LFSR_MEM_DEVICE = 1 } lfsr_mem;

/* Disparity layout.  SHARED: one HR map omega on theta_0's grid used by every
 * view (reading A12).  PER_VIEW (the paper's omega_k, P:L580-582;
 * reading A34): [n_views][H][W], view k is warped with its own map omega_k on
 * theta_0's grid (W_k x (z) = x(z + dtheta_k omega_k(z)), exact transpose kept);
 * the occlusion weight uses omega_{ref_view}.  Costs one extra global read of
 * omega_k per E row and view in the fused kernel. */
typedef enum { LFSR_DISP_SHARED = 0, LFSR_DISP_PER_VIEW = 1 } lfsr_disp_mode;

typedef struct {
  int32_t n_views;      /* s_k >= 1                                         */
  int32_t lr_height;    /* s_y >= 1                                                  */
  int32_t lr_width;     /* s_x >= 1                                                  */
  int32_t scale;        /* zeta in {2,3,4}                              */
  int32_t ref_view;     /* index of theta_0 in [0, n_views)                  */
  int32_t nltv_radius;  /* r in [1,4]; window (2r+1)^2, s_d = (2r+1)^2-1 (A9) */
  float lambda1;        /* >= 0, l1 data weight                          */
  float lambda2;        /* >= 0, l2 data weight; lambda1 + lambda2 > 0                */
  float lambda_reg;     /* >= 0 multiplier on W_d (A19); J itself has none   */
  float sigma_s;        /* > 0 spatial weight falloff w_d = exp(-|d|^2/sigma_s) (A8)  */
  float sigma_e;        /* > 0 edge weight falloff (A8); INFINITY disables    */
  float sigma_o1;       /* > 0 occlusion-boundary falloff (Eq. weight_occ); INF off   */
  float sigma_o2;       /* > 0 projection-error falloff (Eq. weight_occ); INF off     */
  float theta;          /* > 0 ADMM penalty vartheta                         */
  int32_t cg_max_iters; /* K in [1, 64]                                      */
  float cg_tol;         /* tau >= 0 on <r,r>; 0 => always K steps (A1, A18)   */
  int32_t reweight_every_iter; /* 1 = paper (weights from x^{n-1}); 0 = W
                                  frozen at the value computed from x^0              */
  int32_t device;       /* CUDA device ordinal                                       */
  int32_t rank;         /* this process's strip in [0, n_ranks) (NCCL mode), or -1 with
                           n_ranks > 1: all strips in this ctx on one device ("virtual
                           ranks": the same decomposition and exchange schedule with
                           device copies instead of NCCL; for testing)               */
  int32_t n_ranks;      /* >= 1 HR row strips (DESIGN 10)                  */
  const void* nccl_unique_id; /* NCCL mode: 128-byte ncclUniqueId (same on all ranks),
                                 e.g. broadcast over a torch.distributed group; else NULL */
  void* stream;         /* cudaStream_t to run on (e.g. torch.cuda.current_stream()
                           .cuda_stream), or NULL for a ctx-owned stream             */
  const float* offset_weights; /* NULL: w_d = exp(-|d|^2/sigma_s) (A8).  Else s_d finite
                           weights >= 0 in the offset order of reading A9 (row-major dy,
                           dx over the window, centre skipped), copied at lfsr_create --
                           e.g. BTV's alpha^(|dx|+|dy|) for the MISR use (P:L404-412,
                           P:L1110-1116).  Host memory.              */
  const float* psf;     /* NULL: the Gaussian blur of P:L579 (A11).  Else a user blur kernel
                           k [(2 psf_radius+1)][(2 psf_radius+1)] row-major, finite, host
                           memory, copied at lfsr_create: (B x)(Y,X) = sum_{u,v} k[u][v]
                           x(Y-u, X-v), zero padding (P:L962 motion blur, SURVEY 8f NEXT-4,
                           reading A36).  Not with LFSR_DISP_PER_VIEW (UNSUPPORTED).  */
  int32_t psf_radius;   /* 0..7 (up to 15x15).  Kernels within the Gaussian's window
                           (radius <= 2 at zeta = 2, <= 3 at zeta = 3, 4) run in the
                           default tile instances, larger ones in the radius-7 instances
                           (narrower tiles); those are single-strip only (n_ranks > 1:
                           UNSUPPORTED).  INVALID_ARG outside 0..7.                    */
  int32_t paper_adjoint; /* 0 (default): A^T uses the exact transpose W_k^T of the warp (A12).
                           1: the paper's own adjoint warp W_k^* -- a backward warp with
                           omega_0, (W_k^* u)(z) = u(z - dtheta_k omega_0(z)) (P:L583,
                           reading A37) -- in A^T, v and the CG operator, which is then not
                           symmetric (Alg. 1/2 run unchanged).  Single strip, Gaussian blur
                           and shared disparity only (else UNSUPPORTED).  SURVEY 8f NEXT-2. */
} lfsr_params;

/* Per-ADMM-iteration record.  J terms refer to x^{n-1} and the
 * weights computed from it (reading A26): J = lambda1*data_l1 + lambda2*data_l2
 * + reg_l1.  primal_res = |w^n - w^{n-1}|_2 in scaled units (A27).  cg_pi0 =
 * <r0,r0>, cg_pi_last = <r,r> after the last CG step taken. */
typedef struct {
  int32_t iter;       /* 1-based ADMM iteration index since set_observations */
  int32_t cg_iters;   /* CG steps taken (<= K)                              */
  int32_t breakdown;  /* 1 if CG stopped on <p,Mp> <= 0                     */
  int32_t nonfinite;  /* 1 if x or J became non-finite                      */
  double J, data_l1, data_l2, reg_l1, primal_res, cg_pi0, cg_pi_last;
} lfsr_iter_stats;

/* Create a ctx on params->device and allocate nothing large yet.  NCCL mode
 * (n_ranks > 1, rank >= 0) initialises the communicator: every rank must call
 * lfsr_create collectively.
 * Errors: LFSR_ERR_INVALID_ARG (any field out of range; `out` untouched),
 * LFSR_ERR_NCCL (libnccl missing or init failed), LFSR_ERR_CUDA (no usable device). */
LFSR_API lfsr_status lfsr_create(const lfsr_params* params, lfsr_ctx** out);

/* Load the observations and reset the solver state (x = x0, w = 0) (Alg.1
 * lines 1-2).
 *   lr_views     [n_views][lr_height][lr_width]  y_k
 *   view_offsets [n_views][2] = (drho_k, dtau_k) = theta_k - theta_0 in angular
 *                steps; drho shifts along X (columns), dtau along Y (rows) (A13)
 *   disparity    [H][W] omega on theta_0's HR grid, HR px per angular step (SHARED),
 *                or [n_views][H][W] omega_k (PER_VIEW)
 *   x0           [H][W] initial guess, or NULL => bicubic (Catmull-Rom a=-0.5)
 *                up-sampling of the reference view (A15)
 * Also computes the static occlusion weight w_o (Eq. weight_occ, P:L424-444,
 * A16/A17) and the weight map from x0.  Synchronises the ctx stream (it needs
 * max|omega| and the view offsets on the host to size the kernel halos).
 * Errors: INVALID_ARG (NULL arrays, non-finite offsets or disparity, unknown
 * disp_mode), UNSUPPORTED (disparity range too large for the shared-memory
 * tile), OOM, CUDA, STATE. */
LFSR_API lfsr_status lfsr_set_observations(lfsr_ctx* ctx, const float* lr_views, const float* view_offsets,
                                  const float* disparity, lfsr_disp_mode disp_mode,
                                  const float* x0, lfsr_mem mem);

/* Run n_iters >= 0 ADMM iterations (Alg.1 lines 3-10) continuing from the
 * current (x, w_A, w_S): run(a); run(b) == run(a+b).  Each iteration is one
 * CUDA-graph launch on the ctx stream.  Blocks until done.  stats: NULL or an
 * array of n_iters records.  Errors: STATE (before set_observations, or after
 * lfsr_gd_run iterations since it), DIVERGED (non-finite x/J; the state is kept for inspection), CUDA. */
LFSR_API lfsr_status lfsr_admm_run(lfsr_ctx* ctx, int32_t n_iters, lfsr_iter_stats* stats);

/* Enqueue n_iters >= 0 ADMM iterations (graph launches) on the ctx stream and
 * return immediately (no host synchronisation, no divergence check).  The
 * iterations' records can be read later with lfsr_admm_stats.  Errors: STATE,
 * INVALID_ARG, CUDA. */
LFSR_API lfsr_status lfsr_admm_enqueue(lfsr_ctx* ctx, int32_t n_iters);

/* Blocking read of the records of iterations [first_iter, first_iter+n_iters)
 * (1-based, counted since set_observations; the device keeps the last 4096).
 * stats may be NULL (divergence check only).  Returns LFSR_ERR_DIVERGED if any
 * of them saw a non-finite x or cost; INVALID_ARG if outside the window. */
LFSR_API lfsr_status lfsr_admm_stats(lfsr_ctx* ctx, int32_t first_iter, int32_t n_iters, lfsr_iter_stats* stats);

/* Bench/profiling: enable (1) or disable (0) external event-record nodes around
 * every kernel of the iteration graph (rebuilds the graph; resets the
 * accumulators).  lfsr_profile_read adds the per-kernel device times of the
 * MOST RECENT replay to three accumulators and returns them: ms[0] wz-step
 * (tile kernel, mode WZ), ms[1] CG normal operator (tile kernel, mode NORMAL),
 * ms[2] CG update; launches[i] = number of kernel launches accumulated. */
LFSR_API lfsr_status lfsr_profile(lfsr_ctx* ctx, int32_t enable);
LFSR_API lfsr_status lfsr_profile_read(lfsr_ctx* ctx, double* ms /*[3]*/, int64_t* launches /*[3]*/);
/* With the assembled CG operator (lfsr_normal_path == 2), the split of ms[1] above: ms[0] the
 * stencil kernel (k_asm_normal), ms[1] the irregular-row kernels; passes = CG operator passes
 * accumulated (0 on the other paths).  Reset by lfsr_profile. */
LFSR_API lfsr_status lfsr_profile_read_split(lfsr_ctx* ctx, double* ms /*[2]*/, int64_t* passes);

/* Copy the current HR estimate x [H][W] into x_out.  HOST: blocks;
 * DEVICE: stream-ordered on the ctx stream. */
LFSR_API lfsr_status lfsr_get_hr(lfsr_ctx* ctx, float* x_out, lfsr_mem mem);

/* Dump the state for parity checks: w_A [n_views][h][w], w_S [s_d][H][W]
 * (scaled duals, A6), x [H][W], m [H][W] (current weight map, W_d = w_d m).
 * Any pointer may be NULL.  Blocks for HOST. */
LFSR_API lfsr_status lfsr_get_state(lfsr_ctx* ctx, float* w_A, float* w_S, float* x, float* m, lfsr_mem mem);

/* Test/bench operators on the current state (frozen weight map m):
 *   A       : in HR [H][W]            -> out [n_views][h][w]   A_k x
 *   AT      : in [n_views][h][w]      -> out HR                sum_k A_k^T r_k
 *   S       : in HR                   -> out [s_d][H][W]       W_d (.) Delta_d x
 *   ST      : in [s_d][H][W]          -> out HR                div^{U,V}
 *   NORMAL  : in HR                   -> out HR                M x (A7)
 *   WEIGHTS : in HR x                 -> out HR m(x) = lambda_reg w_o w_e(x)
 * NORMAL/A/AT run the same tile kernels as lfsr_admm_run, GRAD the one of lfsr_gd_run.
 * Blocks for HOST. */
typedef enum {
  LFSR_OP_A = 0,
  LFSR_OP_AT = 1,
  LFSR_OP_S = 2,
  LFSR_OP_ST = 3,
  LFSR_OP_NORMAL = 4,
  LFSR_OP_WEIGHTS = 5,
  LFSR_OP_GRAD = 6,    /* in HR x -> out HR subgradient of J at x with the current m:
                          sum_k A_k^T (l1 sgn(e_k) + 2 l2 e_k) + S_w^T sgn(S_w x) (A30) */
  LFSR_OP_BICUBIC = 7  /* in LR [h][w] -> out HR: the bicubic up-sampling of x0 (A15),
                          used for the Cb / Cr planes of colour input */
} lfsr_op;
LFSR_API lfsr_status lfsr_op_apply(lfsr_ctx* ctx, lfsr_op op, const float* in, float* out, lfsr_mem mem);

/* Gradient-descent baselines of the paper's solver comparison (P:L910-933:
 * "gradient descent solver (GD) without and with line search denoted as gd and
 * gd-ls"; readings A30-A33 of DESIGN.md §3).  Per iteration,
 * from x = x^{n-1}: m = weights(x) (if reweight_every_iter; A31), cost J(x) and
 * its subgradient g = sum_k A_k^T (l1 sgn(e_k) + 2 l2 e_k) + S_w^T sgn(S_w x)
 * (A30), then
 *   gd    : x := x - step g
 *   gd-ls : Armijo backtracking (A32): the first t < max_trials with
 *           J(x - step 2^-t g) <= J(x) - armijo_c step 2^-t |g|^2 is taken; none
 *           => x unchanged and ls_failed = 1.
 * The same fused tile kernel as the ADMM path computes e, the adjoint and the
 * NLTV term; every step runs on the device (one CUDA graph per iteration, no
 * host round trip inside it). */
typedef struct {
  float step;           /* > 0: the fixed step (gd) or the first trial (gd-ls)        */
  int32_t line_search;  /* 0: gd, 1: gd-ls                                            */
  int32_t max_trials;   /* gd-ls: L in [1, 32] trials step * 2^-t, t < L              */
  float armijo_c;       /* >= 0, Armijo constant (1e-4)                        */
} lfsr_gd_params;

/* Per-gd-iteration record.  J terms at x^{n-1} with m(x^{n-1}) (as lfsr_iter_stats). */
typedef struct {
  int32_t iter;         /* 1-based, counted since set_observations                    */
  int32_t ls_evals;     /* line-search trials evaluated (0 for gd)                     */
  int32_t ls_failed;    /* 1: no trial met the Armijo condition (x unchanged)          */
  int32_t nonfinite;    /* 1: x or J became non-finite                                 */
  int32_t cu;           /* computation units of this iteration: 2 + ls_evals (A33)     */
  int32_t pad;
  double J, data_l1, data_l2, reg_l1;
  double step;          /* step taken (0 if ls_failed)                                 */
  double grad_sq;       /* |g|^2                                                       */
} lfsr_gd_stats;

/* Run n_iters >= 0 gd / gd-ls iterations continuing from the current x (run(a);
 * run(b) == run(a+b)); blocks until done.  One solver per set_observations: after
 * ADMM iterations this returns STATE (and lfsr_admm_run after gd iterations).
 * stats: NULL or n_iters records.  Errors: INVALID_ARG (params), STATE,
 * UNSUPPORTED (strip decompositions, n_ranks > 1), DIVERGED, OOM, CUDA. */
LFSR_API lfsr_status lfsr_gd_run(lfsr_ctx* ctx, const lfsr_gd_params* gd, int32_t n_iters, lfsr_gd_stats* stats);

/* Solve n_fields independent light fields of this ctx's geometry, each exactly as
 * lfsr_set_observations (shared disparity, bicubic x0) + lfsr_admm_run(n_iters) +
 * lfsr_get_hr would, pipelined: field i+1's inputs are copied to the device and its
 * setup maxima computed on a second stream while field i's iterations run, and x_i is
 * copied back asynchronously (the serving path of many light fields, e.g. one per
 * reference view θ0).  All arrays are HOST memory, one pointer per field:
 * lr_views[i] [n_views][h][w], view_offsets[i] [n_views][2], disparity[i] [H][W],
 * x_out[i] [H][W]; page-locked buffers are needed for the copies to overlap (pageable
 * ones work, serialised).  Blocks until every field is done.  Afterwards the ctx holds
 * the last field's state.  Errors: INVALID_ARG, UNSUPPORTED (strip decompositions),
 * DIVERGED (any field), OOM, CUDA. */
LFSR_API lfsr_status lfsr_solve_batch(lfsr_ctx* ctx, int32_t n_fields, const float* const* lr_views,
                                      const float* const* view_offsets, const float* const* disparity,
                                      int32_t n_iters, float* const* x_out);

/* Kernel launches of one gd iteration graph (valid after lfsr_gd_run; 0 before). */
LFSR_API int32_t lfsr_gd_launches_per_iter(const lfsr_ctx* ctx);

/* Colour input ("solve the cost function for Y color channel while
 * applying bi-cubic interpolation for Cb and Cr channel"; reading A35): full-range
 * ITU-R BT.601 on [0, 1] -- Y = 0.299 R + 0.587 G + 0.114 B, Cb = 0.5 + (B - Y)/1.772,
 * Cr = 0.5 + (R - Y)/1.402 -- and its inverse.  rgb is planar [3][n_pixels]; all
 * pointers are DEVICE memory of the current device; stream: cudaStream_t or NULL.
 * Stream-ordered, no ctx.  Errors: INVALID_ARG (NULL or non-device pointers), CUDA. */
LFSR_API lfsr_status lfsr_rgb_to_ycbcr(const float* rgb, float* y, float* cb, float* cr, size_t n_pixels,
                                       void* stream);
LFSR_API lfsr_status lfsr_ycbcr_to_rgb(const float* y, const float* cb, const float* cr, float* rgb,
                                       size_t n_pixels, void* stream);

/* Number of kernel launches one ADMM iteration issues (for the bench's
 * gpu_launches count).  Valid after set_observations; 0 otherwise. */
LFSR_API int32_t lfsr_launches_per_iter(const lfsr_ctx* ctx);

/* Tiling of the fused operator kernel chosen for this context:
 * LR rows per tile, view groups (CTAs per tile), warps per CTA, and warps per
 * CTA of the CG normal-operator launches (may be wider: up to 16 at zeta = 2).
 * A single strip picks them at its first lfsr_set_observations of a geometry by
 * timing the CG normal-operator kernel for a few candidates (cached per process;
 * environment LFSR_TILE_BL / LFSR_TILE_GNW="groups,warps" / LFSR_TILE_NWN force
 * them).  Any out pointer may be NULL.  LFSR_ERR_STATE before set_observations. */
LFSR_API lfsr_status lfsr_tile_config(const lfsr_ctx* ctx, int32_t* tile_rows, int32_t* view_groups,
                                      int32_t* warps_per_cta, int32_t* cg_warps_per_cta);

/* The MISR / global-shift fast path of the CG normal operator.
 * When the disparity map is one constant (every view a global translation, as the MISR frames
 * of P:L1110-1116), lfsr_set_observations assembles the data part of M (A7) as a
 * zeta^2-phase stencil on the host in fp64, and each CG step runs it on the interior rectangle
 * Z_s where it is exact, with the exact tile kernel on the border tiles for the band outside
 * Z_s.  Requires the shared disparity layout, the Gaussian blur, the exact adjoint, a single
 * strip, nltv_radius 2; LFSR_MISR_FAST=0 in the environment at lfsr_set_observations turns it
 * off; lfsr_solve_batch never uses it.  Results match the generic path to fp32 rounding.
 * active: 1 if the current observations use it.  rect (NULL or int32[8]): Z_s as [y0, y1) x
 * [x0, x1), then the HR pixels no border tile owns, same layout.  Errors: INVALID_ARG (ctx or
 * active NULL), STATE (before lfsr_set_observations). */
LFSR_API lfsr_status lfsr_fast_path(const lfsr_ctx* ctx, int32_t* active, int32_t* rect);

/* Which implementation applies the CG normal operator M (A7) for the current
 * observations.  path: 0 = the fused tile kernel (warp / blur / decimate and
 * their adjoints for every view, each CG step); 1 = the MISR fast path (lfsr_fast_path);
 * 2 = the assembled data operator: at lfsr_set_observations the rows a_{k,i} of the stacked
 * A_k = D B W_k whose cells fit a (2R+2)^2 window are summed into a stencil per HR pixel
 * (c_A sum a a^T, the symmetric half stored, (2R+1)-radius), the other rows -- blur windows
 * straddling a depth edge -- are applied as rows (t = c_A a.p, then t a); the NLTV part is formed
 * from the weights m on the fly.  Path 2 needs a single strip, the Gaussian blur, the exact
 * adjoint and nltv_radius <= 2; LFSR_ASM=0 in the environment at lfsr_set_observations keeps
 * path 0.  Results match path 0 to fp32 rounding.  irregular_rows: rows applied as rows (-1 when
 * not read back: lfsr_solve_batch fields after the first), total_rows = n_views h w; setup_ms:
 * wall time of the assembly (synchronised).  Any out pointer except path may be NULL.  Errors:
 * INVALID_ARG (ctx or path NULL), STATE (before lfsr_set_observations). */
LFSR_API lfsr_status lfsr_normal_path(const lfsr_ctx* ctx, int32_t* path, int64_t* irregular_rows,
                                      int64_t* total_rows, double* setup_ms);

/* Row-strip plan of the multi-GPU decomposition (DESIGN 10): rank r
 * owns tile rows [tile_row0, tile_row1) = LR rows [lr_row0, lr_row1) = HR rows
 * [hr_row0, hr_row1); before every operator pass it needs halo_top HR rows above
 * and halo_bottom rows below from its neighbours, and afterwards folds the
 * adjoint contributions it accumulated in those rows back into them.
 * max_shift_rows = ceil(max_k |dtau_k| * max |omega|) (lfsr_set_observations
 * computes it from the data).  Pure host function (no device needed).
 * Errors: INVALID_ARG (params), UNSUPPORTED (a strip thinner than its halo). */
typedef struct {
  int32_t rank, tile_row0, tile_row1, lr_row0, lr_row1, hr_row0, hr_row1, halo_top, halo_bottom;
} lfsr_strip;
LFSR_API lfsr_status lfsr_strip_plan(const lfsr_params* params, int32_t max_shift_rows, lfsr_strip* out /*[n_ranks]*/);

/* The cudaStream_t the ctx runs on (params->stream, or the ctx-owned stream when that
 * was NULL), so a caller that passes device memory can order its own streams against
 * the ctx's (event wait before a call that reads its buffers, and after one that writes
 * them).  Errors: INVALID_ARG (NULL ctx or out). */
LFSR_API lfsr_status lfsr_get_stream(const lfsr_ctx* ctx, void** stream);

/* Free everything; NULL-safe. */
LFSR_API void lfsr_destroy(lfsr_ctx* ctx);

/* Last error message of ctx (or of the last failed lfsr_create if ctx is
 * NULL); owned by the library, valid until the next call on that ctx. */
LFSR_API const char* lfsr_last_error(const lfsr_ctx* ctx);

/* LFSR_ABI_VERSION of the loaded library. */
LFSR_API int32_t lfsr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LFSR_H_ */
