/*
 * oracle.c — plain, slow, obviously-correct fp64 CPU oracle for the ADMM
 * light-field super-resolution hot path of arXiv 2206.05047
 * ("A GPU-Accelerated Light-field Super-resolution Framework Based on Mixed
 * Noise Model and Weighted Regularization").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2206_05047_b200/) never links, imports or calls
 * it, and it shares no code, header, table or constant generator with the
 * CUDA path.
 *
 * Citation key: P:Lnnn = line nnn of PAPER.md (the paper's LaTeX source);
 * S:Lnnn = SPEC.md; readings A1..A27 are listed in DESIGN.md §3 (copied
 * from SURVEY.md §8c.2).  Every operator is its own loop nest in fp64; the
 * composites are literal compositions (A_k = D B W_k) without
 * blocking, fusion or reordering.  Parallelism: OpenMP over output rows of
 * gather-form loops only; the scatter (W_k^T) runs per view into a private
 * buffer and buffers are summed in view order; dot products are per-row
 * partials summed in row order, so results are bit-identical at any thread
 * count.
 *
 * Parity status per function (pins live in tests/test_oracle_pins.py):
 *   or_blur_taps      pinned: App.B closed form, tests/golden/blur_taps.txt
 *   or_apply_D/DT     pinned: definition on 4x4, D D^T = I, adjoint
 *   or_apply_B        pinned: impulse response, constants, adjoint
 *   or_apply_W/WT     pinned: identity, integer/half shifts, axis pairing, adjoint
 *   or_apply_A/AT     pinned: stack adjoint identity
 *   or_apply_S/ST     pinned: constant->0, ramp, adjoint, S^T S brute force
 *   or_weights_m      pinned: sigma->inf limits, constant x
 *   or_setup_wo       pinned: b on ramps, w_o = e^-1 closed form, p~0 noiseless
 *   or_bicubic        pinned: constants, knots, linear reproduction
 *   or_normal         pinned: equals dense c_A A^T A + (th/2) S_W^T S_W, SPD
 *   or_admm           pinned: l2-only == lstsq (P10), == textbook scaled ADMM with exact
 *                     x-step (P11), convergence to an independent minimiser (P12)
 *   or_gradient       pinned: central finite differences of J (P18), J == or_cost
 *   or_apply_WTb      pinned: integer translation == W_k^T in the interior, constants kept,
 *                     inverse of W_k for a constant disparity (P25)
 *   or_apply_Bk/BkT   pinned: the Gaussian outer product == or_apply_B, impulse response
 *                     (convolution orientation), adjoint (P24)
 *   per-view omega    pinned: equal maps == shared mode, view k == shared mode with omega_k,
 *                     adjoint identity (P22)
 *   or_gd             pinned: smooth case with step 1/L decreases J monotonically and reaches the
 *                     lstsq solution (P19); Armijo acceptance checked against or_cost and
 *                     maximality of the step (P20); ADMM below gd at equal CU (P21)
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

#define OR_OK 0
#define OR_ERR_ARG 1
#define OR_ERR_DIVERGED 6

typedef struct {
  int32_t n_views, lr_h, lr_w, scale, ref_view, radius;
  double lambda1, lambda2, lambda_reg;
  double sigma_s, sigma_e, sigma_o1, sigma_o2; /* INFINITY disables a factor */
  double theta;                                 /* ADMM penalty (vartheta) */
  int32_t cg_max_iters;                         /* K */
  double cg_tol;                                /* tau on <r,r> (reading A18) */
  int32_t reweight_every_iter;                  /* 1 = paper */
  const double* offset_weights;                 /* NULL: w_d = exp(-|d|^2/sigma_s); else s_d
                                                   user weights in the U order (BTV, NEXT-1) */
  int32_t disp_per_view;                        /* 0: one omega [H][W] on theta_0's grid for every
                                                   view (A12); 1: omega [n_views][H][W], view k
                                                   warped with its own omega_k (P:L580-582,
                                                   NEXT-2, reading A34) */
  const double* psf;                            /* NULL: the Gaussian B (A11); else a user
                                                   convolution kernel [(2 psf_radius+1)^2]
                                                   row-major (NEXT-4, reading A36) */
  int32_t psf_radius;
  int32_t paper_adjoint;                        /* 0: A_k^T uses the exact transpose W_k^T (A12);
                                                   1: the paper's backward warp W_k^* with omega_0
                                                   in its place (NEXT-2, reading A37) */
} or_params;

/* The disparity map view k is warped with ("for each perspective theta_k, we
 * need to find the disparity map omega_k"): omega_k in per-view mode, else the shared map. */
static const double* omega_of(const or_params* P, const double* omega, int k) {
  return P->disp_per_view ? omega + (size_t)k * P->lr_h * P->scale * P->lr_w * P->scale : omega;
}

typedef struct {
  int32_t iter, cg_iters, breakdown, nonfinite;
  double J, data_l1, data_l2, reg_l1, primal_res, cg_pi0, cg_pi_last;
} or_iter_stats;

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ---------------------------------------------------------------------------
 * Blur taps.  P:L579: "a simple Gaussian kernel with a standard deviation of
 * sigma = 1/4 sqrt(zeta^2 - 1) and a size of 3 sigma" -> reading A11: radius
 * R = ceil(3 sigma), normalised 1-D taps, 2-D kernel = outer product.
 * Returns R; taps[0..2R] (caller provides >= 2R+1 doubles).
 * ------------------------------------------------------------------------- */
int or_blur_taps(int scale, double* taps) {
  double sigma = 0.25 * sqrt((double)scale * scale - 1.0);
  int R = (int)ceil(3.0 * sigma);
  double sum = 0.0;
  for (int u = -R; u <= R; ++u) {
    taps[u + R] = exp(-(double)(u * u) / (2.0 * sigma * sigma));
    sum += taps[u + R];
  }
  for (int u = -R; u <= R; ++u) taps[u + R] /= sum;
  return R;
}

/* D: top-left pick of each zeta x zeta block, P:L577 (reading A14). */
void or_apply_D(int H, int W, int scale, const double* x, double* out) {
  int h = H / scale, w = W / scale;
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < w; ++j) out[(size_t)i * w + j] = x[(size_t)(scale * i) * W + scale * j];
}

/* D^T (D*): put the LR pixel back at the top-left location, zero elsewhere. */
void or_apply_DT(int H, int W, int scale, const double* y, double* out) {
  int h = H / scale, w = W / scale;
  memset(out, 0, sizeof(double) * (size_t)H * W);
  for (int i = 0; i < h; ++i)
    for (int j = 0; j < w; ++j) out[(size_t)(scale * i) * W + scale * j] = y[(size_t)i * w + j];
}

/* B: 2-D Gaussian convolution with zero padding outside Omega (reading A11).
 * (B x)(Y,X) = sum_{u,v} g[u] g[v] x(Y+u, X+v), terms outside Omega dropped.
 * The kernel is symmetric, so B is its own transpose. */
void or_apply_B(int H, int W, int R, const double* taps, const double* x, double* out) {
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      double s = 0.0;
      for (int u = -R; u <= R; ++u)
        for (int v = -R; v <= R; ++v) {
          int yy = Y + u, xx = X + v;
          if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
          s += taps[u + R] * taps[v + R] * x[(size_t)yy * W + xx];
        }
      out[(size_t)Y * W + X] = s;
    }
}

/* B with a user convolution kernel ("the motion blur can be modelled by a
 * convolutional kernel as a realization of the linear operator B"; reading A36):
 *   (B x)(Y,X) = sum_{u,v = -Rp..Rp} k[u+Rp][v+Rp] x(Y-u, X-v), zero outside Omega. */
void or_apply_Bk(int H, int W, int Rp, const double* k, const double* x, double* out) {
  int n = 2 * Rp + 1;
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      double s = 0.0;
      for (int u = -Rp; u <= Rp; ++u)
        for (int v = -Rp; v <= Rp; ++v) {
          int yy = Y - u, xx = X - v;
          if (yy >= 0 && yy < H && xx >= 0 && xx < W) s += k[(u + Rp) * n + (v + Rp)] * x[(size_t)yy * W + xx];
        }
      out[(size_t)Y * W + X] = s;
    }
}

/* Its transpose: (B^T t)(Y,X) = sum_{u,v} k[u+Rp][v+Rp] t(Y+u, X+v) (zero padding). */
void or_apply_BkT(int H, int W, int Rp, const double* k, const double* t, double* out) {
  int n = 2 * Rp + 1;
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      double s = 0.0;
      for (int u = -Rp; u <= Rp; ++u)
        for (int v = -Rp; v <= Rp; ++v) {
          int yy = Y + u, xx = X + v;
          if (yy >= 0 && yy < H && xx >= 0 && xx < W) s += k[(u + Rp) * n + (v + Rp)] * t[(size_t)yy * W + xx];
        }
      out[(size_t)Y * W + X] = s;
    }
}

/* Bilinear sample point of the warp W_k at HR pixel (Y,X), reading A12/A13:
 * z + dtheta_k * omega(z) with theta = [rho, tau], rho pairs with
 * the column axis X and tau with the row axis Y; the continuous
 * coordinate is replicate-clamped into Omega. */
static void warp_point(int H, int W, int Y, int X, double om, double drho, double dtau,
                       int* y0, int* x0, int* y1, int* x1, double* a, double* b) {
  double sy = clampd((double)Y + dtau * om, 0.0, (double)(H - 1));
  double sx = clampd((double)X + drho * om, 0.0, (double)(W - 1));
  *y0 = (int)floor(sy);
  *x0 = (int)floor(sx);
  *y1 = *y0 + 1 < H ? *y0 + 1 : H - 1;
  *x1 = *x0 + 1 < W ? *x0 + 1 : W - 1;
  *a = sy - *y0;
  *b = sx - *x0;
}

/* W_k: forward warp (bilinear gather), "L^(z,theta_k) = L(z + theta_k w_k, theta_k)". */
void or_apply_W(int H, int W, const double* x, const double* omega, double drho, double dtau,
                double* out) {
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      int y0, x0, y1, x1;
      double a, b;
      warp_point(H, W, Y, X, omega[(size_t)Y * W + X], drho, dtau, &y0, &x0, &y1, &x1, &a, &b);
      out[(size_t)Y * W + X] = (1 - a) * (1 - b) * x[(size_t)y0 * W + x0] +
                               (1 - a) * b * x[(size_t)y0 * W + x1] +
                               a * (1 - b) * x[(size_t)y1 * W + x0] + a * b * x[(size_t)y1 * W + x1];
    }
}

/* W_k^T: the exact transpose of the bilinear gather = scatter of the same four
 * weights to the same four indices (reading A12; the paper's own W_k^* is a
 * backward warp, which is not the transpose).  Serial (a scatter). */
void or_apply_WT(int H, int W, const double* t, const double* omega, double drho, double dtau,
                 double* out) {
  memset(out, 0, sizeof(double) * (size_t)H * W);
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      int y0, x0, y1, x1;
      double a, b;
      warp_point(H, W, Y, X, omega[(size_t)Y * W + X], drho, dtau, &y0, &x0, &y1, &x1, &a, &b);
      double v = t[(size_t)Y * W + X];
      out[(size_t)y0 * W + x0] += (1 - a) * (1 - b) * v;
      out[(size_t)y0 * W + x1] += (1 - a) * b * v;
      out[(size_t)y1 * W + x0] += a * (1 - b) * v;
      out[(size_t)y1 * W + x1] += a * b * v;
    }
}

/* The paper's adjoint warp W_k^* ("the backward warping function W_k^* will warp
 * the input SAI from perspective theta_k to theta_0 using omega_0"), reading A37:
 * (W_k^* u)(z) = u(z - dtheta_k omega_0(z)), bilinear, replicate-clamped coordinate (the
 * mirror of W_k's gather, A12).  Not the transpose of W_k. */
void or_apply_WTb(int H, int W, const double* u, const double* omega0, double drho, double dtau,
                  double* out) {
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      int y0, x0, y1, x1;
      double a, b;
      warp_point(H, W, Y, X, omega0[(size_t)Y * W + X], -drho, -dtau, &y0, &x0, &y1, &x1, &a, &b);
      out[(size_t)Y * W + X] = (1 - a) * (1 - b) * u[(size_t)y0 * W + x0] + (1 - a) * b * u[(size_t)y0 * W + x1] +
                               a * (1 - b) * u[(size_t)y1 * W + x0] + a * b * u[(size_t)y1 * W + x1];
    }
}

/* A_k = D B W_k for every view (Eq. sr_model_vec).  out: [n_views][h][w].
 * view_offsets[k] = (drho_k, dtau_k) = theta_k - theta_0 in angular steps. */
void or_apply_A(const or_params* P, const double* view_offsets, const double* omega,
                const double* x, double* out) {
  int z = P->scale, H = P->lr_h * z, W = P->lr_w * z;
  size_t p = (size_t)H * W, q = (size_t)P->lr_h * P->lr_w;
  double taps[64];
  int R = or_blur_taps(z, taps);
  double* t1 = (double*)malloc(sizeof(double) * p);
  double* t2 = (double*)malloc(sizeof(double) * p);
  for (int k = 0; k < P->n_views; ++k) {
    or_apply_W(H, W, x, omega_of(P, omega, k), view_offsets[2 * k], view_offsets[2 * k + 1], t1);
    if (P->psf) or_apply_Bk(H, W, P->psf_radius, P->psf, t1, t2);
    else or_apply_B(H, W, R, taps, t1, t2);
    or_apply_D(H, W, z, t2, out + k * q);
  }
  free(t1);
  free(t2);
}

/* A^T = sum_k W_k^T B^T D^T (Fig. sr_gpu_admm_as): in [n_views][h][w] -> HR.
 * Paper mode (A37): sum_k W_k^* B^T D^T, so "A^T" and the normal operator built on it are
 * no longer transposes (M is not symmetric); the algorithms are run unchanged. */
void or_apply_AT(const or_params* P, const double* view_offsets, const double* omega,
                 const double* r, double* out) {
  int z = P->scale, H = P->lr_h * z, W = P->lr_w * z;
  size_t p = (size_t)H * W, q = (size_t)P->lr_h * P->lr_w;
  double taps[64];
  int R = or_blur_taps(z, taps);
  double* t1 = (double*)malloc(sizeof(double) * p);
  double* t2 = (double*)malloc(sizeof(double) * p);
  double* t3 = (double*)malloc(sizeof(double) * p);
  memset(out, 0, sizeof(double) * p);
  for (int k = 0; k < P->n_views; ++k) {
    or_apply_DT(H, W, z, r + k * q, t1);
    if (P->psf) or_apply_BkT(H, W, P->psf_radius, P->psf, t1, t2);
    else or_apply_B(H, W, R, taps, t1, t2);   /* the Gaussian B is self-adjoint (A11) */
    if (P->paper_adjoint)   /* W_k^* with omega_0 (A37) */
      or_apply_WTb(H, W, t2, omega_of(P, omega, P->ref_view), view_offsets[2 * k], view_offsets[2 * k + 1], t3);
    else
      or_apply_WT(H, W, t2, omega_of(P, omega, k), view_offsets[2 * k], view_offsets[2 * k + 1], t3);
    for (size_t i = 0; i < p; ++i) out[i] += t3[i];
  }
  free(t1);
  free(t2);
  free(t3);
}

/* Offset set U (reading A9): the (2r+1)^2 window minus its centre, row-major
 * with dy outer; s_d = (2r+1)^2 - 1 (24 for the paper's 5x5 window). */
int or_offsets(int radius, int* dys, int* dxs) {
  int n = 0;
  for (int dy = -radius; dy <= radius; ++dy)
    for (int dx = -radius; dx <= radius; ++dx) {
      if (dy == 0 && dx == 0) continue;
      dys[n] = dy;
      dxs[n] = dx;
      ++n;
    }
  return n;
}

/* Spatial weight w_d = exp(-|d|^2 / sigma_s), P:L418 with the decaying sign (reading A8). */
static double spatial_weight(int dy, int dx, double sigma_s) {
  if (isinf(sigma_s)) return 1.0;
  return exp(-(double)(dy * dy + dx * dx) / sigma_s);
}

/* The s_d offset weights w_d: Gaussian in |d| (above), or the caller's list --
 * e.g. BTV's alpha^(|dx|+|dy|) (the regulariser family is fixed by
 * the choice of N(u) and w; MISR use with l1 + BTV). */
static void offset_weights(int radius, double sigma_s, const double* user, double* wd) {
  int dys[1024], dxs[1024];
  int sd = or_offsets(radius, dys, dxs);
  for (int d = 0; d < sd; ++d) wd[d] = user ? user[d] : spatial_weight(dys[d], dxs[d], sigma_s);
}

/* Weighted directional gradient nabla^{U,V}, reading A10:
 *   g_d(z) = W_d(z) (x(z) - x(z+d)) if z+d in Omega, else 0,
 * W_d(z) = w_d * m(z).  out: [s_d][H][W].  wd: the s_d offset weights. */
void or_apply_Sw(int H, int W, int radius, const double* wds, const double* m, const double* x,
                 double* out) {
  int dys[1024], dxs[1024];
  int sd = or_offsets(radius, dys, dxs);
  size_t p = (size_t)H * W;
  for (int d = 0; d < sd; ++d) {
    double wd = wds[d];
#pragma omp parallel for schedule(static)
    for (int Y = 0; Y < H; ++Y)
      for (int X = 0; X < W; ++X) {
        int yy = Y + dys[d], xx = X + dxs[d];
        double g = 0.0;
        if (yy >= 0 && yy < H && xx >= 0 && xx < W)
          g = wd * m[(size_t)Y * W + X] * (x[(size_t)Y * W + X] - x[(size_t)yy * W + xx]);
        out[d * p + (size_t)Y * W + X] = g;
      }
  }
}

/* Weighted directional divergence div^{U,V} taken as the exact
 * transpose of or_apply_S:
 *   (S^T h)(z) = sum_d [ 1{z+d in Omega} W_d(z) h_d(z) - 1{z-d in Omega} W_d(z-d) h_d(z-d) ]. */
void or_apply_STw(int H, int W, int radius, const double* wds, const double* m, const double* h,
                  double* out) {
  int dys[1024], dxs[1024];
  int sd = or_offsets(radius, dys, dxs);
  size_t p = (size_t)H * W;
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      double s = 0.0;
      for (int d = 0; d < sd; ++d) {
        double wd = wds[d];
        int yf = Y + dys[d], xf = X + dxs[d];
        if (yf >= 0 && yf < H && xf >= 0 && xf < W)
          s += wd * m[(size_t)Y * W + X] * h[d * p + (size_t)Y * W + X];
        int yb = Y - dys[d], xb = X - dxs[d];
        if (yb >= 0 && yb < H && xb >= 0 && xb < W)
          s -= wd * m[(size_t)yb * W + xb] * h[d * p + (size_t)yb * W + xb];
      }
      out[(size_t)Y * W + X] = s;
    }
}

/* The same with the Gaussian offset weights exp(-|d|^2 / sigma_s) (reading A8). */
void or_apply_S(int H, int W, int radius, double sigma_s, const double* m, const double* x, double* out) {
  double wd[1024];
  offset_weights(radius, sigma_s, NULL, wd);
  or_apply_Sw(H, W, radius, wd, m, x, out);
}
void or_apply_ST(int H, int W, int radius, double sigma_s, const double* m, const double* h, double* out) {
  double wd[1024];
  offset_weights(radius, sigma_s, NULL, wd);
  or_apply_STw(H, W, radius, wd, m, h, out);
}

/* Per-pixel weight map m = lambda_R * w_o * w_e (W_d = w_d * m),
 * w_e = exp(-|grad x|^2 / sigma_e) with central differences, replicate border
 * (readings A8, A17, A19).  Recomputed from the current x. */
void or_weights_m(int H, int W, double lambda_reg, double sigma_e, const double* wo,
                  const double* x, double* m) {
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      double gx = 0.5 * (x[(size_t)Y * W + clampi(X + 1, 0, W - 1)] - x[(size_t)Y * W + clampi(X - 1, 0, W - 1)]);
      double gy = 0.5 * (x[(size_t)clampi(Y + 1, 0, H - 1) * W + X] - x[(size_t)clampi(Y - 1, 0, H - 1) * W + X]);
      double we = isinf(sigma_e) ? 1.0 : exp(-(gx * gx + gy * gy) / sigma_e);
      m[(size_t)Y * W + X] = lambda_reg * wo[(size_t)Y * W + X] * we;
    }
}

/* Bilinear sample of an LR image at continuous LR (row, col), clamped (reading A17). */
static double bilin_lr(int h, int w, const double* img, double r, double c) {
  r = clampd(r, 0.0, (double)(h - 1));
  c = clampd(c, 0.0, (double)(w - 1));
  int r0 = (int)floor(r), c0 = (int)floor(c);
  int r1 = r0 + 1 < h ? r0 + 1 : h - 1, c1 = c0 + 1 < w ? c0 + 1 : w - 1;
  double a = r - r0, b = c - c0;
  return (1 - a) * (1 - b) * img[(size_t)r0 * w + c0] + (1 - a) * b * img[(size_t)r0 * w + c1] +
         a * (1 - b) * img[(size_t)r1 * w + c0] + a * b * img[(size_t)r1 * w + c1];
}

/* Static occlusion weight (Eq. weight_occ), readings A16/A17 (per-view
 * disparity: the reference view's omega_0, the map on theta_0's grid, A34):
 *   b(z) = min(0, d_X omega + d_Y omega), forward differences, 0 on last col/row;
 *   p(z) = mean_{k != ref} | y_ref(z/zeta) - y_k((z - dtheta_k omega(z))/zeta) |;
 *   w_o  = exp(-b^2 / (2 s1^2)) exp(-p^2 / (2 s2^2)).
 * Optional outputs b_out / p_out may be NULL. */
void or_setup_wo(const or_params* P, const double* y, const double* view_offsets,
                 const double* omega, double* wo, double* b_out, double* p_out) {
  int z = P->scale, h = P->lr_h, w = P->lr_w, H = h * z, W = w * z;
  size_t q = (size_t)h * w;
  const double* yref = y + (size_t)P->ref_view * q;
  omega = omega_of(P, omega, P->ref_view);
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      double om = omega[(size_t)Y * W + X];
      double dx = X + 1 < W ? omega[(size_t)Y * W + X + 1] - om : 0.0;
      double dy = Y + 1 < H ? omega[(size_t)(Y + 1) * W + X] - om : 0.0;
      double b = dx + dy < 0.0 ? dx + dy : 0.0;
      double p = 0.0;
      int cnt = 0;
      double ref = bilin_lr(h, w, yref, (double)Y / z, (double)X / z);
      for (int k = 0; k < P->n_views; ++k) {
        if (k == P->ref_view) continue;
        double drho = view_offsets[2 * k], dtau = view_offsets[2 * k + 1];
        double v = bilin_lr(h, w, y + k * q, ((double)Y - dtau * om) / z, ((double)X - drho * om) / z);
        p += fabs(ref - v);
        ++cnt;
      }
      if (cnt > 0) p /= cnt;
      double f1 = isinf(P->sigma_o1) ? 1.0 : exp(-b * b / (2.0 * P->sigma_o1 * P->sigma_o1));
      double f2 = isinf(P->sigma_o2) ? 1.0 : exp(-p * p / (2.0 * P->sigma_o2 * P->sigma_o2));
      wo[(size_t)Y * W + X] = f1 * f2;
      if (b_out) b_out[(size_t)Y * W + X] = b;
      if (p_out) p_out[(size_t)Y * W + X] = p;
    }
}

/* Keys cubic convolution kernel, a = -0.5 (Catmull-Rom), reading A15. */
static double keys(double t) {
  const double a = -0.5;
  t = fabs(t);
  if (t <= 1.0) return (a + 2.0) * t * t * t - (a + 3.0) * t * t + 1.0;
  if (t < 2.0) return a * t * t * t - 5.0 * a * t * t + 8.0 * a * t - 4.0 * a;
  return 0.0;
}

/* x0 = bicubic up-sampling of the LR reference view, sampled at (Y/zeta, X/zeta)
 * so LR knots land on D's grid, replicate border (reading A15). */
void or_bicubic(int h, int w, int scale, const double* yref, double* out) {
  int H = h * scale, W = w * scale;
#pragma omp parallel for schedule(static)
  for (int Y = 0; Y < H; ++Y)
    for (int X = 0; X < W; ++X) {
      double fy = (double)Y / scale, fx = (double)X / scale;
      int iy = (int)floor(fy), ix = (int)floor(fx);
      double ty = fy - iy, tx = fx - ix;
      double s = 0.0;
      for (int a = -1; a <= 2; ++a)
        for (int b = -1; b <= 2; ++b)
          s += keys(ty - a) * keys(tx - b) *
               yref[(size_t)clampi(iy + a, 0, h - 1) * w + clampi(ix + b, 0, w - 1)];
      out[(size_t)Y * W + X] = s;
    }
}

static double dot(size_t n, const double* a, const double* b, int rows) {
  /* per-row partials summed in row order: deterministic at any thread count */
  size_t cols = n / rows;
  double* part = (double*)malloc(sizeof(double) * rows);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    double s = 0.0;
    for (size_t c = 0; c < cols; ++c) s += a[r * cols + c] * b[r * cols + c];
    part[r] = s;
  }
  double s = 0.0;
  for (int r = 0; r < rows; ++r) s += part[r];
  free(part);
  return s;
}

/* Normal operator of the x-step least squares (Eq. sr_l1l2l1_lsf) in the raw
 * form of reading A7:  M p = (lambda2 + (th/2) lambda1^2) sum_k A_k^T A_k p + (th/2) S^T S p,
 * where S stacks W_d (x) Delta_d (the S of Eq. sr_admm_compact with the weights). */
void or_normal(const or_params* P, const double* view_offsets, const double* omega,
               const double* m, const double* pvec, double* out) {
  int z = P->scale, H = P->lr_h * z, W = P->lr_w * z;
  size_t p = (size_t)H * W, q = (size_t)P->lr_h * P->lr_w;
  int dys[1024], dxs[1024];
  int sd = or_offsets(P->radius, dys, dxs);
  double* ap = (double*)malloc(sizeof(double) * q * P->n_views);
  double* atap = (double*)malloc(sizeof(double) * p);
  double* sp = (double*)malloc(sizeof(double) * p * sd);
  double* stsp = (double*)malloc(sizeof(double) * p);
  or_apply_A(P, view_offsets, omega, pvec, ap);
  or_apply_AT(P, view_offsets, omega, ap, atap);
  double wds[1024];
  offset_weights(P->radius, P->sigma_s, P->offset_weights, wds);
  or_apply_Sw(H, W, P->radius, wds, m, pvec, sp);
  or_apply_STw(H, W, P->radius, wds, m, sp, stsp);
  double cA = P->lambda2 + 0.5 * P->theta * P->lambda1 * P->lambda1;
  for (size_t i = 0; i < p; ++i) out[i] = cA * atap[i] + 0.5 * P->theta * stsp[i];
  free(ap);
  free(atap);
  free(sp);
  free(stsp);
}

static int validate(const or_params* P) {
  if (!P || P->n_views < 1 || P->lr_h < 1 || P->lr_w < 1 || P->scale < 1) return OR_ERR_ARG;
  if (P->ref_view < 0 || P->ref_view >= P->n_views || P->radius < 1 || P->radius > 15) return OR_ERR_ARG;
  if (!(P->theta > 0) || P->lambda1 < 0 || P->lambda2 < 0 || P->lambda_reg < 0) return OR_ERR_ARG;
  if (P->lambda1 + P->lambda2 <= 0 || P->cg_max_iters < 1 || P->cg_tol < 0) return OR_ERR_ARG;
  if (!(P->sigma_s > 0) || !(P->sigma_e > 0) || !(P->sigma_o1 > 0) || !(P->sigma_o2 > 0)) return OR_ERR_ARG;
  if (P->psf && (P->psf_radius < 0 || P->psf_radius > 8)) return OR_ERR_ARG;
  if (P->offset_weights) {
    int sd = (2 * P->radius + 1) * (2 * P->radius + 1) - 1;
    for (int d = 0; d < sd; ++d)
      if (!(P->offset_weights[d] >= 0) || isinf(P->offset_weights[d])) return OR_ERR_ARG;
  }
  return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Algorithm 1 with the x-step of Algorithm 2, raw
 * residual form (readings A5-A7, A23, A26).  Per ADMM iteration n:
 *   m   = weights(x^{n-1})                               (A16)
 *   e_k = A_k x^{n-1} - y_k                              (Alg.1 line 4; A23)
 *   u_A = lambda1 e + w_A ; z_A = soft(u_A, 1/th) ; w_A+ = u_A - z_A = clamp(u_A, +-1/th)
 *   f_A = 2 w_A+ - w_A                                    (Alg.1 lines 5-8)
 *   g_d = W_d Delta_d x ; u_S = g + w_S ; w_S+ = clamp(u_S) ; f_S = 2 w_S+ - w_S
 *   v   = sum_k A_k^T (lambda2 e_k + (th/2) lambda1 f_A,k) + (th/2) S^T f_S   (Alg.1 line 9)
 *   CG on M dx = -v from x^{n-1} (Alg.2 with readings A1-A4):
 *       r = -v; p = r; pi = <r,r>
 *       for k=1..K: if pi < tau or pi == 0 break; q = M p; pq = <p,q>; if pq <= 0 break;
 *                   a = pi/pq; x += a p; r -= a q; pi' = <r,r>; p = r + (pi'/pi) p; pi = pi'
 * Outputs: x_iters [(N+1)][H][W] (x^0..x^N, may be NULL), wA [n_views][h][w],
 * wS [s_d][H][W] (state in/out if state_in != 0), x (in/out, HR), stats [N] (may be NULL).
 * If x0 == NULL the initial x is the bicubic up-sampling of the reference view.
 * ------------------------------------------------------------------------- */
int or_admm(const or_params* P, const double* y, const double* view_offsets,
            const double* omega, const double* x0, int N, double* x_iters, double* x_out,
            double* wA_out, double* wS_out, or_iter_stats* stats) {
  if (validate(P) != OR_OK || N < 0) return OR_ERR_ARG;
  int z = P->scale, h = P->lr_h, w = P->lr_w, H = h * z, W = w * z, K = P->cg_max_iters;
  size_t p = (size_t)H * W, q = (size_t)h * w, nq = q * P->n_views;
  int dys[1024], dxs[1024];
  int sd = or_offsets(P->radius, dys, dxs);
  size_t ns = p * sd;
  double th = P->theta, l1 = P->lambda1, l2 = P->lambda2, inv_th = 1.0 / th;
  double wds[1024];
  offset_weights(P->radius, P->sigma_s, P->offset_weights, wds);

  double* x = (double*)malloc(sizeof(double) * p);
  double* wo = (double*)malloc(sizeof(double) * p);
  double* m = (double*)malloc(sizeof(double) * p);
  double* wA = (double*)calloc(nq, sizeof(double));
  double* wS = (double*)calloc(ns, sizeof(double));
  double* e = (double*)malloc(sizeof(double) * nq);
  double* rho = (double*)malloc(sizeof(double) * nq);
  double* g = (double*)malloc(sizeof(double) * ns);
  double* fS = (double*)malloc(sizeof(double) * ns);
  double* v = (double*)malloc(sizeof(double) * p);
  double* t = (double*)malloc(sizeof(double) * p);
  double* r = (double*)malloc(sizeof(double) * p);
  double* pv = (double*)malloc(sizeof(double) * p);
  double* qv = (double*)malloc(sizeof(double) * p);

  /* Alg.1 lines 1-2: x^(0) := x_0 (bicubic), w^(0) := 0 */
  if (x0) memcpy(x, x0, sizeof(double) * p);
  else or_bicubic(h, w, z, y + (size_t)P->ref_view * q, x);
  or_setup_wo(P, y, view_offsets, omega, wo, NULL, NULL);
  or_weights_m(H, W, P->lambda_reg, P->sigma_e, wo, x, m);
  if (x_iters) memcpy(x_iters, x, sizeof(double) * p);

  int status = OR_OK;
  for (int n = 1; n <= N; ++n) {
    or_iter_stats st;
    memset(&st, 0, sizeof(st));
    st.iter = n;
    if (P->reweight_every_iter) or_weights_m(H, W, P->lambda_reg, P->sigma_e, wo, x, m);

    /* data part: e = A x - y ; prox / dual (clamp form) */
    or_apply_A(P, view_offsets, omega, x, e);
    double dl1 = 0.0, dl2 = 0.0, res = 0.0;
    for (size_t i = 0; i < nq; ++i) {
      e[i] -= y[i];
      double uA = l1 * e[i] + wA[i];
      double wAn = clampd(uA, -inv_th, inv_th);
      double fA = 2.0 * wAn - wA[i];
      rho[i] = l2 * e[i] + 0.5 * th * l1 * fA;
      res += (wAn - wA[i]) * (wAn - wA[i]);
      wA[i] = wAn;
      dl1 += fabs(e[i]);
      dl2 += e[i] * e[i];
    }
    /* NLTV part */
    or_apply_Sw(H, W, P->radius, wds, m, x, g);
    double reg = 0.0;
    for (size_t i = 0; i < ns; ++i) {
      double uS = g[i] + wS[i];
      double wSn = clampd(uS, -inv_th, inv_th);
      fS[i] = 2.0 * wSn - wS[i];
      res += (wSn - wS[i]) * (wSn - wS[i]);
      wS[i] = wSn;
      reg += fabs(g[i]);
    }
    st.data_l1 = dl1;
    st.data_l2 = dl2;
    st.reg_l1 = reg;
    st.J = l1 * dl1 + l2 * dl2 + reg;
    st.primal_res = sqrt(res);

    /* v = A^T rho + (th/2) S^T f_S */
    or_apply_AT(P, view_offsets, omega, rho, v);
    or_apply_STw(H, W, P->radius, wds, m, fS, t);
    for (size_t i = 0; i < p; ++i) v[i] += 0.5 * th * t[i];

    /* x-step: textbook CG (readings A1-A4, A18) */
    for (size_t i = 0; i < p; ++i) { r[i] = -v[i]; pv[i] = r[i]; }
    double pi = dot(p, r, r, H);
    st.cg_pi0 = pi;
    int k;
    for (k = 0; k < K; ++k) {
      if (pi < P->cg_tol || pi == 0.0) break;
      or_normal(P, view_offsets, omega, m, pv, qv);
      double pq = dot(p, pv, qv, H);
      if (!(pq > 0.0)) { st.breakdown = 1; break; }
      double alpha = pi / pq;
      for (size_t i = 0; i < p; ++i) { x[i] += alpha * pv[i]; r[i] -= alpha * qv[i]; }
      double pin = dot(p, r, r, H);
      double beta = pin / pi;
      for (size_t i = 0; i < p; ++i) pv[i] = r[i] + beta * pv[i];
      pi = pin;
    }
    st.cg_iters = k;
    st.cg_pi_last = pi;
    int bad = !isfinite(st.J);
    for (size_t i = 0; i < p && !bad; ++i) bad = !isfinite(x[i]);
    st.nonfinite = bad;
    if (stats) stats[n - 1] = st;
    if (x_iters) memcpy(x_iters + (size_t)n * p, x, sizeof(double) * p);
    if (bad) { status = OR_ERR_DIVERGED; break; }
  }
  if (x_out) memcpy(x_out, x, sizeof(double) * p);
  if (wA_out) memcpy(wA_out, wA, sizeof(double) * nq);
  if (wS_out) memcpy(wS_out, wS, sizeof(double) * ns);
  free(x); free(wo); free(m); free(wA); free(wS); free(e); free(rho); free(g); free(fS);
  free(v); free(t); free(r); free(pv); free(qv);
  return status;
}

/* Cost J (Eq. sr_fin) of an arbitrary x with a given weight map m. */
double or_cost(const or_params* P, const double* y, const double* view_offsets,
               const double* omega, const double* m, const double* x, double* terms3) {
  int z = P->scale, H = P->lr_h * z, W = P->lr_w * z;
  size_t p = (size_t)H * W, nq = (size_t)P->lr_h * P->lr_w * P->n_views;
  int dys[1024], dxs[1024];
  int sd = or_offsets(P->radius, dys, dxs);
  double* e = (double*)malloc(sizeof(double) * nq);
  double* g = (double*)malloc(sizeof(double) * p * sd);
  or_apply_A(P, view_offsets, omega, x, e);
  double l1 = 0, l2 = 0, reg = 0;
  for (size_t i = 0; i < nq; ++i) { double d = e[i] - y[i]; l1 += fabs(d); l2 += d * d; }
  double wds[1024];
  offset_weights(P->radius, P->sigma_s, P->offset_weights, wds);
  or_apply_Sw(H, W, P->radius, wds, m, x, g);
  for (size_t i = 0; i < p * sd; ++i) reg += fabs(g[i]);
  free(e);
  free(g);
  if (terms3) { terms3[0] = l1; terms3[1] = l2; terms3[2] = reg; }
  return P->lambda1 * l1 + P->lambda2 * l2 + reg;
}

/* ---------------------------------------------------------------------------
 * Gradient-descent baselines of the paper's solver comparison (P:L910-933:
 * "gradient descent solver (GD) without and with line search denoted as gd
 * and gd-ls"), with the readings A30-A33 of DESIGN.md §3:
 *   A30  the subgradient of |.| is sgn, with sgn(0) = 0;
 *   A31  the weight map m is re-estimated from x^{n-1} at the start of every
 *        iteration (as for ADMM, A16) and frozen through that
 *        iteration's line search;
 *   A32  line search = Armijo backtracking (c = 1e-4, halving):
 *        eta_t = eta0 * 2^-t for t = 0..L-1, the first t with
 *        J(x - eta_t g) <= J(x) - c * eta_t * |g|^2 is taken; if none is,
 *        no step is taken (x unchanged) and ls_failed = 1;
 *   A33  CU accounting: the cost J (A and S) is one CU, the
 *        gradient (A^T and S^T) one CU, every line-search trial one CU;
 *        an ADMM iteration counts 2(K+1).
 * ------------------------------------------------------------------------- */
static double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

/* Cost terms and subgradient of J (Eq. sr_fin) at x for a given
 * weight map m (W_d = w_d m):
 *   e_k = A_k x - y_k ,  G = S_w x  (G_d(z) = W_d(z) (x(z) - x(z+d)))
 *   terms3 = (sum|e|, sum e^2, sum|G|)
 *   g = sum_k A_k^T (l1 sgn(e_k) + 2 l2 e_k) + S_w^T sgn(G)           (A30)
 * Returns J = l1 terms3[0] + l2 terms3[1] + terms3[2].  g may be NULL. */
double or_gradient(const or_params* P, const double* y, const double* view_offsets,
                   const double* omega, const double* m, const double* x, double* g,
                   double* terms3) {
  int z = P->scale, H = P->lr_h * z, W = P->lr_w * z;
  size_t p = (size_t)H * W, nq = (size_t)P->lr_h * P->lr_w * P->n_views;
  int dys[1024], dxs[1024];
  int sd = or_offsets(P->radius, dys, dxs);
  size_t ns = p * sd;
  double wds[1024];
  offset_weights(P->radius, P->sigma_s, P->offset_weights, wds);
  double* e = (double*)malloc(sizeof(double) * nq);
  double* G = (double*)malloc(sizeof(double) * ns);
  or_apply_A(P, view_offsets, omega, x, e);
  double l1 = 0.0, l2 = 0.0, reg = 0.0;
  for (size_t i = 0; i < nq; ++i) {
    e[i] -= y[i];
    l1 += fabs(e[i]);
    l2 += e[i] * e[i];
  }
  or_apply_Sw(H, W, P->radius, wds, m, x, G);
  for (size_t i = 0; i < ns; ++i) reg += fabs(G[i]);
  if (g) {
    double* t = (double*)malloc(sizeof(double) * p);
    for (size_t i = 0; i < nq; ++i) e[i] = P->lambda1 * sgn(e[i]) + 2.0 * P->lambda2 * e[i];
    for (size_t i = 0; i < ns; ++i) G[i] = sgn(G[i]);
    or_apply_AT(P, view_offsets, omega, e, g);
    or_apply_STw(H, W, P->radius, wds, m, G, t);
    for (size_t i = 0; i < p; ++i) g[i] += t[i];
    free(t);
  }
  free(e);
  free(G);
  if (terms3) { terms3[0] = l1; terms3[1] = l2; terms3[2] = reg; }
  return P->lambda1 * l1 + P->lambda2 * l2 + reg;
}

typedef struct {
  int32_t iter, ls_evals, ls_failed, nonfinite;
  double J, data_l1, data_l2, reg_l1, step, grad_sq;
} or_gd_stats;

/* gd / gd-ls (A30-A33).  Per iteration n, from x = x^{n-1}:
 *   m = weights(x) (A31) ; J0, g = or_gradient(x, m) ; gsq = <g, g>
 *   fixed step:  x := x - eta0 g
 *   line search: for t = 0..L-1: eta = eta0 2^-t ; if J(x - eta g; m) <= J0 - c eta gsq:
 *                x := x - eta g, stop  (A32)
 * stats[n-1] = (n, trials evaluated, failed, nonfinite, J0 and its terms, eta taken, gsq).
 * x_iters [(N+1)][H][W] (may be NULL), x_out [H][W] (may be NULL); x0 NULL => bicubic. */
int or_gd(const or_params* P, const double* y, const double* view_offsets, const double* omega,
          const double* x0, int N, double step0, int line_search, int max_halvings, double armijo_c,
          double* x_iters, double* x_out, or_gd_stats* stats) {
  if (validate(P) != OR_OK || N < 0 || !(step0 > 0) || max_halvings < 1 || armijo_c < 0) return OR_ERR_ARG;
  int z = P->scale, h = P->lr_h, w = P->lr_w, H = h * z, W = w * z;
  size_t p = (size_t)H * W, q = (size_t)h * w;
  double* x = (double*)malloc(sizeof(double) * p);
  double* xt = (double*)malloc(sizeof(double) * p);
  double* g = (double*)malloc(sizeof(double) * p);
  double* wo = (double*)malloc(sizeof(double) * p);
  double* m = (double*)malloc(sizeof(double) * p);
  if (x0) memcpy(x, x0, sizeof(double) * p);
  else or_bicubic(h, w, z, y + (size_t)P->ref_view * q, x);
  or_setup_wo(P, y, view_offsets, omega, wo, NULL, NULL);
  or_weights_m(H, W, P->lambda_reg, P->sigma_e, wo, x, m);
  if (x_iters) memcpy(x_iters, x, sizeof(double) * p);
  int status = OR_OK;
  for (int n = 1; n <= N; ++n) {
    or_gd_stats st;
    memset(&st, 0, sizeof(st));
    st.iter = n;
    if (P->reweight_every_iter) or_weights_m(H, W, P->lambda_reg, P->sigma_e, wo, x, m);
    double t3[3];
    double J0 = or_gradient(P, y, view_offsets, omega, m, x, g, t3);
    double gsq = dot(p, g, g, H);
    st.J = J0;
    st.data_l1 = t3[0];
    st.data_l2 = t3[1];
    st.reg_l1 = t3[2];
    st.grad_sq = gsq;
    double eta = step0;
    if (line_search) {
      int ok = 0;
      for (int t = 0; t < max_halvings; ++t) {
        double et = ldexp(step0, -t);
        for (size_t i = 0; i < p; ++i) xt[i] = x[i] - et * g[i];
        double Jt = or_gradient(P, y, view_offsets, omega, m, xt, NULL, NULL);
        st.ls_evals = t + 1;
        if (Jt <= J0 - armijo_c * et * gsq) { eta = et; ok = 1; break; }
      }
      if (!ok) { eta = 0.0; st.ls_failed = 1; }
    }
    st.step = eta;
    for (size_t i = 0; i < p; ++i) x[i] -= eta * g[i];
    int bad = !isfinite(J0);
    for (size_t i = 0; i < p && !bad; ++i) bad = !isfinite(x[i]);
    st.nonfinite = bad;
    if (stats) stats[n - 1] = st;
    if (x_iters) memcpy(x_iters + (size_t)n * p, x, sizeof(double) * p);
    if (bad) { status = OR_ERR_DIVERGED; break; }
  }
  if (x_out) memcpy(x_out, x, sizeof(double) * p);
  free(x); free(xt); free(g); free(wo); free(m);
  return status;
}

/* ---------------------------------------------------------------------------
 * Colour input ("solve the cost function for Y color channel while
 * applying bi-cubic interpolation for Cb and Cr channel"), reading A35: full-range
 * ITU-R BT.601 YCbCr on [0, 1]:
 *   Y = 0.299 R + 0.587 G + 0.114 B,  Cb = 0.5 + (B - Y)/1.772,  Cr = 0.5 + (R - Y)/1.402
 * and its inverse.  Planar [3][n] RGB.  (Pinned: P23, tests/test_oracle_color.py.)
 * ------------------------------------------------------------------------- */
void or_rgb_to_ycbcr(size_t n, const double* rgb, double* y, double* cb, double* cr) {
  for (size_t i = 0; i < n; ++i) {
    double r = rgb[i], g = rgb[n + i], b = rgb[2 * n + i];
    y[i] = 0.299 * r + 0.587 * g + 0.114 * b;
    cb[i] = 0.5 + (b - y[i]) / 1.772;
    cr[i] = 0.5 + (r - y[i]) / 1.402;
  }
}

void or_ycbcr_to_rgb(size_t n, const double* y, const double* cb, const double* cr, double* rgb) {
  for (size_t i = 0; i < n; ++i) {
    double r = y[i] + 1.402 * (cr[i] - 0.5);
    double b = y[i] + 1.772 * (cb[i] - 0.5);
    rgb[i] = r;
    rgb[n + i] = (y[i] - 0.299 * r - 0.114 * b) / 0.587;
    rgb[2 * n + i] = b;
  }
}
