// capi.cu — the C ABI of liblfsr (include/lfsr.h): validation, device state,
// CUDA-graph capture of one ADMM iteration (Alg.1) and its replay,
// and the HR row-strip decomposition over several GPUs.
#include "../../include/lfsr.h"
#include "internal.h"
#include "nccl_shim.h"
#include <nvtx3/nvToolsExt.h>   // header-only; ranges show in nsys / ncu when a tool is attached

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

namespace lfsr {
TileGeom make_tile_geom(const Geom& G, int num_sms, int tr0, int tr1);
void tile_static(int scale, int& BL, int& LX, int& R, int& KEEP);
int tile_bl_candidates(int scale, int* out, int cap);
int tile_max_warps(int scale);
int tile_max_warps_normal(int scale);
cudaError_t prepare_tile_kernels(int scale, size_t smem);
cudaError_t launch_tile(int mode, const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                        cudaStream_t st);
cudaError_t launch_setup_wo(const Geom& G, const Views& V, const float* y, const float* omega, float* wo,
                            cudaStream_t st);
cudaError_t launch_bicubic(const Geom& G, const float* y, float* x, cudaStream_t st);
cudaError_t launch_density(const Geom& G, const Views& V, const float* omega, float* D, cudaStream_t st);
cudaError_t launch_weights(const Geom& G, const float* x, const float* wo, float* m, cudaStream_t st);
cudaError_t launch_absmax(const float* v, size_t n, unsigned* out, cudaStream_t st);
cudaError_t launch_cg_update(const Geom& G, float* x, float* r, const float* p, float* q, Control* ctl, int k,
                             int row0, int nrows, int close_here, int num_sms, cudaStream_t st);
cudaError_t launch_close(const Geom& G, Control* ctl, cudaStream_t st);
cudaError_t launch_apply_S(const Geom& G, const float* x, const float* m, float* out, cudaStream_t st);
cudaError_t launch_apply_ST(const Geom& G, const float* h, const float* m, float* out, cudaStream_t st);
cudaError_t launch_fold_rows(float* dst, float* src, size_t n, int zero_src, cudaStream_t st);
cudaError_t launch_allreduce_local(Control* const* ctls, int nparts, int slot0, int count, cudaStream_t st);
cudaError_t launch_gd_gnorm(const Geom& G, const float* g, Control* ctl, int num_sms, cudaStream_t st);
cudaError_t launch_paper_gather(const Geom& G, const Views& V, const float* rho, const float* omega0, const float* p,
                                float* out, float sign, Control* ctl, int slot, int cg_k, int row0, int nrows,
                                cudaStream_t st);
cudaError_t launch_color(int to_ycbcr, const float* a, float* y, float* cb, float* cr, size_t n, int num_sms,
                         cudaStream_t st);
cudaError_t launch_cgcg_update(const Geom& G, float* x, float* r, float* p, float* s, float* w, Control* ctl, int j,
                               int row0, int nrows, int num_sms, cudaStream_t st);
cudaError_t launch_wz_nltv(const Geom& G, const float* x, const float* m, float* wS0, float* wS1, float* r,
                           Control* ctl, int row0, int row1, cudaStream_t st);
cudaError_t launch_omega_const(const Geom& G, const float* omega, unsigned* flag, cudaStream_t st);
cudaError_t launch_misr_normal(const Geom& G, const MisrStencil& S, const MisrArgs& a, cudaStream_t st);
cudaError_t prepare_misr_kernels();
cudaError_t launch_asm_build(const Geom& G, const Views& V, const AsmBuf& B, float om_max, cudaStream_t st);
cudaError_t launch_asm_step(const Geom& G, const Views& V, const AsmBuf& B, const AsmStep& s, bool irr, int num_sms,
                            cudaStream_t st, cudaEvent_t mid, const AsmFork& fk);
cudaError_t prepare_asm_kernels();
int asm_plane_count(int scale);
int asm_row_floats(int scale);
cudaError_t launch_gd_update(const Geom& G, float* x, const float* g, Control* ctl, const GdCfg& cfg, int num_sms,
                             cudaStream_t st);
}  // namespace lfsr

using namespace lfsr;

namespace {

constexpr int kRingCap = 4096;  // stats records kept on the device

enum XMode { X_NONE = 0, X_LOCAL = 1, X_NCCL = 2 };

// One HR row strip: its own rows, full-size buffers (only the own rows and the
// halos are meaningful) and its tile geometry.
struct Part {
  lfsr_strip plan{};
  State S{};
  TileGeom T{};
  // strips: the tiles whose input tile lies in the own rows (no halo needed; they run on the side
  // stream while the halos are exchanged) and the rest (after the exchange)
  TileGeom Tin{}, Tbd{};
  int* d_tl = nullptr;
  double* ring = nullptr;
  float* stage[2] = {nullptr, nullptr};  // NCCL fold staging: [0] rows from the previous rank, [1] from the next
  size_t stage_rows = 0;
};

}  // namespace

struct lfsr_ctx {
  lfsr_params prm{};
  Geom G{};
  Views V{};
  TileGeom Tfull{};          // whole-image tiles (test operators)
  std::vector<Part> parts;   // 1 (single GPU / NCCL rank) or n_ranks (virtual ranks)
  XMode xmode = X_NONE;
  void* comm = nullptr;      // ncclComm_t (NCCL mode)
  Control** d_ctls = nullptr;  // device array of the parts' control blocks (virtual ranks)
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr};   // set_observations: y copy on cap_stream overlapping the omega setup
  // lfsr_solve_batch: the next field's inputs are staged (copied, maxima) on cap_stream while
  // the current field solves; graph execs replaced during a batch are retired, not destroyed
  float* stage_y = nullptr;
  float* stage_om = nullptr;
  float* stage_dens = nullptr;
  unsigned* stage_umax = nullptr;
  unsigned* h_ubits = nullptr;     // pinned [3]
  Control* h_ctl = nullptr;        // pinned control-block image
  double* h_rec = nullptr;         // pinned [batch][T_COUNT] last-iteration records
  int h_rec_cap = 0;
  cudaEvent_t ev_b[2] = {nullptr, nullptr};   // [0] staged, [1] previous field solved
  bool retire = false;
  std::vector<cudaGraphExec_t> retired;
  bool own_stream = false;
  bool poisoned = false;
  bool ready = false;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};  // replay for even / odd iteration parity
  int launches_per_iter = 0;
  std::vector<void*> allocs;
  float* tmp_hr2 = nullptr;
  float* tmp_s = nullptr;
  unsigned* umax = nullptr;
  Control* tune_ctl = nullptr;   // scratch control block for the tile-height timing
  int h_iter = 0;                // iterations enqueued since set_observations
  int solver = 0;                // 0: none yet, 1: ADMM, 2: gd (one solver per set_observations)
  cudaGraphExec_t gd_graph = nullptr;   // one gd / gd-ls iteration (built for gd_cfg)
  GdCfg gd_cfg{};
  int gd_launches = 0;
  float* gd_g = nullptr;         // gd subgradient buffer [H][ps]
  Control* op_ctl = nullptr;     // scratch control block of lfsr_op_apply (keeps the solver sums clean)
  size_t alloc_key[7] = {0, 0, 0, 0, 0, 0, 0};
  bool profile = false;          // event-record nodes around every kernel (single strip)
  std::vector<cudaEvent_t> prof_ev;
  double prof_ms[3] = {0, 0, 0}; // accumulated wz / normal / update milliseconds
  int64_t prof_n[3] = {0, 0, 0};
  // MISR fast path (misr.cu): constant disparity -> the CG operator's data part
  // as a precomputed zeta^2-phase stencil on Z_s, the exact tile kernel on the border tiles
  cudaStream_t side = nullptr;      // strips: interior tiles overlap the halo exchange
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool misr = false;
  bool in_batch = false;           // lfsr_solve_batch swaps fields under one graph: no fast path there
  MisrStencil* misr_S = nullptr;   // host copy (passed by value to k_misr_normal)
  MisrArgs misr_a{};               // regions (pointers filled per launch)
  TileGeom Tborder{};              // c->Tfull restricted to the border tiles
  int* d_tlist = nullptr;
  int tlist_cap = 0;
  float* d_misr_tab = nullptr;     // separable form: T_y [H][2WR+1], T_x [W][2WR+1]
  size_t misr_tab_bytes = 0;
  bool misr_border = true;         // the dense form runs the border tiles through k_tile
  // assembled data normal operator (asm.cu): the regular rows of the stacked A_k as
  // a stencil per HR pixel, the irregular rows (blur windows across a depth edge) applied as rows
  bool asmop = false;
  AsmBuf asmb{};
  int64_t asm_nirr = -1;           // irregular rows (host copy; -1 = not read back: batch fields)
  double asm_ms = 0.0;             // wall time of the last assembly (set_observations, synchronised)
  int batch_iters = 0;             // lfsr_solve_batch: ADMM iterations per field (path choice amortisation)
  std::vector<cudaEvent_t> asm_ev; // profiling: after the stencil kernel of CG step k (index k)
  double prof_asm_ms[2] = {0, 0};  // accumulated stencil-kernel / irregular-row milliseconds
  int64_t prof_asm_n = 0;
  std::string err;
};

static thread_local std::string g_create_err;

// NVTX range for the host side of an API call or a setup phase (SURVEY §5 tracing)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

#define FAIL(ctx, code, msg)          \
  do {                                \
    (ctx)->err = (msg);               \
    return (code);                    \
  } while (0)

static lfsr_status cuda_fail(lfsr_ctx* c, cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error in %s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  c->err = buf;
  c->poisoned = true;
  return LFSR_ERR_CUDA;
}

static lfsr_status nccl_fail(lfsr_ctx* c, int e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof buf, "NCCL error in %s: %s", what, nccl_error(e));
  c->err = buf;
  c->poisoned = true;
  return LFSR_ERR_NCCL;
}

#define CK(c, expr)                                               \
  do {                                                            \
    cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) return cuda_fail((c), _e, #expr);      \
  } while (0)

#define NK(c, expr)                                               \
  do {                                                            \
    int _e = (expr);                                              \
    if (_e != 0) return nccl_fail((c), _e, #expr);                \
  } while (0)

static int round_up(int v, int m) { return (v + m - 1) / m * m; }

static const char* validate(const lfsr_params* p) {
  if (!p) return "params is NULL";
  if (p->n_views < 1 || p->n_views > kMaxViews) return "n_views must be in [1, 1024]";
  if (p->lr_height < 1 || p->lr_width < 1) return "lr_height and lr_width must be >= 1";
  if (p->scale < 2 || p->scale > 4) return "scale must be 2, 3 or 4";
  if (p->ref_view < 0 || p->ref_view >= p->n_views) return "ref_view out of range";
  if (p->nltv_radius < 1 || p->nltv_radius > 4) return "nltv_radius must be in [1, 4]";
  if (!(p->lambda1 >= 0.f) || !(p->lambda2 >= 0.f) || !(p->lambda1 + p->lambda2 > 0.f))
    return "lambda1, lambda2 must be >= 0 with lambda1 + lambda2 > 0";
  if (!(p->lambda_reg >= 0.f) || !std::isfinite(p->lambda_reg)) return "lambda_reg must be finite and >= 0";
  if (!(p->sigma_s > 0.f) || !(p->sigma_e > 0.f) || !(p->sigma_o1 > 0.f) || !(p->sigma_o2 > 0.f))
    return "sigma_s, sigma_e, sigma_o1, sigma_o2 must be > 0 (INFINITY disables)";
  if (!(p->theta > 0.f) || !std::isfinite(p->theta)) return "theta must be finite and > 0";
  if (p->cg_max_iters < 1 || p->cg_max_iters > kMaxK) return "cg_max_iters must be in [1, 64]";
  if (!(p->cg_tol >= 0.f)) return "cg_tol must be >= 0";
  if (p->reweight_every_iter != 0 && p->reweight_every_iter != 1) return "reweight_every_iter must be 0 or 1";
  if (p->offset_weights) {
    const int sd = (2 * p->nltv_radius + 1) * (2 * p->nltv_radius + 1) - 1;
    for (int d = 0; d < sd; ++d)
      if (!(p->offset_weights[d] >= 0.f) || !std::isfinite(p->offset_weights[d]))
        return "offset_weights must be finite and >= 0";
  }
  if (p->psf) {
    // kernels up to the Gaussian's window (R = 2 at scale 2, 3 at 3, 4) run in the default tile
    // instances, larger ones (up to 15x15) in the kPsfBigR instances
    if (p->psf_radius < 0 || p->psf_radius > kPsfBigR) return "psf_radius must be in [0, 7]";
    const int n = (2 * p->psf_radius + 1) * (2 * p->psf_radius + 1);
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(p->psf[i])) return "psf must be finite";
  }
  if (p->paper_adjoint != 0 && p->paper_adjoint != 1) return "paper_adjoint must be 0 or 1";
  if (p->device < 0) return "device must be >= 0";
  if (p->n_ranks < 1 || p->n_ranks > 1024) return "n_ranks must be in [1, 1024]";
  if (p->n_ranks == 1 && p->rank != 0) return "rank must be 0 when n_ranks == 1";
  if (p->n_ranks > 1 && (p->rank < -1 || p->rank >= p->n_ranks)) return "rank must be in [-1, n_ranks)";
  if (p->n_ranks > 1 && p->rank >= 0 && !p->nccl_unique_id) return "NCCL mode (rank >= 0) needs nccl_unique_id";
  if (p->lr_height * (size_t)p->scale > (1u << 20) || p->lr_width * (size_t)p->scale > (1u << 20))
    return "image too large";
  return nullptr;
}

static float inv_or_zero(double s, double mul) { return std::isinf(s) ? 0.f : (float)(1.0 / (mul * s)); }

static void fill_geom(const lfsr_params& p, Geom& G) {
  G = Geom{};
  G.h = p.lr_height;
  G.w = p.lr_width;
  G.scale = p.scale;
  G.H = p.lr_height * p.scale;
  G.W = p.lr_width * p.scale;
  G.ps = round_up(G.W, 32);
  G.lps = round_up(G.w, 32);
  G.n_views = p.n_views;
  G.ref_view = p.ref_view;
  G.radius = p.nltv_radius;
  G.K = p.cg_max_iters;
  G.lambda1 = p.lambda1;
  G.lambda2 = p.lambda2;
  G.lambda_reg = p.lambda_reg;
  G.theta = p.theta;
  G.inv_theta = 1.f / p.theta;
  G.inv_sigma_e = inv_or_zero(p.sigma_e, 1.0);
  G.inv_2s1sq = std::isinf(p.sigma_o1) ? 0.f : (float)(1.0 / (2.0 * (double)p.sigma_o1 * p.sigma_o1));
  G.inv_2s2sq = std::isinf(p.sigma_o2) ? 0.f : (float)(1.0 / (2.0 * (double)p.sigma_o2 * p.sigma_o2));
  G.cg_tol = p.cg_tol;
  G.cA = (float)((double)p.lambda2 + 0.5 * p.theta * (double)p.lambda1 * p.lambda1);
  G.cS = 0.5f * p.theta;
  // Gaussian PSF: sigma = 1/4 sqrt(zeta^2 - 1), radius ceil(3 sigma), normalised (A11)
  double sig = 0.25 * std::sqrt((double)p.scale * p.scale - 1.0);
  int R = (int)std::ceil(3.0 * sig);
  G.R = R;
  double sum = 0.0, t[2 * kMaxTaps + 1];
  for (int u = -R; u <= R; ++u) sum += (t[u + R] = std::exp(-(double)u * u / (2.0 * sig * sig)));
  for (int u = 0; u <= 2 * R; ++u) G.taps[u] = (float)(t[u] / sum);
  auto tap = [&](int u) { return u <= 2 * R ? G.taps[u] : 0.f; };
  for (int v = 0; v <= kMaxTaps; ++v) {
    G.tpe[v] = make_float2(tap(2 * v), tap(2 * v + 1));
    G.tpo[v] = make_float2(tap(2 * v + 1), tap(2 * v + 2));
  }
  double gmax = 0.0;
  for (int ph = 0; ph < p.scale; ++ph) {
    double sp = 0.0;
    for (int u = ph; u <= 2 * R; u += p.scale) sp += t[u] / sum;
    gmax = std::fmax(gmax, sp);
  }
  G.gpoly2 = (float)(gmax * gmax * 1.0001);
  G.ksum = 1.f;
  G.paper = p.paper_adjoint;
  if (p.psf) {   // user blur kernel (A36): flip into the E-offset order of the tile kernel
    G.psf2d = 1;
    const int rp = p.psf_radius, np_ = 2 * rp + 1;
    const int rb = rp > R ? kPsfBigR : R;   // layout radius: the default or the large-kernel instances
    G.psf_rb = rb;
    double ks = 0.0, gp = 0.0;
    for (int u = -rp; u <= rp; ++u)
      for (int v = -rp; v <= rp; ++v) {
        const float k = p.psf[(u + rp) * np_ + (v + rp)];
        G.psf2[rb - u][rb - v] = k;
        ks += std::fabs((double)k);
      }
    // |B^T D^T rho| <= max over phases of the polyphase |k| sums times max|rho|
    for (int py = 0; py < p.scale; ++py)
      for (int px = 0; px < p.scale; ++px) {
        double sp = 0.0;
        for (int a = py; a <= 2 * rb; a += p.scale)
          for (int b = px; b <= 2 * rb; b += p.scale) sp += std::fabs((double)G.psf2[a][b]);
        gp = std::fmax(gp, sp);
      }
    G.ksum = (float)(ks * 1.0001);
    G.gpoly2 = (float)(gp * 1.0001);
  }
  // NLTV offsets U and spatial weights w_d = exp(-|d|^2/sigma_s) (A8, A9)
  int n = 0;
  for (int dy = -p.nltv_radius; dy <= p.nltv_radius; ++dy)
    for (int dx = -p.nltv_radius; dx <= p.nltv_radius; ++dx) {
      if (!dy && !dx) continue;
      G.ody[n] = (int8_t)dy;
      G.odx[n] = (int8_t)dx;
      G.wd[n] = p.offset_weights ? p.offset_weights[n]
                : std::isinf(p.sigma_s) ? 1.f : (float)std::exp(-(double)(dy * dy + dx * dx) / p.sigma_s);
      ++n;
    }
  G.s_d = n;
}

// Row-strip plan: contiguous tile rows per rank, as even as possible.
static lfsr_status make_plan(const Geom& G, int n_ranks, int max_shift_rows, std::vector<lfsr_strip>& out,
                             std::string& err) {
  int BL, LX, R, KEEP;
  tile_static(G.scale, BL, LX, R, KEEP);
  if (G.tile_bl > 0) BL = G.tile_bl;
  const int ntY = (G.h + BL - 1) / BL;
  const int sye = std::max(max_shift_rows, G.radius);
  const int top = R + sye + 1;          // input-tile rows above the own rows (see k_tile)
  const int bot = KEEP - R + sye + 1;   // ... and below
  if (n_ranks > ntY) {
    err = "more ranks than tile rows (" + std::to_string(ntY) + ")";
    return LFSR_ERR_UNSUPPORTED;
  }
  out.assign(n_ranks, lfsr_strip{});
  int tr = 0;
  for (int r = 0; r < n_ranks; ++r) {
    const int cnt = ntY / n_ranks + (r < ntY % n_ranks ? 1 : 0);
    lfsr_strip& s = out[r];
    s.rank = r;
    s.tile_row0 = tr;
    s.tile_row1 = tr + cnt;
    s.lr_row0 = tr * BL;
    s.lr_row1 = std::min((tr + cnt) * BL, G.h);
    s.hr_row0 = s.lr_row0 * G.scale;
    s.hr_row1 = s.lr_row1 * G.scale;
    s.halo_top = r > 0 ? top : 0;
    s.halo_bottom = r + 1 < n_ranks ? bot : 0;
    tr += cnt;
    if (n_ranks > 1 && s.hr_row1 - s.hr_row0 < std::max(top, bot)) {
      err = "strip of " + std::to_string(s.hr_row1 - s.hr_row0) + " HR rows is thinner than its halo (" +
            std::to_string(std::max(top, bot)) + "); use fewer ranks";
      return LFSR_ERR_UNSUPPORTED;
    }
  }
  return LFSR_OK;
}

extern "C" {

int32_t lfsr_abi_version(void) { return LFSR_ABI_VERSION; }

// Colour conversion (reading A35), device arrays, stream-ordered.
static lfsr_status color_call(int to_ycbcr, const float* rgb, float* y, float* cb, float* cr, size_t n_pixels,
                              void* stream) {
  if (!rgb || !y || !cb || !cr) return LFSR_ERR_INVALID_ARG;
  if (n_pixels == 0) return LFSR_OK;
  for (const void* p : {(const void*)rgb, (const void*)y, (const void*)cb, (const void*)cr}) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      return LFSR_ERR_INVALID_ARG;
    }
  }
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (launch_color(to_ycbcr, rgb, y, cb, cr, n_pixels, sms, (cudaStream_t)stream) != cudaSuccess) {
    cudaGetLastError();
    return LFSR_ERR_CUDA;
  }
  return LFSR_OK;
}
lfsr_status lfsr_rgb_to_ycbcr(const float* rgb, float* y, float* cb, float* cr, size_t n_pixels, void* stream) {
  return color_call(1, rgb, y, cb, cr, n_pixels, stream);
}
lfsr_status lfsr_ycbcr_to_rgb(const float* y, const float* cb, const float* cr, float* rgb, size_t n_pixels,
                              void* stream) {
  return color_call(0, rgb, const_cast<float*>(y), const_cast<float*>(cb), const_cast<float*>(cr), n_pixels, stream);
}

lfsr_status lfsr_strip_plan(const lfsr_params* params, int32_t max_shift_rows, lfsr_strip* out) {
  if (const char* why = validate(params)) {
    g_create_err = why;
    return LFSR_ERR_INVALID_ARG;
  }
  if (!out || max_shift_rows < 0) {
    g_create_err = "out is NULL or max_shift_rows < 0";
    return LFSR_ERR_INVALID_ARG;
  }
  Geom G;
  fill_geom(*params, G);
  std::vector<lfsr_strip> plan;
  lfsr_status st = make_plan(G, params->n_ranks, max_shift_rows, plan, g_create_err);
  if (st != LFSR_OK) return st;
  for (int r = 0; r < params->n_ranks; ++r) out[r] = plan[r];
  return LFSR_OK;
}

lfsr_status lfsr_create(const lfsr_params* params, lfsr_ctx** out) {
  NvtxRange nvtx_("lfsr_create");
  if (!out) {
    g_create_err = "out is NULL";
    return LFSR_ERR_INVALID_ARG;
  }
  if (const char* why = validate(params)) {
    g_create_err = why;
    return LFSR_ERR_INVALID_ARG;
  }
  if (params->paper_adjoint && (params->n_ranks > 1 || params->psf)) {
    g_create_err = "the paper-mode adjoint (paper_adjoint) runs on a single strip with the Gaussian blur";
    return LFSR_ERR_UNSUPPORTED;
  }
  if (params->psf && params->n_ranks > 1 && params->psf_radius > (params->scale == 2 ? 2 : 3)) {
    g_create_err = "a user blur kernel larger than the Gaussian window runs on a single strip";
    return LFSR_ERR_UNSUPPORTED;
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev <= params->device) {
    g_create_err = std::string("no usable CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "ordinal out of range");
    return LFSR_ERR_CUDA;
  }
  lfsr_ctx* c = new (std::nothrow) lfsr_ctx();
  if (!c) {
    g_create_err = "host allocation failed";
    return LFSR_ERR_OOM;
  }
  c->prm = *params;
  if ((e = cudaSetDevice(params->device)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, params->device)) != cudaSuccess) {
    g_create_err = std::string("cudaSetDevice/attribute failed: ") + cudaGetErrorString(e);
    delete c;
    return LFSR_ERR_CUDA;
  }
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, params->device);
  if (major != 10) {
    g_create_err = "liblfsr is built for sm_100a (B200) only";
    delete c;
    return LFSR_ERR_UNSUPPORTED;
  }
  if (params->stream) {
    c->stream = (cudaStream_t)params->stream;
  } else {
    if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) {
      g_create_err = cudaGetErrorString(e);
      delete c;
      return LFSR_ERR_CUDA;
    }
    c->own_stream = true;
  }
  if ((e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking)) != cudaSuccess) {
    g_create_err = cudaGetErrorString(e);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return LFSR_ERR_CUDA;
  }
  if (params->n_ranks > 1 &&
      ((e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking)) != cudaSuccess ||
       (e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
       (e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming)) != cudaSuccess)) {
    g_create_err = cudaGetErrorString(e);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    cudaStreamDestroy(c->cap_stream);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return LFSR_ERR_CUDA;
  }
  fill_geom(c->prm, c->G);
  c->prm.stream = c->stream;
  c->prm.offset_weights = nullptr;   // consumed into G (the caller keeps ownership)
  c->prm.psf = nullptr;
  if (params->n_ranks > 1) {
    c->xmode = params->rank < 0 ? X_LOCAL : X_NCCL;
    if (c->xmode == X_NCCL) {
      std::string why;
      if (!nccl_available(&why)) {
        g_create_err = why;
        cudaStreamDestroy(c->cap_stream);
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
        return LFSR_ERR_NCCL;
      }
      int r = nccl_comm_init(&c->comm, params->n_ranks, params->nccl_unique_id, params->rank);
      if (r != 0) {
        g_create_err = std::string("ncclCommInitRank: ") + nccl_error(r);
        cudaStreamDestroy(c->cap_stream);
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
        return LFSR_ERR_NCCL;
      }
    }
  }
  *out = c;
  return LFSR_OK;
}

static void free_graph(lfsr_ctx* c) {
  for (auto& g : c->graph)
    if (g) {
      if (c->retire) c->retired.push_back(g);   // launches may still be pending (lfsr_solve_batch)
      else cudaGraphExecDestroy(g);
      g = nullptr;
    }
  if (c->gd_graph) {
    cudaGraphExecDestroy(c->gd_graph);
    c->gd_graph = nullptr;
  }
}

static void free_state(lfsr_ctx* c) {
  free_graph(c);
  for (void* p : c->allocs) cudaFree(p);
  c->allocs.clear();
  c->parts.clear();
  c->tmp_hr2 = nullptr;
  c->tmp_s = nullptr;
  c->gd_g = nullptr;
  c->stage_y = c->stage_om = c->stage_dens = nullptr;
  c->stage_umax = nullptr;
  c->op_ctl = nullptr;
  c->umax = nullptr;
  c->d_ctls = nullptr;
  c->d_tlist = nullptr;
  c->tlist_cap = 0;
  c->d_misr_tab = nullptr;
  c->misr_tab_bytes = 0;
  c->misr = false;
  c->asmop = false;
  c->asmb = AsmBuf{};
  for (auto& k : c->alloc_key) k = 0;
  c->ready = false;
}

void lfsr_destroy(lfsr_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->prm.device);
  if (!c->poisoned) cudaStreamSynchronize(c->stream);
  free_state(c);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->asm_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_in)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_b)
    if (e) cudaEventDestroy(e);
  for (cudaGraphExec_t g : c->retired) cudaGraphExecDestroy(g);
  if (c->h_ubits) cudaFreeHost(c->h_ubits);
  if (c->h_ctl) cudaFreeHost(c->h_ctl);
  if (c->h_rec) cudaFreeHost(c->h_rec);
  delete c->misr_S;
  if (c->comm) {
    if (c->poisoned) nccl_comm_abort(c->comm);
    else nccl_comm_destroy(c->comm);
  }
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

lfsr_status lfsr_get_stream(const lfsr_ctx* c, void** stream) {
  if (!c || !stream) return LFSR_ERR_INVALID_ARG;
  *stream = (void*)c->stream;
  return LFSR_OK;
}

const char* lfsr_last_error(const lfsr_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int32_t lfsr_launches_per_iter(const lfsr_ctx* c) { return (c && c->ready) ? c->launches_per_iter : 0; }

lfsr_status lfsr_fast_path(const lfsr_ctx* c, int32_t* active, int32_t* rect) {
  if (!c || !active) return LFSR_ERR_INVALID_ARG;
  if (!c->ready) return LFSR_ERR_STATE;
  *active = c->misr ? 1 : 0;
  if (rect) {
    const MisrArgs& a = c->misr_a;
    const int32_t v[8] = {a.zs_y0, a.zs_y1, a.zs_x0, a.zs_x1, a.o_y0, a.o_y1, a.o_x0, a.o_x1};
    for (int i = 0; i < 8; ++i) rect[i] = c->misr ? v[i] : 0;
  }
  return LFSR_OK;
}

lfsr_status lfsr_normal_path(const lfsr_ctx* c, int32_t* path, int64_t* irregular_rows, int64_t* total_rows,
                             double* setup_ms) {
  if (!c || !path) return LFSR_ERR_INVALID_ARG;
  if (!c->ready) return LFSR_ERR_STATE;
  *path = c->misr ? 1 : (c->asmop ? 2 : 0);
  if (irregular_rows) *irregular_rows = c->asmop ? c->asm_nirr : 0;
  if (total_rows) *total_rows = (int64_t)c->G.n_views * c->G.h * c->G.w;
  if (setup_ms) *setup_ms = c->asmop ? c->asm_ms : 0.0;
  return LFSR_OK;
}

lfsr_status lfsr_tile_config(const lfsr_ctx* c, int32_t* tile_rows, int32_t* view_groups, int32_t* warps_per_cta,
                             int32_t* cg_warps_per_cta) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (!c->ready || c->parts.empty()) return LFSR_ERR_STATE;
  const TileGeom& T = c->parts[0].T;
  if (tile_rows) *tile_rows = T.BL;
  if (view_groups) *view_groups = T.groups;
  if (warps_per_cta) *warps_per_cta = T.nwarps;
  if (cg_warps_per_cta) *cg_warps_per_cta = T.nwarps_n;
  return LFSR_OK;
}

static cudaError_t dalloc(lfsr_ctx* c, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess) {
    c->allocs.push_back(*p);
    e = cudaMemsetAsync(*p, 0, bytes, c->stream);
  }
  return e;
}

static lfsr_status check_ptr(lfsr_ctx* c, const void* p, lfsr_mem mem, const char* name) {
  if (!p) {
    c->err = std::string(name) + " is NULL";
    return LFSR_ERR_INVALID_ARG;
  }
  if (mem == LFSR_MEM_DEVICE) {
    cudaPointerAttributes a{};
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess || a.type != cudaMemoryTypeDevice || a.device != c->prm.device) {
      cudaGetLastError();
      c->err = std::string(name) + " is not device memory of the ctx device";
      return LFSR_ERR_INVALID_ARG;
    }
  } else if (mem != LFSR_MEM_HOST) {
    c->err = "mem must be LFSR_MEM_HOST or LFSR_MEM_DEVICE";
    return LFSR_ERR_INVALID_ARG;
  }
  return LFSR_OK;
}

static cudaMemcpyKind kind_in(lfsr_mem mem) { return mem == LFSR_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice; }
static cudaMemcpyKind kind_out(lfsr_mem mem) { return mem == LFSR_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice; }

// Copy a dense [rows][cols] array into a pitched [rows][pitch] device array.
static cudaError_t put2d(lfsr_ctx* c, float* dst, int pitch, const float* src, int cols, size_t rows, lfsr_mem mem,
                         cudaStream_t st = nullptr) {
  return cudaMemcpy2DAsync(dst, (size_t)pitch * 4, src, (size_t)cols * 4, (size_t)cols * 4, rows, kind_in(mem),
                           st ? st : c->stream);
}
static cudaError_t get2d(lfsr_ctx* c, float* dst, int cols, const float* src, int pitch, size_t rows, lfsr_mem mem) {
  return cudaMemcpy2DAsync(dst, (size_t)cols * 4, src, (size_t)pitch * 4, (size_t)cols * 4, rows, kind_out(mem), c->stream);
}

static lfsr_status build_graphs(lfsr_ctx* c);

// Buffers of one strip (full image size: only own rows and halos are meaningful).
static lfsr_status alloc_part(lfsr_ctx* c, Part& P) {
  const Geom& G = c->G;
  State& S = P.S;
  const size_t hr = (size_t)G.H * G.ps, lr = (size_t)G.n_views * G.h * G.lps;
  const size_t ws = (size_t)G.s_d * hr;
  void* p = nullptr;
#define ALLOC(field, bytes)                                                                                 \
  do {                                                                                                      \
    cudaError_t _e = dalloc(c, &p, (bytes));                                                                \
    if (_e != cudaSuccess) {                                                                                \
      cudaGetLastError();                                                                                   \
      free_state(c);                                                                                        \
      FAIL(c, _e == cudaErrorMemoryAllocation ? LFSR_ERR_OOM : LFSR_ERR_CUDA, "device allocation failed"); \
    }                                                                                                       \
    field = (decltype(field))p;                                                                             \
  } while (0)
  ALLOC(S.x, hr * 4);
  ALLOC(S.y, lr * 4);
  ALLOC(S.wA, lr * 4);
  ALLOC(S.wS[0], ws * 4);
  ALLOC(S.wS[1], ws * 4);
  ALLOC(S.density, hr * 4);
  ALLOC(S.omega, hr * 4 * (G.per_view ? (size_t)G.n_views : 1));
  ALLOC(S.wo, hr * 4);
  ALLOC(S.m, hr * 4);
  ALLOC(S.r, hr * 4);
  ALLOC(S.p[0], hr * 4);
  ALLOC(S.p[1], hr * 4);
  ALLOC(S.q, hr * 4);
  ALLOC(S.tmp_hr, hr * 4);
  ALLOC(S.tmp_lr, lr * 4);
  if (G.paper) ALLOC(S.rho, lr * 4);
  ALLOC(S.ctl, sizeof(Control));
  ALLOC(P.ring, (size_t)kRingCap * T_COUNT * sizeof(double));
#undef ALLOC
  return LFSR_OK;
}

static TileIO base_io(const Part& P);

// Strip plan and tile geometry of every part for the current G.tile_bl.
static lfsr_status setup_tiles(lfsr_ctx* c) {
  const Geom& G = c->G;
  const int nparts = (int)c->parts.size();
  lfsr_status st;
  std::vector<lfsr_strip> plan;
  if (c->prm.n_ranks > 1) {
    std::string why;
    if ((st = make_plan(G, c->prm.n_ranks, G.SY, plan, why)) != LFSR_OK) FAIL(c, st, why);
  } else {
    plan.resize(1);
    make_plan(G, 1, G.SY, plan, c->err);
  }
  for (int i = 0; i < nparts; ++i) {
    Part& P = c->parts[i];
    P.plan = plan[c->xmode == X_NCCL ? c->prm.rank : i];
    P.T = make_tile_geom(G, c->num_sms, P.plan.tile_row0, P.plan.tile_row1);
    if (P.T.smem > 227 * 1024) FAIL(c, LFSR_ERR_UNSUPPORTED, "disparity range too large for the shared-memory tile");
    if (c->prm.n_ranks > 1) {   // interior tiles: the input tile (E region + disparity halo) inside the own rows
      const TileGeom& T = P.T;
      const int reach_up = T.SYe + 1 + (T.EY - T.TY) + 0, zt = G.scale * T.BL;
      std::vector<int> in_l, bd_l;
      for (int t = 0; t < T.ntYl; ++t) {
        const int y0 = (T.tY0 + t) * zt;                        // own HR rows of the tile row
        const int R = G.R;
        const int top = y0 - R - T.SYe - 1, bot = y0 + T.EY - R + T.SYe + 1;   // input rows [top, bot)
        (void)reach_up;
        const bool up_ok = P.plan.halo_top == 0 || top >= P.plan.hr_row0;
        const bool dn_ok = P.plan.halo_bottom == 0 || bot <= P.plan.hr_row1;
        for (int tx = 0; tx < T.ntX; ++tx) (up_ok && dn_ok ? in_l : bd_l).push_back(t * T.ntX + tx);
      }
      if (!P.d_tl) {
        void* p = nullptr;
        cudaError_t e;
        if ((e = dalloc(c, &p, (size_t)(T.ntY + 1) * T.ntX * sizeof(int))) != cudaSuccess) return cuda_fail(c, e, "alloc");
        P.d_tl = (int*)p;
      }
      std::vector<int> all(in_l);
      all.insert(all.end(), bd_l.begin(), bd_l.end());
      if (!all.empty())
        CK(c, cudaMemcpyAsync(P.d_tl, all.data(), all.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
      CK(c, cudaStreamSynchronize(c->stream));   // `all` is a local
      P.Tin = T;
      P.Tin.tlist = P.d_tl;
      P.Tin.ntl = (int)in_l.size();
      P.Tbd = T;
      P.Tbd.tlist = P.d_tl + in_l.size();
      P.Tbd.ntl = (int)bd_l.size();
    }
    if (c->xmode == X_NCCL) {  // fold staging, sized by the halos
      const size_t rows = (size_t)std::max(P.plan.halo_top, P.plan.halo_bottom) + 64;
      if (P.stage_rows < rows) {
        void* p = nullptr;
        cudaError_t e;
        if ((e = dalloc(c, &p, rows * G.ps * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
        P.stage[0] = (float*)p;
        if ((e = dalloc(c, &p, rows * G.ps * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
        P.stage[1] = (float*)p;
        P.stage_rows = rows;
      }
    }
  }
  c->Tfull = make_tile_geom(G, c->num_sms, -1, -1);
  if (c->Tfull.smem > 227 * 1024) FAIL(c, LFSR_ERR_UNSUPPORTED, "disparity range too large for the shared-memory tile");
  size_t smem_max = std::max(c->Tfull.smem, c->Tfull.smem_normal);   // must cover every launch
  for (const Part& P : c->parts) smem_max = std::max(smem_max, std::max(P.T.smem, P.T.smem_normal));
  CK(c, prepare_tile_kernels(G.scale, smem_max));

  return LFSR_OK;
}

// Tile height (LR rows per tile).  Wave quantisation and the shared-memory
// footprint make the best value depend on the problem and the GPU, so a single
// strip times the CG normal-operator kernel for a few candidates on the first
// set_observations of a geometry and remembers the winner for the process
// (same geometry => same tiling => bit-identical reruns).  LFSR_TILE_BL=<n>
// forces a height; strip decompositions use the zeta default (their plan must
// match lfsr_strip_plan, which has no observations to tune on).
static std::mutex g_tune_mu;
struct TileChoice {
  int bl, g, nw, nwn;   // nwn: warps of the CG-operator launches
};
static std::map<std::string, TileChoice> g_tuned;

static std::string tune_key(const lfsr_ctx* c) {
  const Geom& G = c->G;
  char k[256];
  snprintf(k, sizeof k, "%d/%d/%d/%d/%d/%d/%d/%d/%d/%d", c->prm.device, G.scale, G.h, G.w, G.n_views, G.SX, G.SY,
           G.radius, c->num_sms, G.psf2d ? G.psf_rb : 0);
  return k;
}

static void initial_tiles(lfsr_ctx* c, bool* tune) {
  Geom& G = c->G;
  *tune = false;
  G.tile_bl = G.tile_g = G.tile_nw = G.tile_nwn = 0;
  if (const char* e = getenv("LFSR_TILE_BL")) {
    const int v = atoi(e);
    if (v > 0) G.tile_bl = v;
  }
  if (const char* e = getenv("LFSR_TILE_GNW")) {   // "groups,warps"
    int g = 0, w = 0;
    if (sscanf(e, "%d,%d", &g, &w) == 2 && g > 0 && w > 0) { G.tile_g = g; G.tile_nw = w; }
  }
  if (const char* e = getenv("LFSR_TILE_NWN")) {   // warps of the CG-operator launches
    const int v = atoi(e);
    if (v > 0) G.tile_nwn = v;
  }
  if (G.tile_bl || G.tile_g || c->xmode != X_NONE) return;
  std::lock_guard<std::mutex> lk(g_tune_mu);
  auto it = g_tuned.find(tune_key(c));
  if (it != g_tuned.end()) {
    G.tile_bl = it->second.bl;
    G.tile_g = it->second.g;
    G.tile_nw = it->second.nw;
    G.tile_nwn = it->second.nwn;
    return;
  }
  *tune = true;
}

static lfsr_status tune_tile_bl(lfsr_ctx* c) {
  Geom& G = c->G;
  Part& P = c->parts[0];
  if (!c->tune_ctl) {
    void* p = nullptr;
    cudaError_t e;
    if ((e = dalloc(c, &p, sizeof(Control))) != cudaSuccess) return cuda_fail(c, e, "alloc");
    c->tune_ctl = (Control*)p;
  }
  int cand[8];
  const int n = tile_bl_candidates(G.scale, cand, 8);
  const bool big = G.psf2d && G.psf_rb == kPsfBigR;   // large user kernel: 8-warp instances
  const int maxw = big ? 8 : tile_max_warps(G.scale);
  cudaEvent_t e0, e1;
  CK(c, cudaEventCreate(&e0));
  CK(c, cudaEventCreate(&e1));
  TileChoice best{0, 0, 0, 0};
  float best_ms = 1e30f;
  for (int i = 0; i < n; ++i) {
    if (cand[i] > G.h && i > 0) continue;
    // per height: the cost model's groups/warps, and 1-3 groups of maximal CTAs
    const int gnw[4][2] = {{0, 0}, {1, maxw}, {2, maxw}, {3, maxw}};
    int model_g = 0, model_w = 0;
    for (int j = 0; j < 4; ++j) {
      G.tile_bl = cand[i];
      G.tile_g = gnw[j][0];
      G.tile_nw = gnw[j][1];
      TileGeom T = make_tile_geom(G, c->num_sms, -1, -1);
      if (T.smem > 227 * 1024) continue;
      if (j == 0) {
        model_g = T.groups;
        model_w = T.nwarps;
      } else if (T.groups == model_g && T.nwarps == model_w) {
        continue;
      }
      CK(c, prepare_tile_kernels(G.scale, T.smem));
      TileIO io = base_io(P);
      io.ctl = c->tune_ctl;
      io.in_hr = P.S.x;
      io.out_hr = P.S.tmp_hr;
      io.cg_k = 0;
      io.do_nltv = 1;
      CK(c, cudaMemsetAsync(c->tune_ctl, 0, sizeof(Control), c->stream));
      CK(c, launch_tile(MODE_NORMAL, G, c->V, T, io, c->stream));     // warm
      CK(c, cudaEventRecord(e0, c->stream));
      for (int r = 0; r < 3; ++r) CK(c, launch_tile(MODE_NORMAL, G, c->V, T, io, c->stream));
      CK(c, cudaEventRecord(e1, c->stream));
      CK(c, cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(c, cudaEventElapsedTime(&ms, e0, e1));
      if (getenv("LFSR_TUNE_VERBOSE"))
        fprintf(stderr, "lfsr tile tuning: BL %d groups %d warps %d  %.1f us\n", cand[i], T.groups, T.nwarps,
                ms * 1000.f / 3);
      if (ms < best_ms * 0.98f) {   // a later candidate must win by 2 % (stable choice)
        best_ms = ms;
        best = TileChoice{cand[i], T.groups, T.nwarps, T.nwarps};
      }
    }
  }
  // the CG-operator launches may use wider CTAs than the wz-step (zeta = 2: up to 16 warps):
  // kept if 2 % faster for the chosen tiling
  const int maxwn = big ? 8 : tile_max_warps_normal(G.scale);
  if (maxwn > best.nw && best.bl > 0) {
    G.tile_bl = best.bl;
    G.tile_g = best.g;
    G.tile_nw = best.nw;
    G.tile_nwn = maxwn;
    TileGeom T = make_tile_geom(G, c->num_sms, -1, -1);
    if (T.smem_normal <= 227 * 1024 && T.nwarps_n == maxwn) {
      CK(c, prepare_tile_kernels(G.scale, std::max(T.smem, T.smem_normal)));
      TileIO io = base_io(P);
      io.ctl = c->tune_ctl;
      io.in_hr = P.S.x;
      io.out_hr = P.S.tmp_hr;
      io.do_nltv = 1;
      CK(c, cudaMemsetAsync(c->tune_ctl, 0, sizeof(Control), c->stream));
      CK(c, launch_tile(MODE_NORMAL, G, c->V, T, io, c->stream));     // warm
      CK(c, cudaEventRecord(e0, c->stream));
      for (int r = 0; r < 3; ++r) CK(c, launch_tile(MODE_NORMAL, G, c->V, T, io, c->stream));
      CK(c, cudaEventRecord(e1, c->stream));
      CK(c, cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(c, cudaEventElapsedTime(&ms, e0, e1));
      if (getenv("LFSR_TUNE_VERBOSE"))
        fprintf(stderr, "lfsr tile tuning: BL %d groups %d warps %d, CG operator %d warps  %.1f us\n", best.bl,
                best.g, best.nw, maxwn, ms * 1000.f / 3);
      if (ms < best_ms * 0.98f) best.nwn = maxwn;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CK(c, cudaMemsetAsync(P.S.tmp_hr, 0, (size_t)G.H * G.ps * 4, c->stream));
  G.tile_bl = best.bl;
  G.tile_g = best.g;
  G.tile_nw = best.nw;
  G.tile_nwn = best.nwn;
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    g_tuned[tune_key(c)] = best;
  }
  return setup_tiles(c);
}

// Halo of the input tile around the E region: S = ceil(max_k |dtheta_k| max|omega|)
// per axis, evaluated in double (a huge finite product must not overflow the int).  The tile
// kernel samples inside the replicate-padded tile without clamping, so a shift reaching past the
// image (every sample of such a view clamps to the border) is outside what it supports.
static lfsr_status set_shift_halo(lfsr_ctx* c, float om_max, float mx_rho, float mx_tau) {
  Geom& G = c->G;
  if (!std::isfinite(om_max)) FAIL(c, LFSR_ERR_INVALID_ARG, "disparity must be finite (NaN or inf found)");
  const double sx = std::ceil((double)mx_rho * (double)om_max), sy = std::ceil((double)mx_tau * (double)om_max);
  if (sx > (double)G.W || sy > (double)G.H)
    FAIL(c, LFSR_ERR_UNSUPPORTED, "max |view offset| x max |disparity| exceeds the image size");
  G.SX = (int)sx;
  G.SY = (int)sy;
  return LFSR_OK;
}


// ---------------------------------------------------------------------------
// MISR fast path (misr.cu).  With a constant disparity c every view is a
// global shift s_k = dtheta_k c; the operator A_k = D B W_k is then, per axis, the composition
// of 1-D maps, A_k = A_k^y (x) A_k^x away from the border, and the data normal operator is the
// zeta^2-phase stencil S[phase][dy][dx] = c_A sum_k T_k^y[phase_y][dy] T_k^x[phase_x][dx] with
// T_k[phi][D] = sum_l A_k[l, z0] A_k[l, z0 + D] (z0 = phi mod zeta, interior).  Assembled here in
// fp64 with the oracle's arithmetic (samples at Y + dtau c, X + drho c in double, A13), rounded
// to fp32 once.  Z_s: the outputs whose contributing LR pixels all have unclamped, unpadded rows
// (per axis, brute force); the border tiles: every tile holding an LR pixel that reaches an output
// outside Z_s, or owning such an output.
// ---------------------------------------------------------------------------
struct Axis1 {
  int lo = 0, hi = 0;          // Z_s on this axis: [lo, hi)
  std::vector<char> lb;        // LR index belongs to a border tile band
};

static void misr_axis(int N, int n, int Z, int R, int rad, const std::vector<int>& nk, const std::vector<double>& fk,
                      Axis1& out) {
  const int K = (int)nk.size();
  auto interior = [&](int l) {
    if (l < 0 || l >= n) return false;
    for (int u = -R; u <= R; ++u) {
      const int a = Z * l + u;
      if (a < 0 || a > N - 1) return false;
      for (int k = 0; k < K; ++k)
        if (a + nk[k] < 0 || a + nk[k] + (fk[k] > 0.0 ? 1 : 0) > N - 1) return false;
    }
    return true;
  };
  std::vector<char> lin(n);
  for (int l = 0; l < n; ++l) lin[l] = interior(l);
  std::vector<char> valid(N, 0);
  for (int z = 0; z < N; ++z) {
    bool ok = z >= rad && z < N - rad;
    for (int k = 0; k < K && ok; ++k)
      for (int e = 0; e <= 1 && ok; ++e)
        for (int u = -R; u <= R && ok; ++u) {
          const int t = z - u - nk[k] - e;   // = Z l
          if (((t % Z) + Z) % Z) continue;
          const int l = (t - ((t % Z) + Z) % Z) / Z;
          if (l < 0 || l >= n || !lin[l]) ok = false;
        }
    valid[z] = ok;
  }
  // largest run of valid outputs
  int best_lo = 0, best_len = 0;
  for (int z = 0; z < N;) {
    if (!valid[z]) { ++z; continue; }
    int e = z;
    while (e < N && valid[e]) ++e;
    if (e - z > best_len) { best_len = e - z; best_lo = z; }
    z = e;
  }
  out.lo = best_lo;
  out.hi = best_lo + best_len;
  out.lb.assign(n, 0);
  for (int l = 0; l < n; ++l)
    for (int k = 0; k < K; ++k)
      for (int e = 0; e <= 1; ++e)
        for (int u = -R; u <= R; ++u) {
          const int z = std::min(std::max(Z * l + u + nk[k] + e, 0), N - 1);
          if (z < out.lo || z >= out.hi) out.lb[l] = 1;
        }
  for (int z = 0; z < N; ++z)
    if (z < out.lo || z >= out.hi) out.lb[std::min(z / Z, n - 1)] = 1;
}

// T[phi][D + 2WR'] for one view along one axis (interior): sum over the LR rows l of A[l, z0] A[l, z0 + D].
static void misr_T(int Z, int R, const std::vector<double>& g, int nk, double fk, std::vector<double>& T) {
  const int WR = 2 * R + 1, NW = 2 * WR + 1;
  T.assign((size_t)Z * NW, 0.0);
  const int L0 = 100000;   // a virtual interior LR index (far from any shift)
  for (int phi = 0; phi < Z; ++phi) {
    const int z0 = Z * L0 + phi;
    const int lc = (z0 - nk) / Z;   // the LR rows that reach z0 lie within R + 1 of z0 - nk
    for (int l = lc - R - 2; l <= lc + R + 2; ++l) {
      // row of A along this axis: positions Z l + u + nk + e with weight g[u] w(e)
      double row[64];
      int base = Z * l - R + nk;   // position of index 0
      for (int i = 0; i < 64; ++i) row[i] = 0.0;
      for (int u = -R; u <= R; ++u) {
        row[u + R] += g[u + R] * (1.0 - fk);
        row[u + R + 1] += g[u + R] * fk;
      }
      const int i0 = z0 - base;
      if (i0 < 0 || i0 > 2 * R + 1 || row[i0] == 0.0) continue;
      for (int i = 0; i <= 2 * R + 1; ++i) {
        const int D = base + i - z0;
        if (D < -WR || D > WR || row[i] == 0.0) continue;
        T[(size_t)phi * NW + D + WR] += row[i0] * row[i];
      }
    }
  }
}

// The exact banded 1-D matrix T = A^T A of one view along one axis, border included: A[l, .] =
// sum_u g[u] x (bilinear weights of the sample at clamp(Z l + u + shift, 0, N - 1)), positions
// Z l + u outside [0, N) dropped (blur zero padding, A11), y1 = min(y0 + 1, N - 1) (A12/A13, the
// oracle's arithmetic in fp64).  Row z holds T[z][z + D], |D| <= 2R + 1.
static void misr_T_exact(int N, int n, int Z, int R, const std::vector<double>& g, double shift,
                         std::vector<double>& T) {
  const int WR = 2 * R + 1, NW = 2 * WR + 1;
  T.assign((size_t)N * NW, 0.0);
  std::vector<std::pair<int, double>> row;
  for (int l = 0; l < n; ++l) {
    row.clear();
    for (int u = -R; u <= R; ++u) {
      const int a = Z * l + u;
      if (a < 0 || a > N - 1) continue;
      const double s = std::fmin(std::fmax((double)a + shift, 0.0), (double)(N - 1));
      const int y0 = (int)std::floor(s), y1 = std::min(y0 + 1, N - 1);
      const double f = s - y0;
      row.emplace_back(y0, g[u + R] * (1.0 - f));
      row.emplace_back(y1, g[u + R] * f);
    }
    for (const auto& i : row)
      for (const auto& j : row) {
        const int D = j.first - i.first;
        if (D < -WR || D > WR) continue;   // cannot happen (|D| <= 2R + 1), kept as a guard
        T[(size_t)i.first * NW + D + WR] += i.second * j.second;
      }
  }
}

static lfsr_status misr_setup(lfsr_ctx* c, float omega_c) {
  Geom& G = c->G;
  c->misr = false;
  const char* env = getenv("LFSR_MISR_FAST");
  if (env && env[0] == '0') return LFSR_OK;
  if (c->in_batch || c->xmode != X_NONE || G.per_view || G.psf2d || G.paper || G.radius != 2 || G.s_d != 24)
    return LFSR_OK;
  const int Z = G.scale, R = G.R, WR = 2 * R + 1, NW = 2 * WR + 1;
  if ((size_t)Z * Z * NW * NW > (size_t)kMisrMaxCoef) return LFSR_OK;
  const int K = G.n_views;
  std::vector<int> ny(K), nx(K);
  std::vector<double> fy(K), fx(K);
  for (int k = 0; k < K; ++k) {
    const double sy = (double)c->V.off[k].y * (double)omega_c, sx = (double)c->V.off[k].x * (double)omega_c;
    ny[k] = (int)std::floor(sy);
    fy[k] = sy - ny[k];
    nx[k] = (int)std::floor(sx);
    fx[k] = sx - nx[k];
  }
  Axis1 ay, ax;
  misr_axis(G.H, G.h, Z, R, G.radius, ny, fy, ay);
  misr_axis(G.W, G.w, Z, R, G.radius, nx, fx, ax);
  const bool interior_ok = ay.hi - ay.lo >= 2 * Z && ax.hi - ax.lo >= 2 * Z;   // dense form: an interior worth it
  // Gaussian taps in fp64 (A11), as fill_geom
  const double sig = 0.25 * std::sqrt((double)Z * Z - 1.0);
  std::vector<double> g(2 * R + 1);
  double sum = 0.0;
  for (int u = -R; u <= R; ++u) sum += (g[u + R] = std::exp(-(double)u * u / (2.0 * sig * sig)));
  for (double& v : g) v /= sum;
  if (!c->misr_S) c->misr_S = new MisrStencil;
  MisrStencil& S = *c->misr_S;
  memset(&S, 0, sizeof S);
  std::vector<double> acc((size_t)Z * Z * NW * NW, 0.0), Ty, Tx;
  const double cA = (double)G.lambda2 + 0.5 * (double)G.theta * (double)G.lambda1 * (double)G.lambda1;
  for (int k = 0; k < K; ++k) {
    misr_T(Z, R, g, ny[k], fy[k], Ty);
    misr_T(Z, R, g, nx[k], fx[k], Tx);
    for (int py = 0; py < Z; ++py)
      for (int px = 0; px < Z; ++px)
        for (int dy = 0; dy < NW; ++dy)
          for (int dx = 0; dx < NW; ++dx)
            acc[(((size_t)py * Z + px) * NW + dy) * NW + dx] += Ty[(size_t)py * NW + dy] * Tx[(size_t)px * NW + dx];
  }
  for (size_t i = 0; i < acc.size(); ++i) S.s[i] = (float)(cA * acc[i]);
  const bool sep = true;   // candidate; the separable form is decided on the exact 1-D matrices below
  double W2 = 0.0;
  for (int d = 0; d < 24; ++d) {
    S.w2[d] = G.wd[d] * G.wd[d];
    S.w2f[d] = G.wd[23 - d] * G.wd[23 - d];   // -d in the A9 order (the window is symmetric)
    W2 += (double)S.w2[d];
  }
  S.W2 = (float)W2;
  // separable NLTV weights: w_d^2 = u[dy] u[dx] (d != 0) with symmetric weights (Gaussian w_d, BTV)
  {
    auto w2 = [&](int dy, int dx) {
      const int lin = (dy + 2) * 5 + (dx + 2);
      return (double)G.wd[lin > 12 ? lin - 1 : lin] * (double)G.wd[lin > 12 ? lin - 1 : lin];
    };
    double u[5] = {0, 0, 0, 0, 0};
    const double w11 = w2(1, 1);
    bool ok = sep && w11 > 0.0;
    if (ok) {
      u[2] = std::sqrt(w2(0, 1) * w2(1, 0) / w11);
      ok = u[2] > 0.0;
    }
    if (ok) {
      for (int t = -2; t <= 2; ++t)
        if (t) u[t + 2] = w2(t, 0) / u[2];
      double emax = 0.0, vmax = 0.0;
      for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
          if (!dy && !dx) continue;
          emax = std::fmax(emax, std::fabs(u[dy + 2] * u[dx + 2] - w2(dy, dx)));
          emax = std::fmax(emax, std::fabs(w2(-dy, -dx) - w2(dy, dx)));   // symmetric (w_{-d} = w_d)
          vmax = std::fmax(vmax, w2(dy, dx));
        }
      ok = emax <= 1e-6 * vmax;
    }
    S.sep = ok ? 1 : 0;
    for (int t = 0; t < 5; ++t) S.u[t] = (float)u[t];
  }
  if (S.sep) {
    // exact 1-D matrices, border included: M_data = c_A sum_a T_y,a (x) X_a with one class left,
    // so the stencil covers the whole image and no border kernel runs
    std::vector<std::pair<double, std::vector<double>>> ycls;   // (y shift, sum of the class's T_x)
    std::vector<double> Ex, Ey;
    for (int k = 0; k < K; ++k) {
      const double sy = (double)c->V.off[k].y * (double)omega_c, sx = (double)c->V.off[k].x * (double)omega_c;
      misr_T_exact(G.W, G.w, Z, R, g, sx, Ex);
      bool found = false;
      for (auto& cl : ycls)
        if (cl.first == sy) {
          for (size_t i = 0; i < Ex.size(); ++i) cl.second[i] += Ex[i];
          found = true;
          break;
        }
      if (!found) ycls.emplace_back(sy, Ex);
    }
    // classes with the same horizontal sum share one T_y sum
    std::vector<double> Tyt((size_t)G.H * NW, 0.0);
    const std::vector<double>& X0 = ycls[0].second;
    double vmax = 0.0;
    for (double v : X0) vmax = std::fmax(vmax, std::fabs(v));
    bool one = true;
    for (const auto& cl : ycls) {
      double dmax = 0.0;
      for (size_t i = 0; i < X0.size(); ++i) dmax = std::fmax(dmax, std::fabs(cl.second[i] - X0[i]));
      if (dmax > 1e-13 * vmax) one = false;
      misr_T_exact(G.H, G.h, Z, R, g, cl.first, Ey);
      for (size_t i = 0; i < Ey.size(); ++i) Tyt[i] += Ey[i];
    }
    if (one) {
      std::vector<float> ty(Tyt.size()), tx(X0.size());
      for (size_t i = 0; i < Tyt.size(); ++i) ty[i] = (float)(cA * Tyt[i]);
      for (size_t i = 0; i < X0.size(); ++i) tx[i] = (float)X0[i];
      const size_t need = (ty.size() + tx.size()) * sizeof(float);
      if (c->misr_tab_bytes < need || !c->d_misr_tab) {
        void* p = nullptr;
        cudaError_t e = dalloc(c, &p, need);
        if (e != cudaSuccess) return cuda_fail(c, e, "alloc");
        c->d_misr_tab = (float*)p;
        c->misr_tab_bytes = need;
      }
      CK(c, cudaMemcpyAsync(c->d_misr_tab, ty.data(), ty.size() * 4, cudaMemcpyHostToDevice, c->stream));
      CK(c, cudaMemcpyAsync(c->d_misr_tab + ty.size(), tx.data(), tx.size() * 4, cudaMemcpyHostToDevice, c->stream));
      CK(c, cudaStreamSynchronize(c->stream));   // host vectors are locals
      c->Tborder = c->Tfull;
      c->Tborder.ntl = 0;
      MisrArgs& a = c->misr_a;
      a = MisrArgs{};
      a.zs_y0 = 0; a.zs_y1 = G.H; a.zs_x0 = 0; a.zs_x1 = G.W;
      a.o_y0 = 0; a.o_y1 = G.H; a.o_x0 = 0; a.o_x1 = G.W;
      a.tyt = c->d_misr_tab;
      a.txt = c->d_misr_tab + ty.size();
      c->misr_border = false;
      CK(c, prepare_misr_kernels());
      c->misr = true;
      return LFSR_OK;
    }
    S.sep = 0;   // not one class: the phase stencil on Z_s and the border kernel
  }
  if (!interior_ok) return LFSR_OK;
  // border tiles of the whole-image tiling
  const TileGeom& T = c->Tfull;
  std::vector<char> brow(T.ntY, 0), bcol(T.ntX, 0);
  for (int l = 0; l < G.h; ++l)
    if (ay.lb[l]) brow[l / T.BL] = 1;
  for (int l = 0; l < G.w; ++l)
    if (ax.lb[l]) bcol[l / T.LX] = 1;
  auto middle = [](const std::vector<char>& b, int& a0, int& a1) {   // non-border range must be contiguous
    a0 = 0;
    while (a0 < (int)b.size() && b[a0]) ++a0;
    a1 = a0;
    while (a1 < (int)b.size() && !b[a1]) ++a1;
    for (int i = a1; i < (int)b.size(); ++i)
      if (!b[i]) return false;
    return true;
  };
  int ty0, ty1, tx0, tx1;
  if (!middle(brow, ty0, ty1) || !middle(bcol, tx0, tx1)) return LFSR_OK;
  std::vector<int> list;
  for (int ty = 0; ty < T.ntY; ++ty)
    for (int tx = 0; tx < T.ntX; ++tx)
      if (brow[ty] || bcol[tx]) list.push_back(ty * T.ntX + tx);
  if (c->tlist_cap < (int)list.size() || !c->d_tlist) {
    void* p = nullptr;
    cudaError_t e = dalloc(c, &p, std::max<size_t>(1, (size_t)T.ntY * T.ntX) * sizeof(int));
    if (e != cudaSuccess) return cuda_fail(c, e, "alloc");
    c->d_tlist = (int*)p;
    c->tlist_cap = T.ntY * T.ntX;
  }
  if (!list.empty())
    CK(c, cudaMemcpyAsync(c->d_tlist, list.data(), list.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));   // the host list is a local
  c->Tborder = T;
  c->Tborder.tlist = c->d_tlist;
  c->Tborder.ntl = (int)list.size();
  MisrArgs& a = c->misr_a;
  a = MisrArgs{};
  a.zs_y0 = ay.lo; a.zs_y1 = ay.hi; a.zs_x0 = ax.lo; a.zs_x1 = ax.hi;
  a.o_y0 = std::min(Z * T.BL * ty0, G.H); a.o_y1 = std::min(Z * T.BL * ty1, G.H);
  a.o_x0 = std::min(Z * T.LX * tx0, G.W); a.o_x1 = std::min(Z * T.LX * tx1, G.W);
  c->misr_border = true;
  CK(c, prepare_misr_kernels());
  c->misr = true;
  return LFSR_OK;
}

// q = M p on the MISR fast path: the exact tile kernel on the border tiles (flush masked to the
// band outside Z_s, no <p, Mp> share), then the stencil kernel (Z_s, p_k / pi_0 on the pixels no
// border tile owns, <p, q> over the image).  k >= 1: CG step k of part P; k = 0: plain operator
// from `in` into `out`.
static lfsr_status misr_normal(lfsr_ctx* c, Part& P, int k, const float* in, float* out, Control* ctl,
                               cudaStream_t st) {
  const Geom& G = c->G;
  TileIO n = base_io(P);
  n.ctl = ctl;
  n.out_hr = out;
  n.do_nltv = 1;
  n.zs_on = 1;
  n.zs_y0 = c->misr_a.zs_y0; n.zs_y1 = c->misr_a.zs_y1; n.zs_x0 = c->misr_a.zs_x0; n.zs_x1 = c->misr_a.zs_x1;
  n.no_pq = 1;
  MisrArgs a = c->misr_a;
  a.m = P.S.m;
  a.q = out;
  a.ctl = ctl;
  a.cg_k = k;
  a.do_nltv = 1;
  if (k >= 1) {
    n.in_hr = P.S.r;
    n.in_hr2 = P.S.p[(k - 1) & 1];
    n.p_out = P.S.p[k & 1];
    n.cg_k = k;
    a.r = P.S.r;
    a.p_prev = P.S.p[(k - 1) & 1];
    a.p_out = P.S.p[k & 1];
  } else {
    n.in_hr = in;
    a.p_in = in;
  }
  if (c->misr_border && c->Tborder.ntl > 0) CK(c, launch_tile(MODE_NORMAL, G, c->V, c->Tborder, n, st));
  CK(c, launch_misr_normal(G, *c->misr_S, a, st));
  return LFSR_OK;
}

// ---------------------------------------------------------------------------
// Assembled data normal operator (asm.cu).  The data part of M does not change
// during a solve (omega, the blur and the views are fixed), so its regular rows are summed once
// into a stencil per HR pixel and each CG step streams the stencil instead of re-running the
// warp / blur / decimate chain and its adjoint for every view.  Used on a single strip with the
// Gaussian blur and the exact adjoint (the MISR fast path takes constant disparities);
// LFSR_ASM=0 keeps the direct tile kernel.
// ---------------------------------------------------------------------------
static bool asm_wanted(const lfsr_ctx* c) {
  const Geom& G = c->G;
  return c->xmode == X_NONE && !G.paper && !G.psf2d && G.radius == 2 && G.s_d == 24 && G.scale >= 2 && G.scale <= 4 &&
         G.H < 65536 && G.W < 65536;   // (y << 16 | x) packing of the irregular lists
}

static lfsr_status asm_setup(lfsr_ctx* c, float om_max, bool read_count) {
  Geom& G = c->G;
  State& S = c->parts[0].S;
  c->asmop = false;
  if (!asm_wanted(c)) return LFSR_OK;
  const int NH = asm_plane_count(G.scale);   // stencil planes (full window)
  AsmBuf& B = c->asmb;
  const int psS = round_up(G.W + 3 * kAsmPad, 32);   // >= W + 24: shifted float4 reads stay in the padding
  const size_t plane = (size_t)(G.H + 2 * kAsmPad) * psS;
  const size_t nrows = (size_t)G.n_views * G.h * G.w;
  const size_t npos = (size_t)G.n_views * G.H * G.W;
  const int pmw = (G.W + 31) / 32;
  if (!B.st) {
    const size_t need = (size_t)NH * plane * 4 + nrows * (12 + 4 * (size_t)asm_row_floats(G.scale)) + npos * 12 +
                        (size_t)G.n_views * G.H * pmw * 4 + 512;
    size_t fr = 0, tot = 0;
    CK(c, cudaMemGetInfo(&fr, &tot));
    if (need > fr / 2) return LFSR_OK;   // no room: the direct tile kernel
    void* p = nullptr;
    cudaError_t e;
    if ((e = dalloc(c, &p, (size_t)NH * plane * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    B.st = (float*)p;
    if ((e = dalloc(c, &p, nrows * 8)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    B.list = (int2*)p;
    if ((e = dalloc(c, &p, nrows * asm_row_floats(G.scale) * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    B.rows = (float*)p;
    if ((e = dalloc(c, &p, nrows * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    B.tdense = (float*)p;
    if ((e = dalloc(c, &p, npos * 8)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    B.plist = (uint2*)p;
    if ((e = dalloc(c, &p, npos * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    B.udense = (float*)p;
    if ((e = dalloc(c, &p, (size_t)G.n_views * G.H * pmw * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    B.pmask = (unsigned*)p;
    if ((e = dalloc(c, &p, 64)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    B.count = (unsigned*)p;
    B.pmw = pmw;
    B.psS = psS;
    B.plane = plane;
  }
  B.omega = S.omega;
  B.om_max = om_max;
  CK(c, prepare_asm_kernels());
  const auto t0 = std::chrono::steady_clock::now();
  CK(c, launch_asm_build(G, c->V, B, om_max, c->stream));
  c->asm_nirr = -1;
  if (read_count) {
    unsigned n = 0;
    CK(c, cudaMemcpyAsync(&n, B.count, sizeof n, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    c->asm_nirr = n;
    c->asm_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  c->asmop = true;
  return LFSR_OK;
}

// q = M p through the assembled operator: t of the irregular rows, then the stencil kernel.
// k >= 1: CG step k of part P (p_k formed and written, pi_0, <p, q>); k = 0: plain operator.
static lfsr_status asm_normal(lfsr_ctx* c, Part& P, int k, const float* in, float* out, Control* ctl,
                              cudaStream_t st, int* launches) {
  AsmStep s{};
  s.r = P.S.r;
  s.p_prev = k >= 2 ? P.S.p[(k - 1) & 1] : nullptr;
  s.p_in = in;
  s.p_out = k >= 1 ? P.S.p[k & 1] : nullptr;
  s.m = P.S.m;
  s.q = out;
  s.ctl = ctl;
  s.cg_k = k;
  const bool irr = c->asm_nirr != 0;
  cudaEvent_t mid = (c->profile && k >= 1 && k < (int)c->asm_ev.size()) ? c->asm_ev[k] : nullptr;
  AsmFork fk{nullptr, nullptr, nullptr};
  const char* fe = getenv("LFSR_ASM_FORK");
  if (irr && !c->profile && !(fe && fe[0] == '0')) {   // (profiling keeps the kernels serial for the split)
    if (!c->side) {
      CK(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      CK(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      CK(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    fk = AsmFork{c->side, c->ev_fork, c->ev_join};
  }
  CK(c, launch_asm_step(c->G, c->V, c->asmb, s, irr, c->num_sms, st, mid, fk));
  if (launches) *launches += irr ? 4 : 1;   // k_asm_normal [+ k_asm_irr_u, _t, _scatter]
  return LFSR_OK;
}

// Path choice: the assembled operator runs when one CG operator pass through it is >= 5 % faster
// than through the tile kernel (both timed here on this light field), and -- for lfsr_solve_batch,
// whose fields each pay their own assembly -- when the per-field saving N K (t_tile - t_asm) also
// exceeds the assembly time.  The timings are cached per geometry (a batch decides before assembling
// once one field of the geometry was timed; the first set_observations of a geometry in the process
// times, later ones reuse the decision).  LFSR_ASM=1 / 0 forces either path.
struct AsmTiming {
  float t_tile = 0.f, t_asm = 0.f;   // ms per CG operator pass
  double setup_ms = 0.0;
};
static std::map<std::string, AsmTiming> g_asm_timing;

static bool asm_forced(bool* on) {
  const char* e = getenv("LFSR_ASM");
  if (!e || !e[0]) return false;
  *on = e[0] != '0';
  return true;
}

static bool asm_pays(const lfsr_ctx* c, const AsmTiming& t) {
  if (!(t.t_asm < 0.95f * t.t_tile)) return false;
  if (c->batch_iters > 0)
    return (double)(t.t_tile - t.t_asm) * c->batch_iters * c->G.K > t.setup_ms;
  return true;
}

// ms per pass of the CG operator (plain, k = 0) through the current path, 3 timed passes
static lfsr_status time_normal_pass(lfsr_ctx* c, bool asm_path, float* ms_out) {
  Part& P = c->parts[0];
  const Geom& G = c->G;
  cudaEvent_t e0, e1;
  CK(c, cudaEventCreate(&e0));
  CK(c, cudaEventCreate(&e1));
  auto pass = [&]() -> lfsr_status {
    if (asm_path) return asm_normal(c, P, 0, P.S.x, c->tmp_hr2, P.S.ctl, c->stream, nullptr);
    TileIO io = base_io(P);
    io.in_hr = P.S.x;
    io.out_hr = c->tmp_hr2;
    io.do_nltv = 1;
    CK(c, launch_tile(MODE_NORMAL, G, c->V, P.T, io, c->stream));
    return LFSR_OK;
  };
  lfsr_status st = pass();   // warm
  CK(c, cudaEventRecord(e0, c->stream));
  for (int r = 0; r < 3 && st == LFSR_OK; ++r) st = pass();
  CK(c, cudaEventRecord(e1, c->stream));
  CK(c, cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(c, cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_out = ms / 3.f;
  return st;
}

static lfsr_status choose_normal_path(lfsr_ctx* c, float om_max) {
  c->asmop = false;
  bool forced_on = false;
  const bool forced = asm_forced(&forced_on);
  if (forced && !forced_on) return LFSR_OK;
  if (!asm_wanted(c)) return LFSR_OK;
  const std::string key = tune_key(c);
  bool cached = false;
  if (!forced) {   // a timed geometry: decide before assembling (stable choice within the process)
    std::lock_guard<std::mutex> lk(g_tune_mu);
    auto it = g_asm_timing.find(key);
    if (it != g_asm_timing.end()) {
      if (!asm_pays(c, it->second)) return LFSR_OK;
      cached = true;
    }
  }
  lfsr_status st;
  {
    NvtxRange r_("normal operator assembly");
    if ((st = asm_setup(c, om_max, true)) != LFSR_OK) return st;
  }
  if (!c->asmop || forced || cached) return LFSR_OK;
  AsmTiming t;
  if ((st = time_normal_pass(c, false, &t.t_tile)) != LFSR_OK) return st;
  if ((st = time_normal_pass(c, true, &t.t_asm)) != LFSR_OK) return st;
  t.setup_ms = c->asm_ms;
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    g_asm_timing[key] = t;
  }
  if (getenv("LFSR_TUNE_VERBOSE"))
    fprintf(stderr, "lfsr normal path: tile %.1f us, assembled %.1f us, assembly %.2f ms, batch N %d\n",
            t.t_tile * 1000.f, t.t_asm * 1000.f, t.setup_ms, c->batch_iters);
  c->asmop = asm_pays(c, t);
  return LFSR_OK;
}

lfsr_status lfsr_set_observations(lfsr_ctx* c, const float* lr_views, const float* view_offsets,
                                  const float* disparity, lfsr_disp_mode disp_mode, const float* x0, lfsr_mem mem) {
  NvtxRange nvtx_("lfsr_set_observations");
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA/NCCL error");
  if (disp_mode != LFSR_DISP_SHARED && disp_mode != LFSR_DISP_PER_VIEW) FAIL(c, LFSR_ERR_INVALID_ARG, "unknown disp_mode");
  if (disp_mode == LFSR_DISP_PER_VIEW && (c->G.psf2d || c->G.paper))
    FAIL(c, LFSR_ERR_UNSUPPORTED, "per-view disparity maps with a user blur kernel or the paper-mode adjoint are not in this build");
  lfsr_status st;
  if ((st = check_ptr(c, lr_views, mem, "lr_views")) != LFSR_OK) return st;
  if ((st = check_ptr(c, view_offsets, mem, "view_offsets")) != LFSR_OK) return st;
  if ((st = check_ptr(c, disparity, mem, "disparity")) != LFSR_OK) return st;
  if (x0 && (st = check_ptr(c, x0, mem, "x0")) != LFSR_OK) return st;
  CK(c, cudaSetDevice(c->prm.device));
  const auto ts0 = std::chrono::steady_clock::now();

  // view offsets to the host (needed for halo sizing) and validation
  const int nv = c->prm.n_views;
  std::vector<float> off(2 * (size_t)nv);
  CK(c, cudaMemcpyAsync(off.data(), view_offsets, off.size() * 4,
                        mem == LFSR_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  for (float v : off)
    if (!std::isfinite(v)) FAIL(c, LFSR_ERR_INVALID_ARG, "view_offsets must be finite");

  Geom& G = c->G;
  const size_t hr = (size_t)G.H * G.ps, lr = (size_t)G.n_views * G.h * G.lps;
  const size_t ws = (size_t)G.s_d * hr;
  const int nparts = c->xmode == X_LOCAL ? c->prm.n_ranks : 1;
  G.per_view = disp_mode == LFSR_DISP_PER_VIEW ? 1 : 0;
  const size_t n_om = G.per_view ? (size_t)G.n_views : 1;   // disparity maps
  const size_t key[7] = {(size_t)G.n_views, (size_t)G.h, (size_t)G.w, (size_t)G.scale, (size_t)G.s_d,
                         (size_t)nparts, n_om};
  c->ready = false;
  free_graph(c);
  if (memcmp(key, c->alloc_key, sizeof key) != 0) {
    free_state(c);
    c->parts.assign(nparts, Part{});
    for (Part& P : c->parts)
      if ((st = alloc_part(c, P)) != LFSR_OK) return st;
    void* p = nullptr;
    cudaError_t e;
    if ((e = dalloc(c, &p, hr * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    c->tmp_hr2 = (float*)p;
    if ((e = dalloc(c, &p, 4 * sizeof(unsigned))) != cudaSuccess) return cuda_fail(c, e, "alloc");
    c->umax = (unsigned*)p;
    if (nparts > 1) {
      if ((e = dalloc(c, &p, sizeof(Control*) * nparts)) != cudaSuccess) return cuda_fail(c, e, "alloc");
      c->d_ctls = (Control**)p;
      std::vector<Control*> h(nparts);
      for (int i = 0; i < nparts; ++i) h[i] = c->parts[i].S.ctl;
      CK(c, cudaMemcpyAsync(c->d_ctls, h.data(), sizeof(Control*) * nparts, cudaMemcpyHostToDevice, c->stream));
    }
    memcpy(c->alloc_key, key, sizeof key);
  } else {  // same geometry: reset the state in place (Alg.1 lines 1-2: w = 0)
    for (Part& P : c->parts) {
      State& S = P.S;
      CK(c, cudaMemsetAsync(S.wA, 0, lr * 4, c->stream));
      CK(c, cudaMemsetAsync(S.wS[0], 0, ws * 4, c->stream));
      CK(c, cudaMemsetAsync(S.wS[1], 0, ws * 4, c->stream));
      CK(c, cudaMemsetAsync(S.density, 0, hr * 4, c->stream));
      CK(c, cudaMemsetAsync(S.r, 0, hr * 4, c->stream));
      CK(c, cudaMemsetAsync(S.q, 0, hr * 4, c->stream));
      CK(c, cudaMemsetAsync(S.p[0], 0, hr * 4, c->stream));
      CK(c, cudaMemsetAsync(S.p[1], 0, hr * 4, c->stream));
    }
  }
  c->h_iter = 0;
  c->solver = 0;
  unsigned* umax = c->umax;
  for (Part& P : c->parts) {
    Control h{};
    h.ring = P.ring;
    h.cap = kRingCap;
    CK(c, cudaMemcpyAsync(P.S.ctl, &h, sizeof(Control), cudaMemcpyHostToDevice, c->stream));
    CK(c, put2d(c, P.S.omega, G.ps, disparity, G.W, (size_t)G.H * n_om, mem));
  }
  // the observations (the large copy) go on the capture stream, so the omega-only setup
  // below (max|omega|, the splat density) overlaps the transfer
  for (cudaEvent_t& e : c->ev_in)
    if (!e) CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(c, cudaEventRecord(c->ev_in[0], c->stream));
  CK(c, cudaStreamWaitEvent(c->cap_stream, c->ev_in[0], 0));
  for (Part& P : c->parts) CK(c, put2d(c, P.S.y, G.lps, lr_views, G.w, (size_t)G.n_views * G.h, mem, c->cap_stream));
  CK(c, cudaEventRecord(c->ev_in[1], c->cap_stream));
  State& S0 = c->parts[0].S;

  // three maxima with one round trip: max|omega| (halo sizes S = ceil(max_k |dtheta_k|
  // max|omega|) per axis, in fp32 like the kernels), and the fixed-point bounds max|y| and
  // the splat density max_z sum_k (W_k^T 1)(z)
  for (int k = 0; k < nv; ++k) c->V.off[k] = make_float2(off[2 * k], off[2 * k + 1]);
  CK(c, cudaMemsetAsync(umax, 0, 4 * sizeof(unsigned), c->stream));
  CK(c, launch_absmax(S0.omega, hr * n_om, umax, c->stream));
  // constant disparity (global shifts: the MISR fast path, misr_setup) -- shared map only
  if (!G.per_view) CK(c, launch_omega_const(G, S0.omega, umax + 3, c->stream));
  else CK(c, cudaMemsetAsync(umax + 3, 0xff, sizeof(unsigned), c->stream));
  CK(c, launch_density(G, c->V, S0.omega, S0.density, c->stream));
  CK(c, launch_absmax(S0.density, hr, umax + 1, c->stream));
  CK(c, cudaStreamWaitEvent(c->stream, c->ev_in[1], 0));   // y is in place
  CK(c, launch_absmax(S0.y, lr, umax + 2, c->stream));
  unsigned ubits[4] = {0, 0, 0, 0};
  float omega00 = 0.f;
  CK(c, cudaMemcpyAsync(ubits, umax, sizeof ubits, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(&omega00, S0.omega, sizeof omega00, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  float om_max;
  memcpy(&om_max, &ubits[0], 4);
  float mx_rho = 0.f, mx_tau = 0.f;
  for (int k = 0; k < nv; ++k) {
    mx_rho = std::fmax(mx_rho, std::fabs(off[2 * k]));
    mx_tau = std::fmax(mx_tau, std::fabs(off[2 * k + 1]));
  }
  if ((st = set_shift_halo(c, om_max, mx_rho, mx_tau)) != LFSR_OK) return st;
  memcpy(&G.dmax, &ubits[1], 4);
  memcpy(&G.ymax, &ubits[2], 4);
  if (!std::isfinite(G.ymax)) G.ymax = 0.f;  // non-finite observations surface as DIVERGED

  // tile height and the strip plan / tile geometry of every part
  bool tune = false;
  initial_tiles(c, &tune);
  if ((st = setup_tiles(c)) != LFSR_OK) return st;

  // a1 (every strip, whole image): x0 (bicubic unless given), static w_o, m from x0, density
  for (Part& P : c->parts) {
    State& S = P.S;
    if (x0) {
      CK(c, put2d(c, S.x, G.ps, x0, G.W, (size_t)G.H, mem));
    } else {
      CK(c, launch_bicubic(G, S.y, S.x, c->stream));
    }
    const float* om_ref = S.omega + (G.per_view ? (size_t)G.ref_view * hr : 0);   // omega_0 (A34)
    CK(c, launch_setup_wo(G, c->V, S.y, om_ref, S.wo, c->stream));
    CK(c, launch_weights(G, S.x, S.wo, S.m, c->stream));
  }
  if (tune) {
    NvtxRange r_("tile tuning");
    if ((st = tune_tile_bl(c)) != LFSR_OK) return st;
  }
  c->misr = false;
  if (ubits[3] == 0) {
    NvtxRange r_("MISR stencil assembly");
    if ((st = misr_setup(c, omega00)) != LFSR_OK) return st;
  }
  c->asmop = false;
  if (!c->misr && (st = choose_normal_path(c, om_max)) != LFSR_OK) return st;
  const auto tg0 = std::chrono::steady_clock::now();
  lfsr_status gs = build_graphs(c);
  if (gs != LFSR_OK) return gs;
  const auto tg1 = std::chrono::steady_clock::now();
  CK(c, cudaStreamSynchronize(c->stream));
  if (getenv("LFSR_TRACE_SETUP"))
    fprintf(stderr, "lfsr set_observations: graph build %.3f ms, total %.3f ms\n",
            std::chrono::duration<double, std::milli>(tg1 - tg0).count(),
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts0).count());
  c->ready = true;
  return LFSR_OK;
}

static TileIO base_io(const Part& P) {
  TileIO io{};
  io.rho_out = P.S.rho;   // paper mode only (A37)
  io.omega = P.S.omega;
  io.ctl = P.S.ctl;
  io.m = P.S.m;
  return io;
}

// ---------------------------------------------------------------------------
// Halo exchange between strips.  Buffers are full size, so a
// row has the same address offset in every strip.
//   fill(buf):  rows [Y0 - top, Y0) <- previous strip, [Y1, Y1 + bot) <- next
//   fold(buf):  rows [Y0 - top, Y0) -> added into the previous strip (its own
//               rows), [Y1, Y1 + bot) -> into the next; then zeroed here.
// planes/plane_stride: the same row ranges in each of `planes` planes (w_S).
// ---------------------------------------------------------------------------
struct Rows {
  int a, b;  // [a, b)
};

static lfsr_status xfill(lfsr_ctx* c, cudaStream_t st, float* const* bufs, int top, int bot, int planes = 1,
                         size_t plane_stride = 0, float* const* bufs2 = nullptr) {
  const Geom& G = c->G;
  const size_t rowf = (size_t)G.ps;
  if (bufs2 && c->xmode == X_LOCAL) {   // two single-plane buffer sets: one after the other
    lfsr_status s1 = xfill(c, st, bufs, top, bot, planes, plane_stride);
    return s1 != LFSR_OK ? s1 : xfill(c, st, bufs2, top, bot, planes, plane_stride);
  }
  if (c->xmode == X_LOCAL) {
    const int n = (int)c->parts.size();
    for (int i = 0; i < n; ++i) {
      const lfsr_strip& s = c->parts[i].plan;
      Rows up{std::max(s.hr_row0 - top, 0), s.hr_row0}, dn{s.hr_row1, std::min(s.hr_row1 + bot, G.H)};
      if (i > 0 && up.b > up.a)
        CK(c, cudaMemcpy2DAsync(bufs[i] + up.a * rowf, plane_stride * 4, bufs[i - 1] + up.a * rowf, plane_stride * 4,
                                (up.b - up.a) * rowf * 4, planes, cudaMemcpyDeviceToDevice, st));
      if (i + 1 < n && dn.b > dn.a)
        CK(c, cudaMemcpy2DAsync(bufs[i] + dn.a * rowf, plane_stride * 4, bufs[i + 1] + dn.a * rowf, plane_stride * 4,
                                (dn.b - dn.a) * rowf * 4, planes, cudaMemcpyDeviceToDevice, st));
    }
    return LFSR_OK;
  }
  if (c->xmode == X_NCCL) {
    const lfsr_strip& s = c->parts[0].plan;
    const int r = s.rank, n = c->prm.n_ranks;
    NK(c, nccl_group_start());   // one group (one NCCL launch) for both buffer sets
    for (int pl = 0; pl < planes * (bufs2 ? 2 : 1); ++pl) {
      float* bp = pl < planes ? bufs[0] + pl * plane_stride : bufs2[0] + (pl - planes) * plane_stride;
      if (r > 0) {  // my first `bot` rows are the previous strip's lower halo; receive my upper halo
        const int sa = s.hr_row0, sb = std::min(s.hr_row0 + bot, s.hr_row1);
        NK(c, nccl_send_f32(bp + sa * rowf, (sb - sa) * rowf, r - 1, c->comm, st));
        const int ra = std::max(s.hr_row0 - top, 0);
        NK(c, nccl_recv_f32(bp + ra * rowf, (s.hr_row0 - ra) * rowf, r - 1, c->comm, st));
      }
      if (r + 1 < n) {
        const int sa = std::max(s.hr_row1 - top, s.hr_row0), sb = s.hr_row1;
        NK(c, nccl_send_f32(bp + sa * rowf, (sb - sa) * rowf, r + 1, c->comm, st));
        const int rb = std::min(s.hr_row1 + bot, G.H);
        NK(c, nccl_recv_f32(bp + s.hr_row1 * rowf, (rb - s.hr_row1) * rowf, r + 1, c->comm, st));
      }
    }
    NK(c, nccl_group_end());
  }
  return LFSR_OK;
}

static lfsr_status xfold(lfsr_ctx* c, cudaStream_t st, float* const* bufs, int top, int bot) {
  const Geom& G = c->G;
  const size_t rowf = (size_t)G.ps;
  if (c->xmode == X_LOCAL) {
    const int n = (int)c->parts.size();
    for (int i = 0; i < n; ++i) {
      const lfsr_strip& s = c->parts[i].plan;
      if (i > 0) {
        const int a = std::max(s.hr_row0 - top, 0);
        CK(c, launch_fold_rows(bufs[i - 1] + a * rowf, bufs[i] + a * rowf, (s.hr_row0 - a) * rowf, 1, st));
      }
      if (i + 1 < n) {
        const int b = std::min(s.hr_row1 + bot, G.H);
        CK(c, launch_fold_rows(bufs[i + 1] + s.hr_row1 * rowf, bufs[i] + s.hr_row1 * rowf, (b - s.hr_row1) * rowf, 1,
                               st));
      }
    }
    return LFSR_OK;
  }
  if (c->xmode == X_NCCL) {
    Part& P = c->parts[0];
    const lfsr_strip& s = P.plan;
    const int r = s.rank, n = c->prm.n_ranks;
    float* b = bufs[0];
    const int ua = std::max(s.hr_row0 - top, 0);          // my upper ring rows [ua, Y0)
    const int db = std::min(s.hr_row1 + bot, G.H);        // my lower ring rows [Y1, db)
    const int pa = s.hr_row0, pb = std::min(s.hr_row0 + bot, s.hr_row1);  // rows the previous strip folds into mine
    const int na = std::max(s.hr_row1 - top, s.hr_row0), nb = s.hr_row1;  // rows the next strip folds into mine
    NK(c, nccl_group_start());
    if (r > 0) {
      NK(c, nccl_send_f32(b + ua * rowf, (s.hr_row0 - ua) * rowf, r - 1, c->comm, st));
      NK(c, nccl_recv_f32(P.stage[0], (pb - pa) * rowf, r - 1, c->comm, st));
    }
    if (r + 1 < n) {
      NK(c, nccl_send_f32(b + s.hr_row1 * rowf, (db - s.hr_row1) * rowf, r + 1, c->comm, st));
      NK(c, nccl_recv_f32(P.stage[1], (nb - na) * rowf, r + 1, c->comm, st));
    }
    NK(c, nccl_group_end());
    if (r > 0) {
      CK(c, launch_fold_rows(b + pa * rowf, P.stage[0], (pb - pa) * rowf, 0, st));
      CK(c, cudaMemsetAsync(b + ua * rowf, 0, (s.hr_row0 - ua) * rowf * 4, st));
    }
    if (r + 1 < n) {
      CK(c, launch_fold_rows(b + na * rowf, P.stage[1], (nb - na) * rowf, 0, st));
      CK(c, cudaMemsetAsync(b + s.hr_row1 * rowf, 0, (db - s.hr_row1) * rowf * 4, st));
    }
  }
  return LFSR_OK;
}

static lfsr_status xallreduce(lfsr_ctx* c, cudaStream_t st, int slot0, int count) {
  if (c->xmode == X_LOCAL) {
    CK(c, launch_allreduce_local(c->d_ctls, (int)c->parts.size(), slot0, count, st));
  } else if (c->xmode == X_NCCL) {
    NK(c, nccl_allreduce_sum_f64(c->parts[0].S.ctl->cur + slot0, count, c->comm, st));
  }
  return LFSR_OK;
}

// One ADMM iteration = k_wz + K x (k_normal, k_cg_update), captured once (per
// parity of the iteration count: the w_S buffers alternate).  With several
// strips the exchanges of DESIGN.md §10 sit between the kernels.  In profiling
// mode (single strip) an external event-record node brackets every kernel.
static lfsr_status enqueue_iteration(lfsr_ctx* c, cudaStream_t st, int parity) {
  const Geom& G = c->G;
  const int np = (int)c->parts.size();
  const bool multi = c->xmode != X_NONE;
  int ev = 0, launches = 0;
  auto mark = [&]() -> cudaError_t {
    if (!c->profile || multi) return cudaSuccess;
    return cudaEventRecordWithFlags(c->prof_ev[ev++], st, cudaEventRecordExternal);
  };
  std::vector<float*> xs(np), rs(np), qs(np), ms(np), wsw(np), pk(np);
  for (int i = 0; i < np; ++i) {
    xs[i] = c->parts[i].S.x;
    rs[i] = c->parts[i].S.r;
    qs[i] = c->parts[i].S.q;
    ms[i] = c->parts[i].S.m;
    wsw[i] = c->parts[i].S.wS[parity ^ 1];   // written by this iteration's wz-step
  }
  const int top = multi ? c->parts[0].plan.halo_top + c->parts[0].plan.halo_bottom : 0;  // see below
  (void)top;
  // halo widths are the same for every strip boundary
  int ht = 0, hb = 0;
  for (const Part& P : c->parts) {
    ht = std::max(ht, P.plan.halo_top);
    hb = std::max(hb, P.plan.halo_bottom);
  }
  if (c->xmode == X_NCCL) {  // a single strip sees only its own halos; both directions have the plan widths
    std::vector<lfsr_strip> plan;
    std::string why;
    make_plan(G, c->prm.n_ranks, G.SY, plan, why);
    for (const lfsr_strip& s : plan) {
      ht = std::max(ht, s.halo_top);
      hb = std::max(hb, s.halo_bottom);
    }
  }
  const int r = G.radius;
  // NLTV rows of the wz-step in their own streaming kernel (nltv.cu) for large images (measured: C5
  // 2048^2 -11 % wz-step time, M2 2048^2 even, C2 / C3 512^2 +5 % -- there the tile kernel's phase
  // 3 hides the stream behind its view passes); LFSR_NLTV_SPLIT=0 / 1 forces either
  const char* ns_env = getenv("LFSR_NLTV_SPLIT");
  const bool nltv_big = (size_t)G.H * G.W >= ((size_t)1 << 21);
  const bool nltv_split = G.radius == 2 && (ns_env && ns_env[0] ? ns_env[0] == '1' : nltv_big);
  lfsr_status s_;
#define XC(expr)                                 \
  do {                                           \
    if ((s_ = (expr)) != LFSR_OK) return s_;     \
  } while (0)

  // strips: the tiles whose input tile lies in the own rows run on the side stream while the halo is
  // exchanged (fork / join inside the captured graph); the boundary tiles after the exchange
  const char* ov_env = getenv("LFSR_STRIP_OVERLAP");
  const bool overlap = multi && c->side && !(ov_env && ov_env[0] == '0');
  auto split_launch = [&](auto&& fill, auto&& launch_part) -> lfsr_status {
    if (!overlap) {
      lfsr_status q_ = fill();
      if (q_ != LFSR_OK) return q_;
      for (Part& P : c->parts) {
        if ((q_ = launch_part(P, P.T, st)) != LFSR_OK) return q_;
      }
      return LFSR_OK;
    }
    CK(c, cudaEventRecord(c->ev_fork, st));
    CK(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    lfsr_status q_;
    for (Part& P : c->parts)
      if (P.Tin.ntl > 0 && (q_ = launch_part(P, P.Tin, c->side)) != LFSR_OK) return q_;
    CK(c, cudaEventRecord(c->ev_join, c->side));
    if ((q_ = fill()) != LFSR_OK) return q_;
    for (Part& P : c->parts)
      if (P.Tbd.ntl > 0 && (q_ = launch_part(P, P.Tbd, st)) != LFSR_OK) return q_;
    CK(c, cudaStreamWaitEvent(st, c->ev_join, 0));
    return LFSR_OK;
  };
  CK(c, mark());
  XC(split_launch([&]() { return multi ? xfill(c, st, xs.data(), ht, hb) : LFSR_OK; },   // x halo
                  [&](Part& P, const TileGeom& T, cudaStream_t s2) -> lfsr_status {
                    TileIO io = base_io(P);
                    io.in_hr = P.S.x;
                    io.y = P.S.y;
                    io.wA = P.S.wA;
                    io.wS0 = P.S.wS[0];
                    io.wS1 = P.S.wS[1];
                    io.wo = P.S.wo;
                    io.out_hr = P.S.r;
                    io.reweight = c->prm.reweight_every_iter;
                    io.wz_no_nltv = nltv_split ? 1 : 0;
                    CK(c, launch_tile(MODE_WZ, G, c->V, T, io, s2));
                    ++launches;
                    return LFSR_OK;
                  }));
  for (Part& P : c->parts) {
    if (G.paper) {   // v's data part through the paper's backward warp (A37): r = -v
      CK(c, launch_paper_gather(G, c->V, P.S.rho, P.S.omega, nullptr, P.S.r, -1.f, P.S.ctl, -1, 0, 0, G.H, st));
      ++launches;
    }
  }
  if (nltv_split) {   // the NLTV rows of the wz-step as a streaming kernel (nltv.cu), own rows
    if (multi) XC(xfill(c, st, ms.data(), r, r));                         // m of the neighbours' rows
    for (Part& P : c->parts) {
      CK(c, launch_wz_nltv(G, P.S.x, P.S.m, P.S.wS[0], P.S.wS[1], P.S.r, P.S.ctl, P.plan.hr_row0, P.plan.hr_row1, st));
      ++launches;
    }
  }
  CK(c, mark());
  if (multi) {
    XC(xfold(c, st, rs.data(), ht, hb));                                  // r = -v rings
    XC(xfill(c, st, ms.data(), r, r));                                    // m for the NLTV normal term
    XC(xfill(c, st, wsw.data(), r, r, G.s_d, (size_t)G.H * G.ps));        // new w_S for the next wz-step
    XC(xallreduce(c, st, S_L1, 4));                                       // J terms, |dw|^2
  }
  // strips: CG in the Chronopoulos-Gear form -- one operator pass on r and ONE all-reduce of
  // (gamma, delta) per step, one halo fill (r only); LFSR_STRIP_CG=standard keeps Alg.2's two
  const char* cg_env = getenv("LFSR_STRIP_CG");
  const bool cgcg = multi && !G.paper && !(cg_env && cg_env[0] == 's');
  for (int j = 0; cgcg && j < G.K; ++j) {
    XC(split_launch([&]() { return xfill(c, st, rs.data(), ht, hb); },   // r_j halo
                    [&](Part& P, const TileGeom& T, cudaStream_t s2) -> lfsr_status {
                      TileIO n = base_io(P);
                      n.in_hr = P.S.r;
                      n.out_hr = P.S.q;   // w_j = M r_j
                      n.cg_k = 1;
                      n.cgcg_slot = S_CG + 2 * j;
                      n.cgcg_step = j;
                      n.do_nltv = 1;
                      CK(c, launch_tile(MODE_NORMAL, G, c->V, T, n, s2));
                      ++launches;
                      return LFSR_OK;
                    }));
    XC(xfold(c, st, qs.data(), ht, hb));
    XC(xallreduce(c, st, S_CG + 2 * j, 2));   // (gamma_j, delta_j)
    for (Part& P : c->parts) {
      const lfsr_strip& sp = P.plan;
      CK(c, launch_cgcg_update(G, P.S.x, P.S.r, P.S.p[0], P.S.p[1], P.S.q, P.S.ctl, j, sp.hr_row0,
                               sp.hr_row1 - sp.hr_row0, c->num_sms, st));
      ++launches;
    }
    if (j == G.K - 1) {
      XC(xallreduce(c, st, S_PI + G.K, 1));   // pi_K for the record
      XC(xallreduce(c, st, S_NF, 1));
      for (Part& P : c->parts) {   // r's halo rows start the next wz-step at zero (see below)
        const lfsr_strip& sp = P.plan;
        const int a = std::max(sp.hr_row0 - ht, 0), b = std::min(sp.hr_row1 + hb, G.H);
        if (sp.hr_row0 > a) CK(c, cudaMemsetAsync(P.S.r + (size_t)a * G.ps, 0, (size_t)(sp.hr_row0 - a) * G.ps * 4, st));
        if (b > sp.hr_row1)
          CK(c, cudaMemsetAsync(P.S.r + (size_t)sp.hr_row1 * G.ps, 0, (size_t)(b - sp.hr_row1) * G.ps * 4, st));
      }
    }
  }
  for (int k = 1; !cgcg && k <= G.K; ++k) {
    if (c->misr) {   // constant shifts: border tiles + the precomputed stencil (misr.cu)
      Part& P = c->parts[0];
      XC(misr_normal(c, P, k, nullptr, P.S.q, P.S.ctl, st));
      launches += (c->misr_border && c->Tborder.ntl > 0) ? 2 : 1;
    } else if (c->asmop) {   // the assembled operator (asm.cu)
      Part& P = c->parts[0];
      XC(asm_normal(c, P, k, nullptr, P.S.q, P.S.ctl, st, &launches));
    }
    if (!c->misr && !c->asmop) {
      for (int i = 0; i < np; ++i) pk[i] = c->parts[i].S.p[(k - 1) & 1];
      // the halos of r (and of p_{k-1} from k = 2) for this step's operator, overlapped with the
      // interior tiles (k = 1: r_0 = -v after the wz-step's fold)
      XC(split_launch([&]() -> lfsr_status {
                        if (!multi) return LFSR_OK;
                        return k == 1 ? xfill(c, st, rs.data(), ht, hb)
                                      : xfill(c, st, rs.data(), ht, hb, 1, 0, pk.data());
                      },
                      [&](Part& P, const TileGeom& T, cudaStream_t s2) -> lfsr_status {
                        TileIO n = base_io(P);
                        n.in_hr = P.S.r;
                        n.in_hr2 = P.S.p[(k - 1) & 1];
                        n.p_out = P.S.p[k & 1];
                        n.out_hr = P.S.q;
                        n.cg_k = k;
                        n.do_nltv = 1;
                        CK(c, launch_tile(MODE_NORMAL, G, c->V, T, n, s2));
                        ++launches;
                        return LFSR_OK;
                      }));
      if (G.paper) {   // q's data part and its share of <p, q> (A37; single strip)
        Part& P = c->parts[0];
        CK(c, launch_paper_gather(G, c->V, P.S.rho, P.S.omega, P.S.p[k & 1], P.S.q, 1.f, P.S.ctl, S_PQ + k, k, 0,
                                  G.H, st));
        ++launches;
      }
    }
    CK(c, mark());
    if (multi) {
      XC(xfold(c, st, qs.data(), ht, hb));
      XC(xallreduce(c, st, S_PQ + k, 1));
      if (k == 1) XC(xallreduce(c, st, S_PI, 1));
    }
    for (Part& P : c->parts) {
      const lfsr_strip& s = P.plan;
      CK(c, launch_cg_update(G, P.S.x, P.S.r, P.S.p[k & 1], P.S.q, P.S.ctl, k, s.hr_row0, s.hr_row1 - s.hr_row0,
                             multi ? 0 : 1, c->num_sms, st));
      ++launches;
    }
    CK(c, mark());
    if (multi) {
      XC(xallreduce(c, st, S_PI + k, 1));
      if (k == G.K) {
        XC(xallreduce(c, st, S_NF, 1));
        // the r halo rows hold filled neighbour values; the next wz-step accumulates
        // its ring into them, so they must start at zero like the own rows
        for (Part& P : c->parts) {
          const lfsr_strip& s = P.plan;
          const int a = std::max(s.hr_row0 - ht, 0), b = std::min(s.hr_row1 + hb, G.H);
          if (s.hr_row0 > a) CK(c, cudaMemsetAsync(P.S.r + (size_t)a * G.ps, 0, (size_t)(s.hr_row0 - a) * G.ps * 4, st));
          if (b > s.hr_row1)
            CK(c, cudaMemsetAsync(P.S.r + (size_t)s.hr_row1 * G.ps, 0, (size_t)(b - s.hr_row1) * G.ps * 4, st));
        }
      }   // (k < K: the r and p halos are exchanged at the start of step k + 1, next to its interior tiles)
    }
  }
  if (multi) {
    for (Part& P : c->parts) {
      CK(c, launch_close(G, P.S.ctl, st));
      ++launches;
    }
  }
#undef XC
  c->launches_per_iter = launches;
  return LFSR_OK;
}

static lfsr_status build_graphs(lfsr_ctx* c) {
  NvtxRange r_("ADMM iteration graph capture");
  free_graph(c);
  if (c->profile) {
    size_t need = 2 + 2 * (size_t)c->G.K;
    while (c->prof_ev.size() < need) {
      cudaEvent_t e;
      CK(c, cudaEventCreate(&e));
      c->prof_ev.push_back(e);
    }
    while (c->asm_ev.size() < (size_t)c->G.K + 1) {
      cudaEvent_t e;
      CK(c, cudaEventCreate(&e));
      c->asm_ev.push_back(e);
    }
  }
  const int ngraphs = c->xmode == X_NONE ? 1 : 2;  // the strip exchanges name the w_S buffer of each parity
  for (int g = 0; g < ngraphs; ++g) {
    CK(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    lfsr_status st = enqueue_iteration(c, c->cap_stream, g);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->cap_stream, &graph);
    if (st != LFSR_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&c->graph[g], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate");
  }
  return LFSR_OK;
}

static lfsr_status check_run(lfsr_ctx* c) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA/NCCL error");
  if (!c->ready) FAIL(c, LFSR_ERR_STATE, "ADMM call before lfsr_set_observations");
  return LFSR_OK;
}

lfsr_status lfsr_admm_enqueue(lfsr_ctx* c, int32_t n_iters) {
  NvtxRange nvtx_("lfsr_admm_enqueue");
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (n_iters < 0) FAIL(c, LFSR_ERR_INVALID_ARG, "n_iters must be >= 0");
  if (c->solver == 2) FAIL(c, LFSR_ERR_STATE, "gd iterations ran since lfsr_set_observations (one solver per solve)");
  c->solver = 1;
  CK(c, cudaSetDevice(c->prm.device));
  for (int n = 0; n < n_iters; ++n) {
    cudaGraphExec_t g = c->graph[c->graph[1] ? (c->h_iter + n) & 1 : 0];
    CK(c, cudaGraphLaunch(g, c->stream));
  }
  c->h_iter += n_iters;
  return LFSR_OK;
}

// Blocking read of the device records of iterations [first, first + n) (1-based).
static lfsr_status read_records(lfsr_ctx* c, int first_iter, int n_iters, std::vector<double>& rec) {
  CK(c, cudaSetDevice(c->prm.device));
  const double* ring = c->parts[0].ring;
  rec.assign((size_t)n_iters * T_COUNT, 0.0);
  int done = 0;
  while (done < n_iters) {  // at most two contiguous pieces of the ring
    int slot = (first_iter - 1 + done) % kRingCap;
    int cnt = std::min(n_iters - done, kRingCap - slot);
    CK(c, cudaMemcpyAsync(rec.data() + (size_t)done * T_COUNT, ring + (size_t)slot * T_COUNT,
                          (size_t)cnt * T_COUNT * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    done += cnt;
  }
  CK(c, cudaStreamSynchronize(c->stream));
  return LFSR_OK;
}

lfsr_status lfsr_admm_stats(lfsr_ctx* c, int32_t first_iter, int32_t n_iters, lfsr_iter_stats* stats) {
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (n_iters < 0 || first_iter < 1 || first_iter + n_iters - 1 > c->h_iter || first_iter <= c->h_iter - kRingCap)
    FAIL(c, LFSR_ERR_INVALID_ARG, "requested iterations are not in the stats window");
  if (n_iters == 0) return LFSR_OK;
  std::vector<double> rec;
  if ((st = read_records(c, first_iter, n_iters, rec)) != LFSR_OK) return st;
  bool bad = false;
  for (int n = 0; n < n_iters; ++n) {
    const double* r = rec.data() + (size_t)n * T_COUNT;
    if (r[T_NF] != 0.0) bad = true;
    if (stats) {
      lfsr_iter_stats& s = stats[n];
      s.iter = (int32_t)r[T_ITER];
      s.cg_iters = (int32_t)r[T_CGIT];
      s.breakdown = (int32_t)r[T_BREAK];
      s.nonfinite = (int32_t)r[T_NF];
      s.J = r[T_J];
      s.data_l1 = r[T_L1];
      s.data_l2 = r[T_L2];
      s.reg_l1 = r[T_REG];
      s.primal_res = r[T_RES];
      s.cg_pi0 = r[T_PI0];
      s.cg_pi_last = r[T_PILAST];
    }
  }
  if (bad) FAIL(c, LFSR_ERR_DIVERGED, "non-finite x or cost during the ADMM iterations");
  return LFSR_OK;
}

lfsr_status lfsr_admm_run(lfsr_ctx* c, int32_t n_iters, lfsr_iter_stats* stats) {
  NvtxRange nvtx_("lfsr_admm_run");
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (n_iters < 0) FAIL(c, LFSR_ERR_INVALID_ARG, "n_iters must be >= 0");
  if (n_iters == 0) return LFSR_OK;
  const int n_read = std::min(n_iters, kRingCap);
  if (stats && n_read < n_iters) FAIL(c, LFSR_ERR_INVALID_ARG, "stats requested for more than 4096 iterations");
  const int first = c->h_iter + 1;
  if ((st = lfsr_admm_enqueue(c, n_iters)) != LFSR_OK) return st;
  return lfsr_admm_stats(c, first + (n_iters - n_read), n_read, stats);
}

// ---------------------------------------------------------------------------
// gd / gd-ls (readings A30-A33).  One iteration is
// one graph: zero g -> k_tile<GRAD> (m from x, cost terms, g) [-> |g|^2 -> L
// trial launches of k_tile<J>, each a no-op once an earlier trial met Armijo]
// -> k_gd_update (step choice, x -= eta g, record).
// ---------------------------------------------------------------------------
static lfsr_status enqueue_gd(lfsr_ctx* c, cudaStream_t st, const GdCfg& cfg) {
  const Geom& G = c->G;
  Part& P = c->parts[0];
  int launches = 0;
  CK(c, cudaMemsetAsync(c->gd_g, 0, (size_t)G.H * G.ps * 4, st));
  TileIO io = base_io(P);
  io.in_hr = P.S.x;
  io.y = P.S.y;
  io.wo = P.S.wo;
  io.out_hr = c->gd_g;
  io.reweight = c->prm.reweight_every_iter;
  CK(c, launch_tile(MODE_GRAD, G, c->V, P.T, io, st));
  ++launches;
  if (G.paper) {
    CK(c, launch_paper_gather(G, c->V, P.S.rho, P.S.omega, nullptr, c->gd_g, 1.f, P.S.ctl, -1, 0, 0, G.H, st));
    ++launches;
  }
  if (cfg.ls) {
    CK(c, launch_gd_gnorm(G, c->gd_g, P.S.ctl, c->num_sms, st));
    ++launches;
    for (int t = 0; t < cfg.L; ++t) {
      TileIO j = base_io(P);
      j.in_hr = P.S.x;
      j.in_hr2 = c->gd_g;
      j.y = P.S.y;
      j.ls_t = t;
      j.eta0 = cfg.eta0;
      j.armijo_c = cfg.armijo_c;
      CK(c, launch_tile(MODE_J, G, c->V, P.T, j, st));
      ++launches;
    }
  }
  CK(c, launch_gd_update(G, P.S.x, c->gd_g, P.S.ctl, cfg, c->num_sms, st));
  ++launches;
  c->gd_launches = launches;
  return LFSR_OK;
}

lfsr_status lfsr_gd_run(lfsr_ctx* c, const lfsr_gd_params* gp, int32_t n_iters, lfsr_gd_stats* stats) {
  NvtxRange nvtx_("lfsr_gd_run");
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (!gp) FAIL(c, LFSR_ERR_INVALID_ARG, "gd params must not be NULL");
  if (n_iters < 0) FAIL(c, LFSR_ERR_INVALID_ARG, "n_iters must be >= 0");
  if (!(gp->step > 0.f) || !std::isfinite(gp->step)) FAIL(c, LFSR_ERR_INVALID_ARG, "step must be finite and > 0");
  if (gp->line_search && (gp->max_trials < 1 || gp->max_trials > kMaxLs))
    FAIL(c, LFSR_ERR_INVALID_ARG, "max_trials must be in [1, 32]");
  if (!(gp->armijo_c >= 0.f) || !std::isfinite(gp->armijo_c)) FAIL(c, LFSR_ERR_INVALID_ARG, "armijo_c must be >= 0");
  if (c->xmode != X_NONE) FAIL(c, LFSR_ERR_UNSUPPORTED, "gd runs on a single strip");
  if (n_iters > kRingCap && stats) FAIL(c, LFSR_ERR_INVALID_ARG, "stats requested for more than 4096 iterations");
  if (c->solver == 1) FAIL(c, LFSR_ERR_STATE, "ADMM iterations ran since lfsr_set_observations (one solver per solve)");
  c->solver = 2;
  if (n_iters == 0) return LFSR_OK;
  CK(c, cudaSetDevice(c->prm.device));
  const Geom& G = c->G;
  if (!c->gd_g) {
    void* p = nullptr;
    cudaError_t e = dalloc(c, &p, (size_t)G.H * G.ps * 4);
    if (e != cudaSuccess) {
      cudaGetLastError();
      FAIL(c, LFSR_ERR_OOM, "device allocation failed");
    }
    c->gd_g = (float*)p;
  }
  GdCfg cfg{gp->step, gp->armijo_c, gp->line_search ? 1 : 0, gp->line_search ? gp->max_trials : 0};
  if (!c->gd_graph || memcmp(&cfg, &c->gd_cfg, sizeof cfg) != 0) {
    if (c->gd_graph) {
      CK(c, cudaStreamSynchronize(c->stream));
      cudaGraphExecDestroy(c->gd_graph);
      c->gd_graph = nullptr;
    }
    CK(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    lfsr_status es = enqueue_gd(c, c->cap_stream, cfg);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->cap_stream, &graph);
    if (es != LFSR_OK) {
      if (graph) cudaGraphDestroy(graph);
      return es;
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&c->gd_graph, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate");
    c->gd_cfg = cfg;
  }
  const int first = c->h_iter + 1;
  for (int n = 0; n < n_iters; ++n) CK(c, cudaGraphLaunch(c->gd_graph, c->stream));
  c->h_iter += n_iters;
  const int n_read = std::min(n_iters, kRingCap);
  std::vector<double> rec;
  if ((st = read_records(c, first + (n_iters - n_read), n_read, rec)) != LFSR_OK) return st;
  bool bad = false;
  for (int n = 0; n < n_read; ++n) {
    const double* r = rec.data() + (size_t)n * T_COUNT;
    if (r[T_NF] != 0.0) bad = true;
    if (stats) {
      lfsr_gd_stats& s = stats[n];
      s.iter = (int32_t)r[T_ITER];
      s.ls_evals = (int32_t)r[T_CGIT];
      s.ls_failed = (int32_t)r[T_BREAK];
      s.nonfinite = (int32_t)r[T_NF];
      s.cu = 2 + s.ls_evals;
      s.pad = 0;
      s.J = r[T_J];
      s.data_l1 = r[T_L1];
      s.data_l2 = r[T_L2];
      s.reg_l1 = r[T_REG];
      s.step = r[T_RES];
      s.grad_sq = r[T_PI0];
    }
  }
  if (bad) FAIL(c, LFSR_ERR_DIVERGED, "non-finite x or cost during the gd iterations");
  return LFSR_OK;
}

int32_t lfsr_gd_launches_per_iter(const lfsr_ctx* c) { return (c && c->gd_graph) ? c->gd_launches : 0; }

// ---------------------------------------------------------------------------
// Batch of independent light fields through one ctx (the serving path): field i + 1's
// inputs are copied to the device and its setup maxima computed on the capture stream
// while field i's ADMM iterations run on the ctx stream; x_i comes back asynchronously.
// Per field the device work is the same as set_observations + admm_run + get_hr.
// ---------------------------------------------------------------------------
static lfsr_status batch_stage(lfsr_ctx* c, const float* y, const float* off, const float* disp, Views& V2) {
  const Geom& G = c->G;
  const size_t hr = (size_t)G.H * G.ps, lr = (size_t)G.n_views * G.h * G.lps;
  cudaStream_t cs = c->cap_stream;
  CK(c, cudaStreamWaitEvent(cs, c->ev_b[1], 0));   // the buffers of field i - 1 are free
  CK(c, put2d(c, c->stage_om, G.ps, disp, G.W, (size_t)G.H, LFSR_MEM_HOST, cs));
  CK(c, put2d(c, c->stage_y, G.lps, y, G.w, (size_t)G.n_views * G.h, LFSR_MEM_HOST, cs));
  CK(c, cudaMemsetAsync(c->stage_dens, 0, hr * 4, cs));
  CK(c, cudaMemsetAsync(c->stage_umax, 0, 3 * sizeof(unsigned), cs));
  for (int k = 0; k < G.n_views; ++k) V2.off[k] = make_float2(off[2 * k], off[2 * k + 1]);
  CK(c, launch_absmax(c->stage_om, hr, c->stage_umax, cs));
  CK(c, launch_density(G, V2, c->stage_om, c->stage_dens, cs));
  CK(c, launch_absmax(c->stage_dens, hr, c->stage_umax + 1, cs));
  CK(c, launch_absmax(c->stage_y, lr, c->stage_umax + 2, cs));
  CK(c, cudaMemcpyAsync(c->h_ubits, c->stage_umax, 3 * sizeof(unsigned), cudaMemcpyDeviceToHost, cs));
  CK(c, cudaEventRecord(c->ev_b[0], cs));
  return LFSR_OK;
}

static lfsr_status batch_finish(lfsr_ctx* c, const float* off, const Views& V2) {
  Geom& G = c->G;
  const size_t hr = (size_t)G.H * G.ps, lr = (size_t)G.n_views * G.h * G.lps, ws = (size_t)G.s_d * hr;
  CK(c, cudaEventSynchronize(c->ev_b[0]));   // the maxima (the ctx stream keeps solving meanwhile)
  float om_max, mx_rho = 0.f, mx_tau = 0.f;
  memcpy(&om_max, &c->h_ubits[0], 4);
  for (int k = 0; k < G.n_views; ++k) {
    if (!std::isfinite(off[2 * k]) || !std::isfinite(off[2 * k + 1]))
      FAIL(c, LFSR_ERR_INVALID_ARG, "view_offsets must be finite");
    mx_rho = std::fmax(mx_rho, std::fabs(off[2 * k]));
    mx_tau = std::fmax(mx_tau, std::fabs(off[2 * k + 1]));
  }
  c->ready = false;   // nothing below may leave a half-switched ctx usable (set again by lfsr_solve_batch)
  lfsr_status st;
  if ((st = set_shift_halo(c, om_max, mx_rho, mx_tau)) != LFSR_OK) return st;
  State& S = c->parts[0].S;
  std::swap(S.y, c->stage_y);          // the staged inputs become the state; the old ones are staged into next
  std::swap(S.omega, c->stage_om);
  std::swap(S.density, c->stage_dens);
  c->V = V2;
  memcpy(&G.dmax, &c->h_ubits[1], 4);
  memcpy(&G.ymax, &c->h_ubits[2], 4);
  if (!std::isfinite(G.ymax)) G.ymax = 0.f;
  bool tune = false;
  initial_tiles(c, &tune);
  if ((st = setup_tiles(c)) != LFSR_OK) return st;
  // reset (Alg.1 lines 1-2) and a1 on the ctx stream, after field i's iterations and x_i's copy
  CK(c, cudaMemsetAsync(S.wA, 0, lr * 4, c->stream));
  CK(c, cudaMemsetAsync(S.wS[0], 0, ws * 4, c->stream));
  CK(c, cudaMemsetAsync(S.wS[1], 0, ws * 4, c->stream));
  CK(c, cudaMemsetAsync(S.r, 0, hr * 4, c->stream));
  CK(c, cudaMemsetAsync(S.q, 0, hr * 4, c->stream));
  CK(c, cudaMemsetAsync(S.p[0], 0, hr * 4, c->stream));
  CK(c, cudaMemsetAsync(S.p[1], 0, hr * 4, c->stream));
  CK(c, cudaMemcpyAsync(S.ctl, c->h_ctl, sizeof(Control), cudaMemcpyHostToDevice, c->stream));
  c->h_iter = 0;
  c->solver = 0;
  CK(c, launch_bicubic(G, S.y, S.x, c->stream));
  CK(c, launch_setup_wo(G, c->V, S.y, S.omega, S.wo, c->stream));
  CK(c, launch_weights(G, S.x, S.wo, S.m, c->stream));
  if (tune && (st = tune_tile_bl(c)) != LFSR_OK) return st;
  if (c->asmop && (st = asm_setup(c, om_max, false)) != LFSR_OK) return st;   // this field's operator
  if ((st = build_graphs(c)) != LFSR_OK) return st;
  c->ready = true;
  return LFSR_OK;
}

lfsr_status lfsr_solve_batch(lfsr_ctx* c, int32_t n_fields, const float* const* lr_views,
                             const float* const* view_offsets, const float* const* disparity, int32_t n_iters,
                             float* const* x_out) {
  NvtxRange nvtx_("lfsr_solve_batch");
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA/NCCL error");
  if (n_fields < 1 || n_iters < 1 || !lr_views || !view_offsets || !disparity || !x_out)
    FAIL(c, LFSR_ERR_INVALID_ARG, "n_fields, n_iters >= 1 and non-NULL pointer arrays required");
  if (c->xmode != X_NONE) FAIL(c, LFSR_ERR_UNSUPPORTED, "lfsr_solve_batch runs on a single strip");
  if (n_iters > kRingCap) FAIL(c, LFSR_ERR_INVALID_ARG, "n_iters must be <= 4096");
  lfsr_status st;
  for (int i = 0; i < n_fields; ++i) {
    if ((st = check_ptr(c, lr_views[i], LFSR_MEM_HOST, "lr_views[i]")) != LFSR_OK) return st;
    if ((st = check_ptr(c, view_offsets[i], LFSR_MEM_HOST, "view_offsets[i]")) != LFSR_OK) return st;
    if ((st = check_ptr(c, disparity[i], LFSR_MEM_HOST, "disparity[i]")) != LFSR_OK) return st;
    if ((st = check_ptr(c, x_out[i], LFSR_MEM_HOST, "x_out[i]")) != LFSR_OK) return st;
  }
  struct BatchFlag {   // the MISR fast path is per field (its stencil depends on the disparity)
    lfsr_ctx* c;
    ~BatchFlag() {
      c->in_batch = false;
      c->batch_iters = 0;
    }
  } batch_flag{c};
  c->in_batch = true;
  c->batch_iters = n_iters;
  // field 0: the ordinary path (allocation, tiling, graphs)
  if ((st = lfsr_set_observations(c, lr_views[0], view_offsets[0], disparity[0], LFSR_DISP_SHARED, nullptr,
                                  LFSR_MEM_HOST)) != LFSR_OK)
    return st;
  const Geom& G = c->G;
  const size_t hr = (size_t)G.H * G.ps, lr = (size_t)G.n_views * G.h * G.lps;
  if (!c->stage_y) {
    void* p = nullptr;
    cudaError_t e;
    if ((e = dalloc(c, &p, lr * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    c->stage_y = (float*)p;
    if ((e = dalloc(c, &p, hr * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    c->stage_om = (float*)p;
    if ((e = dalloc(c, &p, hr * 4)) != cudaSuccess) return cuda_fail(c, e, "alloc");
    c->stage_dens = (float*)p;
    if ((e = dalloc(c, &p, 4 * sizeof(unsigned))) != cudaSuccess) return cuda_fail(c, e, "alloc");
    c->stage_umax = (unsigned*)p;
  }
  if (!c->h_ubits) CK(c, cudaMallocHost(&c->h_ubits, 4 * sizeof(unsigned)));
  if (!c->h_ctl) {
    CK(c, cudaMallocHost(&c->h_ctl, sizeof(Control)));
    Control h{};
    h.ring = c->parts[0].ring;
    h.cap = kRingCap;
    *c->h_ctl = h;
  }
  if (c->h_rec_cap < n_fields) {
    if (c->h_rec) cudaFreeHost(c->h_rec);
    c->h_rec = nullptr;
    c->h_rec_cap = 0;
    CK(c, cudaMallocHost(&c->h_rec, (size_t)n_fields * T_COUNT * sizeof(double)));
    c->h_rec_cap = n_fields;
  }
  for (cudaEvent_t& e : c->ev_b)
    if (!e) CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(c, cudaEventRecord(c->ev_b[1], c->stream));   // nothing of this batch is using the staging buffers
  c->retire = true;
  Views V2;
  st = LFSR_OK;
  for (int i = 0; i < n_fields && st == LFSR_OK; ++i) {
    if ((st = lfsr_admm_enqueue(c, n_iters)) != LFSR_OK) break;
    const double* rec = c->parts[0].ring + (size_t)((c->h_iter - 1) % kRingCap) * T_COUNT;
    cudaError_t e = get2d(c, x_out[i], G.W, c->parts[0].S.x, G.ps, (size_t)G.H, LFSR_MEM_HOST);
    if (e != cudaSuccess) { st = cuda_fail(c, e, "x_out copy"); break; }
    e = cudaMemcpyAsync(c->h_rec + (size_t)i * T_COUNT, rec, T_COUNT * sizeof(double), cudaMemcpyDeviceToHost,
                        c->stream);
    if (e != cudaSuccess) { st = cuda_fail(c, e, "record copy"); break; }
    if (i + 1 < n_fields) {
      if ((st = batch_stage(c, lr_views[i + 1], view_offsets[i + 1], disparity[i + 1], V2)) != LFSR_OK) break;
      if ((e = cudaEventRecord(c->ev_b[1], c->stream)) != cudaSuccess) { st = cuda_fail(c, e, "event"); break; }
      st = batch_finish(c, view_offsets[i + 1], V2);
    }
  }
  cudaError_t e = cudaStreamSynchronize(c->stream);
  c->retire = false;
  for (cudaGraphExec_t g : c->retired) cudaGraphExecDestroy(g);
  c->retired.clear();
  if (st != LFSR_OK) return st;
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamSynchronize");
  for (int i = 0; i < n_fields; ++i)
    if (c->h_rec[(size_t)i * T_COUNT + T_NF] != 0.0) FAIL(c, LFSR_ERR_DIVERGED, "non-finite x or cost in a batch field");
  return LFSR_OK;
}

lfsr_status lfsr_profile(lfsr_ctx* c, int32_t enable) {
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  for (int i = 0; i < 3; ++i) c->prof_ms[i] = 0.0, c->prof_n[i] = 0;
  c->prof_asm_ms[0] = c->prof_asm_ms[1] = 0.0;
  c->prof_asm_n = 0;
  if (c->xmode != X_NONE) return LFSR_OK;  // per-kernel events only for a single strip
  if ((enable != 0) == c->profile) return LFSR_OK;
  CK(c, cudaSetDevice(c->prm.device));
  CK(c, cudaStreamSynchronize(c->stream));
  c->profile = enable != 0;
  return build_graphs(c);
}

lfsr_status lfsr_profile_read_split(lfsr_ctx* c, double* ms, int64_t* passes) {
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (!ms || !passes) FAIL(c, LFSR_ERR_INVALID_ARG, "ms and passes must not be NULL");
  ms[0] = c->prof_asm_ms[0];
  ms[1] = c->prof_asm_ms[1];
  *passes = c->prof_asm_n;
  return LFSR_OK;
}

lfsr_status lfsr_profile_read(lfsr_ctx* c, double* ms, int64_t* launches) {
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (!ms || !launches) FAIL(c, LFSR_ERR_INVALID_ARG, "ms and launches must not be NULL");
  if (c->profile && c->h_iter > 0) {
    CK(c, cudaEventSynchronize(c->prof_ev[1 + 2 * c->G.K]));
    float t = 0.f;
    CK(c, cudaEventElapsedTime(&t, c->prof_ev[0], c->prof_ev[1]));
    c->prof_ms[0] += t;
    c->prof_n[0] += 1;
    for (int k = 1; k <= c->G.K; ++k) {
      CK(c, cudaEventElapsedTime(&t, c->prof_ev[2 * k - 1], c->prof_ev[2 * k]));
      c->prof_ms[1] += t;
      c->prof_n[1] += 1;
      if (c->asmop && !c->misr) {   // the assembled operator: stencil kernel | irregular rows
        float t1 = 0.f;
        CK(c, cudaEventElapsedTime(&t1, c->prof_ev[2 * k - 1], c->asm_ev[k]));
        c->prof_asm_ms[0] += t1;
        c->prof_asm_ms[1] += t - t1;
        c->prof_asm_n += 1;
      }
      CK(c, cudaEventElapsedTime(&t, c->prof_ev[2 * k], c->prof_ev[2 * k + 1]));
      c->prof_ms[2] += t;
      c->prof_n[2] += 1;
    }
  }
  for (int i = 0; i < 3; ++i) ms[i] = c->prof_ms[i], launches[i] = c->prof_n[i];
  return LFSR_OK;
}

// Gather every strip's own rows of the solver state into strip 0's buffers
// (virtual ranks: device copies; NCCL: broadcast from each rank).
// Collect the strips' rows of the state on strip 0 / every rank: what = G_X (x, lfsr_get_hr), | G_M
// (the weight map, lfsr_op_apply), | G_W (the duals w_A, w_S, lfsr_get_state).
enum GatherWhat : int { G_X = 1, G_M = 2, G_W = 4 };
static lfsr_status gather(lfsr_ctx* c, int what) {
  if (c->xmode == X_NONE) return LFSR_OK;
  const Geom& G = c->G;
  const size_t rowf = G.ps, lrowf = G.lps, plane = (size_t)G.H * G.ps;
  const int cur = c->h_iter & 1;
  if (c->xmode == X_LOCAL) {
    State& D = c->parts[0].S;
    for (size_t i = 1; i < c->parts.size(); ++i) {
      const State& S = c->parts[i].S;
      const lfsr_strip& s = c->parts[i].plan;
      const size_t a = s.hr_row0 * rowf, n = (size_t)(s.hr_row1 - s.hr_row0) * rowf;
      if (what & G_X) CK(c, cudaMemcpyAsync(D.x + a, S.x + a, n * 4, cudaMemcpyDeviceToDevice, c->stream));
      if (what & G_M) CK(c, cudaMemcpyAsync(D.m + a, S.m + a, n * 4, cudaMemcpyDeviceToDevice, c->stream));
      if (what & G_W) {
        CK(c, cudaMemcpy2DAsync(D.wS[cur] + a, plane * 4, S.wS[cur] + a, plane * 4, n * 4, G.s_d,
                                cudaMemcpyDeviceToDevice, c->stream));
        const size_t la = s.lr_row0 * lrowf, ln = (size_t)(s.lr_row1 - s.lr_row0) * lrowf;
        CK(c, cudaMemcpy2DAsync(D.wA + la, (size_t)G.h * lrowf * 4, S.wA + la, (size_t)G.h * lrowf * 4, ln * 4,
                                G.n_views, cudaMemcpyDeviceToDevice, c->stream));
      }
    }
    return LFSR_OK;
  }
  // NCCL: every rank broadcasts its strip of what was asked for (lfsr_get_hr: x only)
  std::vector<lfsr_strip> plan;
  std::string why;
  make_plan(G, c->prm.n_ranks, G.SY, plan, why);
  State& D = c->parts[0].S;
  NK(c, nccl_group_start());
  for (const lfsr_strip& s : plan) {
    const size_t a = s.hr_row0 * rowf, n = (size_t)(s.hr_row1 - s.hr_row0) * rowf;
    if (what & G_X) NK(c, nccl_bcast_f32(D.x + a, n, s.rank, c->comm, c->stream));
    if (what & G_M) NK(c, nccl_bcast_f32(D.m + a, n, s.rank, c->comm, c->stream));
    if (what & G_W) {
      for (int d = 0; d < G.s_d; ++d)
        NK(c, nccl_bcast_f32(D.wS[cur] + d * plane + a, n, s.rank, c->comm, c->stream));
      const size_t la = s.lr_row0 * lrowf, ln = (size_t)(s.lr_row1 - s.lr_row0) * lrowf;
      for (int k = 0; k < G.n_views; ++k)
        NK(c, nccl_bcast_f32(D.wA + (size_t)k * G.h * lrowf + la, ln, s.rank, c->comm, c->stream));
    }
  }
  NK(c, nccl_group_end());
  return LFSR_OK;
}

lfsr_status lfsr_get_hr(lfsr_ctx* c, float* x_out, lfsr_mem mem) {
  NvtxRange nvtx_("lfsr_get_hr");
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA/NCCL error");
  if (!c->ready) FAIL(c, LFSR_ERR_STATE, "lfsr_get_hr before lfsr_set_observations");
  lfsr_status st;
  if ((st = check_ptr(c, x_out, mem, "x_out")) != LFSR_OK) return st;
  CK(c, cudaSetDevice(c->prm.device));
  if ((st = gather(c, G_X)) != LFSR_OK) return st;
  CK(c, get2d(c, x_out, c->G.W, c->parts[0].S.x, c->G.ps, (size_t)c->G.H, mem));
  if (mem == LFSR_MEM_HOST) CK(c, cudaStreamSynchronize(c->stream));
  return LFSR_OK;
}

lfsr_status lfsr_get_state(lfsr_ctx* c, float* w_A, float* w_S, float* x, float* m, lfsr_mem mem) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA/NCCL error");
  if (!c->ready) FAIL(c, LFSR_ERR_STATE, "lfsr_get_state before lfsr_set_observations");
  const Geom& G = c->G;
  lfsr_status st;
  CK(c, cudaSetDevice(c->prm.device));
  if ((st = gather(c, G_X | G_M | G_W)) != LFSR_OK) return st;   // the same collectives on every rank
  const State& S = c->parts[0].S;
  if (w_A) {
    if ((st = check_ptr(c, w_A, mem, "w_A")) != LFSR_OK) return st;
    CK(c, get2d(c, w_A, G.w, S.wA, G.lps, (size_t)G.n_views * G.h, mem));
  }
  if (w_S) {
    if ((st = check_ptr(c, w_S, mem, "w_S")) != LFSR_OK) return st;
    CK(c, get2d(c, w_S, G.W, S.wS[c->h_iter & 1], G.ps, (size_t)G.s_d * G.H, mem));
  }
  if (x) {
    if ((st = check_ptr(c, x, mem, "x")) != LFSR_OK) return st;
    CK(c, get2d(c, x, G.W, S.x, G.ps, (size_t)G.H, mem));
  }
  if (m) {
    if ((st = check_ptr(c, m, mem, "m")) != LFSR_OK) return st;
    CK(c, get2d(c, m, G.W, S.m, G.ps, (size_t)G.H, mem));
  }
  if (mem == LFSR_MEM_HOST) CK(c, cudaStreamSynchronize(c->stream));
  return LFSR_OK;
}

lfsr_status lfsr_op_apply(lfsr_ctx* c, lfsr_op op, const float* in, float* out, lfsr_mem mem) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA/NCCL error");
  if (!c->ready) FAIL(c, LFSR_ERR_STATE, "lfsr_op_apply before lfsr_set_observations");
  lfsr_status st;
  if ((st = check_ptr(c, in, mem, "in")) != LFSR_OK) return st;
  if ((st = check_ptr(c, out, mem, "out")) != LFSR_OK) return st;
  CK(c, cudaSetDevice(c->prm.device));
  if ((st = gather(c, G_M)) != LFSR_OK) return st;   // the current weight map m on strip 0
  const Geom& G = c->G;
  Part& P0 = c->parts[0];
  State& S = P0.S;
  const TileGeom& T = c->Tfull;   // the operators act on the whole image
  const size_t hr = (size_t)G.H * G.ps;
  cudaStream_t s = c->stream;
  if ((op == LFSR_OP_S || op == LFSR_OP_ST) && !c->tmp_s) {
    void* p = nullptr;
    cudaError_t e = dalloc(c, &p, (size_t)G.s_d * hr * 4);
    if (e != cudaSuccess) {
      cudaGetLastError();
      FAIL(c, LFSR_ERR_OOM, "device allocation failed");
    }
    c->tmp_s = (float*)p;
  }
  switch (op) {
    case LFSR_OP_A: {
      CK(c, put2d(c, S.tmp_hr, G.ps, in, G.W, (size_t)G.H, mem));
      TileIO io = base_io(P0);
      io.in_hr = S.tmp_hr;
      io.out_lr = S.tmp_lr;
      CK(c, launch_tile(MODE_A, G, c->V, T, io, s));
      CK(c, get2d(c, out, G.w, S.tmp_lr, G.lps, (size_t)G.n_views * G.h, mem));
      break;
    }
    case LFSR_OP_AT: {
      CK(c, put2d(c, S.tmp_lr, G.lps, in, G.w, (size_t)G.n_views * G.h, mem));
      CK(c, cudaMemsetAsync(c->tmp_hr2, 0, hr * 4, s));
      CK(c, cudaMemsetAsync(c->umax, 0, 4, s));
      CK(c, launch_absmax(S.tmp_lr, (size_t)G.n_views * G.h * G.lps, c->umax, s));
      unsigned ub = 0;
      CK(c, cudaMemcpyAsync(&ub, c->umax, 4, cudaMemcpyDeviceToHost, s));
      CK(c, cudaStreamSynchronize(s));
      TileIO io = base_io(P0);
      memcpy(&io.tmax_in, &ub, 4);
      io.in_lr = S.tmp_lr;
      io.out_hr = c->tmp_hr2;
      if (G.paper)   // sum_k W_k^* B^T D^T (A37)
        CK(c, launch_paper_gather(G, c->V, S.tmp_lr, S.omega, nullptr, c->tmp_hr2, 1.f, S.ctl, -1, 0, 0, G.H, s));
      else
        CK(c, launch_tile(MODE_AT, G, c->V, T, io, s));
      CK(c, get2d(c, out, G.W, c->tmp_hr2, G.ps, (size_t)G.H, mem));
      break;
    }
    case LFSR_OP_NORMAL: {
      CK(c, put2d(c, S.tmp_hr, G.ps, in, G.W, (size_t)G.H, mem));
      CK(c, cudaMemsetAsync(c->tmp_hr2, 0, hr * 4, s));
      TileIO io = base_io(P0);
      io.in_hr = S.tmp_hr;
      io.out_hr = c->tmp_hr2;
      io.do_nltv = 1;
      if (c->misr) {
        if ((st = misr_normal(c, P0, 0, S.tmp_hr, c->tmp_hr2, S.ctl, s)) != LFSR_OK) return st;
      } else if (c->asmop) {
        if ((st = asm_normal(c, P0, 0, S.tmp_hr, c->tmp_hr2, S.ctl, s, nullptr)) != LFSR_OK) return st;
      } else {
        CK(c, launch_tile(MODE_NORMAL, G, c->V, T, io, s));
      }
      if (G.paper)
        CK(c, launch_paper_gather(G, c->V, S.rho, S.omega, nullptr, c->tmp_hr2, 1.f, S.ctl, -1, 0, 0, G.H, s));
      CK(c, get2d(c, out, G.W, c->tmp_hr2, G.ps, (size_t)G.H, mem));
      break;
    }
    case LFSR_OP_S: {
      CK(c, put2d(c, S.tmp_hr, G.ps, in, G.W, (size_t)G.H, mem));
      CK(c, launch_apply_S(G, S.tmp_hr, S.m, c->tmp_s, s));
      CK(c, get2d(c, out, G.W, c->tmp_s, G.ps, (size_t)G.s_d * G.H, mem));
      break;
    }
    case LFSR_OP_ST: {
      CK(c, put2d(c, c->tmp_s, G.ps, in, G.W, (size_t)G.s_d * G.H, mem));
      CK(c, launch_apply_ST(G, c->tmp_s, S.m, c->tmp_hr2, s));
      CK(c, get2d(c, out, G.W, c->tmp_hr2, G.ps, (size_t)G.H, mem));
      break;
    }
    case LFSR_OP_GRAD: {
      if (!c->op_ctl) {
        void* p = nullptr;
        cudaError_t e = dalloc(c, &p, sizeof(Control));
        if (e != cudaSuccess) {
          cudaGetLastError();
          FAIL(c, LFSR_ERR_OOM, "device allocation failed");
        }
        c->op_ctl = (Control*)p;
      }
      CK(c, cudaMemsetAsync(c->op_ctl, 0, sizeof(Control), s));
      CK(c, put2d(c, S.tmp_hr, G.ps, in, G.W, (size_t)G.H, mem));
      CK(c, cudaMemsetAsync(c->tmp_hr2, 0, hr * 4, s));
      TileIO io = base_io(P0);
      io.ctl = c->op_ctl;
      io.in_hr = S.tmp_hr;
      io.y = S.y;
      io.wo = S.wo;
      io.out_hr = c->tmp_hr2;
      io.reweight = 0;   // the current weight map m
      CK(c, launch_tile(MODE_GRAD, G, c->V, T, io, s));
      if (G.paper)
        CK(c, launch_paper_gather(G, c->V, S.rho, S.omega, nullptr, c->tmp_hr2, 1.f, c->op_ctl, -1, 0, 0, G.H, s));
      CK(c, get2d(c, out, G.W, c->tmp_hr2, G.ps, (size_t)G.H, mem));
      break;
    }
    case LFSR_OP_BICUBIC: {   // through the ref-view slot of the LR scratch (k_bicubic reads that view)
      float* slot = S.tmp_lr + (size_t)G.ref_view * G.h * G.lps;
      CK(c, put2d(c, slot, G.lps, in, G.w, (size_t)G.h, mem));
      CK(c, launch_bicubic(G, S.tmp_lr, c->tmp_hr2, s));
      CK(c, get2d(c, out, G.W, c->tmp_hr2, G.ps, (size_t)G.H, mem));
      break;
    }
    case LFSR_OP_WEIGHTS: {
      CK(c, put2d(c, S.tmp_hr, G.ps, in, G.W, (size_t)G.H, mem));
      CK(c, launch_weights(G, S.tmp_hr, S.wo, c->tmp_hr2, s));
      CK(c, get2d(c, out, G.W, c->tmp_hr2, G.ps, (size_t)G.H, mem));
      break;
    }
    default:
      FAIL(c, LFSR_ERR_INVALID_ARG, "unknown op");
  }
  if (mem == LFSR_MEM_HOST) CK(c, cudaStreamSynchronize(s));
  return LFSR_OK;
}

}  // extern "C"
