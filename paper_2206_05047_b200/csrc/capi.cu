// capi.cu — the C ABI of liblfsr (include/lfsr.h): validation, device state,
// CUDA-graph capture of one ADMM iteration (Alg.1) and its replay.
#include "../../include/lfsr.h"
#include "internal.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

namespace lfsr {
TileGeom make_tile_geom(const Geom& G, int num_sms);
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
                             int num_sms, cudaStream_t st);
cudaError_t launch_apply_S(const Geom& G, const float* x, const float* m, float* out, cudaStream_t st);
cudaError_t launch_apply_ST(const Geom& G, const float* h, const float* m, float* out, cudaStream_t st);

}  // namespace lfsr

using namespace lfsr;

struct lfsr_ctx {
  lfsr_params prm{};
  Geom G{};
  Views V{};
  TileGeom T{};
  State S{};
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cap_stream = nullptr;
  bool own_stream = false;
  bool poisoned = false;
  bool ready = false;
  cudaGraphExec_t graph = nullptr;
  int launches_per_iter = 0;
  std::vector<void*> allocs;
  float* tmp_hr2 = nullptr;
  float* tmp_s = nullptr;
  unsigned* umax = nullptr;
  double* ring = nullptr;        // device stats ring [ring_cap][T_COUNT]
  int ring_cap = 0;
  int h_iter = 0;                // iterations enqueued since set_observations
  size_t alloc_key[6] = {0, 0, 0, 0, 0, 0};
  bool profile = false;          // event-record nodes around every kernel of the graph
  std::vector<cudaEvent_t> prof_ev;
  double prof_ms[3] = {0, 0, 0}; // accumulated wz / normal / update milliseconds
  int64_t prof_n[3] = {0, 0, 0};
  std::string err;
};

static thread_local std::string g_create_err;

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

#define CK(c, expr)                                               \
  do {                                                            \
    cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) return cuda_fail((c), _e, #expr);      \
  } while (0)

static constexpr int kRingCap = 4096;  // stats records kept on the device

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
  if (p->device < 0) return "device must be >= 0";
  if (p->rank < 0 || p->n_ranks < 1 || p->rank >= p->n_ranks) return "rank/n_ranks invalid";
  if (p->lr_height * (size_t)p->scale > (1u << 20) || p->lr_width * (size_t)p->scale > (1u << 20))
    return "image too large";
  return nullptr;
}

static float inv_or_zero(double s, double mul) { return std::isinf(s) ? 0.f : (float)(1.0 / (mul * s)); }

static void fill_geom(lfsr_ctx* c) {
  const lfsr_params& p = c->prm;
  Geom& G = c->G;
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
  double gmax = 0.0;
  for (int ph = 0; ph < p.scale; ++ph) {
    double sp = 0.0;
    for (int u = ph; u <= 2 * R; u += p.scale) sp += t[u] / sum;
    gmax = std::fmax(gmax, sp);
  }
  G.gpoly2 = (float)(gmax * gmax * 1.0001);
  // NLTV offsets U and spatial weights w_d = exp(-|d|^2/sigma_s) (A8, A9)
  int n = 0;
  for (int dy = -p.nltv_radius; dy <= p.nltv_radius; ++dy)
    for (int dx = -p.nltv_radius; dx <= p.nltv_radius; ++dx) {
      if (!dy && !dx) continue;
      G.ody[n] = (int8_t)dy;
      G.odx[n] = (int8_t)dx;
      G.wd[n] = std::isinf(p.sigma_s) ? 1.f : (float)std::exp(-(double)(dy * dy + dx * dx) / p.sigma_s);
      ++n;
    }
  G.s_d = n;
}

extern "C" {

int32_t lfsr_abi_version(void) { return LFSR_ABI_VERSION; }

lfsr_status lfsr_create(const lfsr_params* params, lfsr_ctx** out) {
  if (!out) {
    g_create_err = "out is NULL";
    return LFSR_ERR_INVALID_ARG;
  }
  if (const char* why = validate(params)) {
    g_create_err = why;
    return LFSR_ERR_INVALID_ARG;
  }
  if (params->n_ranks != 1) {
    g_create_err = "multi-rank strips are not in this build (n_ranks must be 1)";
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
  fill_geom(c);
  c->prm.stream = c->stream;
  *out = c;
  return LFSR_OK;
}

static void free_graph(lfsr_ctx* c) {
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
}

static void free_state(lfsr_ctx* c) {
  free_graph(c);
  for (void* p : c->allocs) cudaFree(p);
  c->allocs.clear();
  c->S = State{};
  c->tmp_hr2 = nullptr;
  c->tmp_s = nullptr;
  c->umax = nullptr;
  c->ring = nullptr;
  c->ring_cap = 0;
  for (auto& k : c->alloc_key) k = 0;
  c->ready = false;
}

void lfsr_destroy(lfsr_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->prm.device);
  if (!c->poisoned) cudaStreamSynchronize(c->stream);
  free_state(c);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* lfsr_last_error(const lfsr_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int32_t lfsr_launches_per_iter(const lfsr_ctx* c) { return (c && c->ready) ? c->launches_per_iter : 0; }

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
static cudaError_t put2d(lfsr_ctx* c, float* dst, int pitch, const float* src, int cols, size_t rows, lfsr_mem mem) {
  return cudaMemcpy2DAsync(dst, (size_t)pitch * 4, src, (size_t)cols * 4, (size_t)cols * 4, rows, kind_in(mem), c->stream);
}
static cudaError_t get2d(lfsr_ctx* c, float* dst, int cols, const float* src, int pitch, size_t rows, lfsr_mem mem) {
  return cudaMemcpy2DAsync(dst, (size_t)cols * 4, src, (size_t)pitch * 4, (size_t)cols * 4, rows, kind_out(mem), c->stream);
}

static lfsr_status build_graph(lfsr_ctx* c);

lfsr_status lfsr_set_observations(lfsr_ctx* c, const float* lr_views, const float* view_offsets,
                                  const float* disparity, lfsr_disp_mode disp_mode, const float* x0, lfsr_mem mem) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA error");
  if (disp_mode == LFSR_DISP_PER_VIEW) FAIL(c, LFSR_ERR_UNSUPPORTED, "per-view disparity maps are not in this build");
  if (disp_mode != LFSR_DISP_SHARED) FAIL(c, LFSR_ERR_INVALID_ARG, "unknown disp_mode");
  lfsr_status st;
  if ((st = check_ptr(c, lr_views, mem, "lr_views")) != LFSR_OK) return st;
  if ((st = check_ptr(c, view_offsets, mem, "view_offsets")) != LFSR_OK) return st;
  if ((st = check_ptr(c, disparity, mem, "disparity")) != LFSR_OK) return st;
  if (x0 && (st = check_ptr(c, x0, mem, "x0")) != LFSR_OK) return st;
  CK(c, cudaSetDevice(c->prm.device));

  // view offsets to the host (needed for halo sizing) and validation
  const int nv = c->prm.n_views;
  std::vector<float> off(2 * (size_t)nv);
  CK(c, cudaMemcpyAsync(off.data(), view_offsets, off.size() * 4, mem == LFSR_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  for (float v : off)
    if (!std::isfinite(v)) FAIL(c, LFSR_ERR_INVALID_ARG, "view_offsets must be finite");

  Geom& G = c->G;
  State& S = c->S;
  const size_t hr = (size_t)G.H * G.ps, lr = (size_t)G.n_views * G.h * G.lps;
  const size_t ws = (size_t)G.s_d * hr;
  const size_t key[6] = {(size_t)G.n_views, (size_t)G.h, (size_t)G.w, (size_t)G.scale, (size_t)G.s_d, 1};
  c->ready = false;
  free_graph(c);
  if (memcmp(key, c->alloc_key, sizeof key) != 0) {
    free_state(c);
    void* p = nullptr;
#define ALLOC(field, bytes)                                           \
  do {                                                                \
    cudaError_t _e = dalloc(c, &p, (bytes));                          \
    if (_e != cudaSuccess) {                                          \
      cudaGetLastError();                                             \
      free_state(c);                                                  \
      FAIL(c, _e == cudaErrorMemoryAllocation ? LFSR_ERR_OOM : LFSR_ERR_CUDA, "device allocation failed"); \
    }                                                                 \
    field = (decltype(field))p;                                       \
  } while (0)
    ALLOC(S.x, hr * 4);
    ALLOC(S.y, lr * 4);
    ALLOC(S.wA, lr * 4);
    ALLOC(S.wS[0], ws * 4);
    ALLOC(S.wS[1], ws * 4);
    ALLOC(S.density, hr * 4);
    ALLOC(S.omega, hr * 4);
    ALLOC(S.wo, hr * 4);
    ALLOC(S.m, hr * 4);
    ALLOC(S.r, hr * 4);
    ALLOC(S.p[0], hr * 4);
    ALLOC(S.p[1], hr * 4);
    ALLOC(S.q, hr * 4);
    ALLOC(S.tmp_hr, hr * 4);
    ALLOC(S.tmp_lr, lr * 4);
    ALLOC(c->tmp_hr2, hr * 4);
    ALLOC(S.ctl, sizeof(Control));
    ALLOC(c->ring, (size_t)kRingCap * T_COUNT * sizeof(double));
    ALLOC(c->umax, sizeof(unsigned));
#undef ALLOC
    c->ring_cap = kRingCap;
    memcpy(c->alloc_key, key, sizeof key);
  } else {  // same geometry: reset the state in place (Alg.1 lines 1-2: w = 0)
    CK(c, cudaMemsetAsync(S.wA, 0, lr * 4, c->stream));
    CK(c, cudaMemsetAsync(S.wS[0], 0, ws * 4, c->stream));
    CK(c, cudaMemsetAsync(S.wS[1], 0, ws * 4, c->stream));
    CK(c, cudaMemsetAsync(S.density, 0, hr * 4, c->stream));
    CK(c, cudaMemsetAsync(S.r, 0, hr * 4, c->stream));
    CK(c, cudaMemsetAsync(S.q, 0, hr * 4, c->stream));
    CK(c, cudaMemsetAsync(S.p[0], 0, hr * 4, c->stream));
    CK(c, cudaMemsetAsync(S.p[1], 0, hr * 4, c->stream));
    CK(c, cudaMemsetAsync(c->umax, 0, 4, c->stream));
  }
  unsigned* umax = c->umax;
  {
    Control h{};
    h.ring = c->ring;
    h.cap = c->ring_cap;
    CK(c, cudaMemcpyAsync(S.ctl, &h, sizeof(Control), cudaMemcpyHostToDevice, c->stream));
  }
  c->h_iter = 0;
  CK(c, put2d(c, S.y, G.lps, lr_views, G.w, (size_t)G.n_views * G.h, mem));
  CK(c, put2d(c, S.omega, G.ps, disparity, G.W, (size_t)G.H, mem));

  // halo sizes: S = ceil(max_k |dtheta_k| * max |omega|) per axis, in fp32 like the kernels
  CK(c, launch_absmax(S.omega, hr, umax, c->stream));
  unsigned ubits = 0;
  CK(c, cudaMemcpyAsync(&ubits, umax, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  float om_max;
  memcpy(&om_max, &ubits, 4);
  if (!std::isfinite(om_max)) FAIL(c, LFSR_ERR_INVALID_ARG, "disparity must be finite");
  float mx_rho = 0.f, mx_tau = 0.f;
  for (int k = 0; k < nv; ++k) {
    c->V.off[k] = make_float2(off[2 * k], off[2 * k + 1]);
    mx_rho = std::fmax(mx_rho, std::fabs(off[2 * k]));
    mx_tau = std::fmax(mx_tau, std::fabs(off[2 * k + 1]));
  }
  G.SX = (int)std::ceil(mx_rho * om_max);
  G.SY = (int)std::ceil(mx_tau * om_max);
  if (G.SX > G.W || G.SY > G.H) {
    G.SX = std::min(G.SX, G.W);
    G.SY = std::min(G.SY, G.H);
  }
  // fixed-point bounds: max |y| and the splat density max_z sum_k (W_k^T 1)(z)
  CK(c, launch_density(G, c->V, S.omega, S.density, c->stream));
  CK(c, cudaMemsetAsync(umax, 0, 4, c->stream));
  CK(c, launch_absmax(S.density, hr, umax, c->stream));
  CK(c, cudaMemcpyAsync(&ubits, umax, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  memcpy(&G.dmax, &ubits, 4);
  CK(c, cudaMemsetAsync(umax, 0, 4, c->stream));
  CK(c, launch_absmax(S.y, lr, umax, c->stream));
  CK(c, cudaMemcpyAsync(&ubits, umax, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  memcpy(&G.ymax, &ubits, 4);
  if (!std::isfinite(G.ymax)) G.ymax = 0.f;  // non-finite observations surface as DIVERGED
  c->T = make_tile_geom(G, c->num_sms);
  if (c->T.smem > 227 * 1024) {
    FAIL(c, LFSR_ERR_UNSUPPORTED, "disparity range too large for the shared-memory tile (halo > ~60 px)");
  }
  CK(c, prepare_tile_kernels(G.scale, c->T.smem));

  // a1: x0 (bicubic unless given), static w_o, weight map m from x0
  if (x0) {
    CK(c, put2d(c, S.x, G.ps, x0, G.W, (size_t)G.H, mem));
  } else {
    CK(c, launch_bicubic(G, S.y, S.x, c->stream));
  }
  CK(c, launch_setup_wo(G, c->V, S.y, S.omega, S.wo, c->stream));
  CK(c, launch_weights(G, S.x, S.wo, S.m, c->stream));
  lfsr_status gs = build_graph(c);
  if (gs != LFSR_OK) return gs;
  CK(c, cudaStreamSynchronize(c->stream));
  c->ready = true;
  return LFSR_OK;
}

static TileIO base_io(lfsr_ctx* c) {
  TileIO io{};
  io.omega = c->S.omega;
  io.ctl = c->S.ctl;
  io.m = c->S.m;
  return io;
}

// One ADMM iteration = k_wz + K x (k_normal, k_cg_update), captured once.  In
// profiling mode an external event-record node brackets every kernel so the
// bench can read per-kernel device times of each replay.
static lfsr_status enqueue_iteration(lfsr_ctx* c, cudaStream_t st) {
  State& S = c->S;
  const Geom& G = c->G;
  int ev = 0;
  auto mark = [&]() -> cudaError_t {
    if (!c->profile) return cudaSuccess;
    return cudaEventRecordWithFlags(c->prof_ev[ev++], st, cudaEventRecordExternal);
  };
  CK(c, mark());
  TileIO io = base_io(c);
  io.in_hr = S.x;
  io.y = S.y;
  io.wA = S.wA;
  io.wS0 = S.wS[0];
  io.wS1 = S.wS[1];
  io.wo = S.wo;
  io.out_hr = S.r;
  io.reweight = c->prm.reweight_every_iter;
  CK(c, launch_tile(MODE_WZ, G, c->V, c->T, io, st));
  CK(c, mark());
  for (int k = 1; k <= G.K; ++k) {
    TileIO n = base_io(c);
    n.in_hr = S.r;
    n.in_hr2 = S.p[(k - 1) & 1];
    n.p_out = S.p[k & 1];
    n.out_hr = S.q;
    n.cg_k = k;
    n.do_nltv = 1;
    CK(c, launch_tile(MODE_NORMAL, G, c->V, c->T, n, st));
    CK(c, mark());
    CK(c, launch_cg_update(G, S.x, S.r, S.p[k & 1], S.q, S.ctl, k, c->num_sms, st));
    CK(c, mark());
  }
  c->launches_per_iter = 1 + 2 * G.K;
  return LFSR_OK;
}

static lfsr_status build_graph(lfsr_ctx* c) {
  free_graph(c);
  if (c->profile) {
    size_t need = 2 + 2 * (size_t)c->G.K;
    while (c->prof_ev.size() < need) {
      cudaEvent_t e;
      CK(c, cudaEventCreate(&e));
      c->prof_ev.push_back(e);
    }
  }
  CK(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
  lfsr_status st = enqueue_iteration(c, c->cap_stream);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
  if (st != LFSR_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&c->graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate");
  return LFSR_OK;
}

static lfsr_status check_run(lfsr_ctx* c) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA error");
  if (!c->ready) FAIL(c, LFSR_ERR_STATE, "ADMM call before lfsr_set_observations");
  return LFSR_OK;
}

lfsr_status lfsr_admm_enqueue(lfsr_ctx* c, int32_t n_iters) {
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (n_iters < 0) FAIL(c, LFSR_ERR_INVALID_ARG, "n_iters must be >= 0");
  CK(c, cudaSetDevice(c->prm.device));
  for (int n = 0; n < n_iters; ++n) CK(c, cudaGraphLaunch(c->graph, c->stream));
  c->h_iter += n_iters;
  return LFSR_OK;
}

lfsr_status lfsr_admm_stats(lfsr_ctx* c, int32_t first_iter, int32_t n_iters, lfsr_iter_stats* stats) {
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (n_iters < 0 || first_iter < 1 || first_iter + n_iters - 1 > c->h_iter ||
      first_iter <= c->h_iter - c->ring_cap)
    FAIL(c, LFSR_ERR_INVALID_ARG, "requested iterations are not in the stats window");
  if (n_iters == 0) return LFSR_OK;
  CK(c, cudaSetDevice(c->prm.device));
  std::vector<double> rec((size_t)n_iters * T_COUNT);
  // records [first-1, first-1+n) modulo the ring (at most two contiguous pieces)
  int done = 0;
  while (done < n_iters) {
    int slot = (first_iter - 1 + done) % c->ring_cap;
    int cnt = std::min(n_iters - done, c->ring_cap - slot);
    CK(c, cudaMemcpyAsync(rec.data() + (size_t)done * T_COUNT, c->ring + (size_t)slot * T_COUNT,
                          (size_t)cnt * T_COUNT * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    done += cnt;
  }
  CK(c, cudaStreamSynchronize(c->stream));
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
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  if (n_iters < 0) FAIL(c, LFSR_ERR_INVALID_ARG, "n_iters must be >= 0");
  if (n_iters == 0) return LFSR_OK;
  const int first = c->h_iter + 1;
  if ((st = lfsr_admm_enqueue(c, n_iters)) != LFSR_OK) return st;
  // divergence is checked over the whole run even when only the last ring window is readable
  const int n_read = std::min(n_iters, c->ring_cap);
  if (stats && n_read < n_iters) FAIL(c, LFSR_ERR_INVALID_ARG, "stats requested for more than 4096 iterations");
  return lfsr_admm_stats(c, first + (n_iters - n_read), n_read, stats);
}

lfsr_status lfsr_profile(lfsr_ctx* c, int32_t enable) {
  lfsr_status st = check_run(c);
  if (st != LFSR_OK) return st;
  for (int i = 0; i < 3; ++i) c->prof_ms[i] = 0.0, c->prof_n[i] = 0;
  if ((enable != 0) == c->profile) return LFSR_OK;
  CK(c, cudaSetDevice(c->prm.device));
  CK(c, cudaStreamSynchronize(c->stream));
  c->profile = enable != 0;
  return build_graph(c);
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
      CK(c, cudaEventElapsedTime(&t, c->prof_ev[2 * k], c->prof_ev[2 * k + 1]));
      c->prof_ms[2] += t;
      c->prof_n[2] += 1;
    }
  }
  for (int i = 0; i < 3; ++i) ms[i] = c->prof_ms[i], launches[i] = c->prof_n[i];
  return LFSR_OK;
}

lfsr_status lfsr_get_hr(lfsr_ctx* c, float* x_out, lfsr_mem mem) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA error");
  if (!c->ready) FAIL(c, LFSR_ERR_STATE, "lfsr_get_hr before lfsr_set_observations");
  lfsr_status st;
  if ((st = check_ptr(c, x_out, mem, "x_out")) != LFSR_OK) return st;
  CK(c, cudaSetDevice(c->prm.device));
  CK(c, get2d(c, x_out, c->G.W, c->S.x, c->G.ps, (size_t)c->G.H, mem));
  if (mem == LFSR_MEM_HOST) CK(c, cudaStreamSynchronize(c->stream));
  return LFSR_OK;
}

lfsr_status lfsr_get_state(lfsr_ctx* c, float* w_A, float* w_S, float* x, float* m, lfsr_mem mem) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA error");
  if (!c->ready) FAIL(c, LFSR_ERR_STATE, "lfsr_get_state before lfsr_set_observations");
  const Geom& G = c->G;
  lfsr_status st;
  CK(c, cudaSetDevice(c->prm.device));
  if (w_A) {
    if ((st = check_ptr(c, w_A, mem, "w_A")) != LFSR_OK) return st;
    CK(c, get2d(c, w_A, G.w, c->S.wA, G.lps, (size_t)G.n_views * G.h, mem));
  }
  if (w_S) {
    if ((st = check_ptr(c, w_S, mem, "w_S")) != LFSR_OK) return st;
    CK(c, get2d(c, w_S, G.W, c->S.wS[c->h_iter & 1], G.ps, (size_t)G.s_d * G.H, mem));
  }
  if (x) {
    if ((st = check_ptr(c, x, mem, "x")) != LFSR_OK) return st;
    CK(c, get2d(c, x, G.W, c->S.x, G.ps, (size_t)G.H, mem));
  }
  if (m) {
    if ((st = check_ptr(c, m, mem, "m")) != LFSR_OK) return st;
    CK(c, get2d(c, m, G.W, c->S.m, G.ps, (size_t)G.H, mem));
  }
  if (mem == LFSR_MEM_HOST) CK(c, cudaStreamSynchronize(c->stream));
  return LFSR_OK;
}

lfsr_status lfsr_op_apply(lfsr_ctx* c, lfsr_op op, const float* in, float* out, lfsr_mem mem) {
  if (!c) return LFSR_ERR_INVALID_ARG;
  if (c->poisoned) FAIL(c, LFSR_ERR_STATE, "ctx is poisoned by an earlier CUDA error");
  if (!c->ready) FAIL(c, LFSR_ERR_STATE, "lfsr_op_apply before lfsr_set_observations");
  lfsr_status st;
  if ((st = check_ptr(c, in, mem, "in")) != LFSR_OK) return st;
  if ((st = check_ptr(c, out, mem, "out")) != LFSR_OK) return st;
  CK(c, cudaSetDevice(c->prm.device));
  const Geom& G = c->G;
  State& S = c->S;
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
      TileIO io = base_io(c);
      io.in_hr = S.tmp_hr;
      io.out_lr = S.tmp_lr;
      CK(c, launch_tile(MODE_A, G, c->V, c->T, io, s));
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
      TileIO io = base_io(c);
      memcpy(&io.tmax_in, &ub, 4);
      io.in_lr = S.tmp_lr;
      io.out_hr = c->tmp_hr2;
      CK(c, launch_tile(MODE_AT, G, c->V, c->T, io, s));
      CK(c, get2d(c, out, G.W, c->tmp_hr2, G.ps, (size_t)G.H, mem));
      break;
    }
    case LFSR_OP_NORMAL: {
      CK(c, put2d(c, S.tmp_hr, G.ps, in, G.W, (size_t)G.H, mem));
      CK(c, cudaMemsetAsync(c->tmp_hr2, 0, hr * 4, s));
      TileIO io = base_io(c);
      io.in_hr = S.tmp_hr;
      io.out_hr = c->tmp_hr2;
      io.do_nltv = 1;
      CK(c, launch_tile(MODE_NORMAL, G, c->V, c->T, io, s));
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
