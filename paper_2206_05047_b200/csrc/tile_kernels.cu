// tile_kernels.cu — host side of the tile kernel: tile geometry (tile height,
// view groups, warps per CTA, shared-memory footprint) and the per-zeta dispatch.
// The kernel itself is in tile_impl.cuh (instantiated in tile_z2/3/4.cu).
#include "tile_cfg.h"
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <utility>

namespace lfsr {

// --------------------------------------------------------------------------------
// Host-side geometry and launchers
// --------------------------------------------------------------------------------
template <int Z, int RB = TileCfg<Z>::R>
static void fill_static(TileGeom& T) {
  using C = TCR<Z, RB>;
  if (T.BL <= 0) T.BL = C::BL;
  T.LX = C::LX; T.TY = Z * T.BL; T.TX = C::TX;
  T.EY = Z * T.BL + C::KEEP; T.ECOL = C::ECOL; T.EXv = C::EXv;
}

static size_t smem_bytes(const TileGeom& T, int nwarps) {
  const bool dummy = LFSR_DUMMY_MASK & (1 << (T.ECOL / 32));   // TC<zeta>::DUMMY
  size_t words = 3 * (size_t)(T.PH + (dummy ? 2 : 0)) * T.PW + (size_t)T.EY * T.ECOL + (size_t)T.MH * T.MW +
                 (size_t)T.TY * T.TX + 8;
  return words * 4 + (size_t)nwarps * 4 * sizeof(double);
}

cudaError_t tile_launch_z2(int, const Geom&, const Views&, const TileGeom&, const TileIO&, cudaStream_t);
cudaError_t tile_launch_z3(int, const Geom&, const Views&, const TileGeom&, const TileIO&, cudaStream_t);
cudaError_t tile_launch_z4(int, const Geom&, const Views&, const TileGeom&, const TileIO&, cudaStream_t);
cudaError_t tile_prepare_z2(size_t);
cudaError_t tile_prepare_z3(size_t);
cudaError_t tile_prepare_z4(size_t);
int tile_occupancy_z2(int, size_t);
int tile_occupancy_z3(int, size_t);
int tile_occupancy_z4(int, size_t);

static int occupancy_for(int scale, int threads, size_t smem) {
  switch (scale) {
    case 2: return tile_occupancy_z2(threads, smem);
    case 3: return tile_occupancy_z3(threads, smem);
    default: return tile_occupancy_z4(threads, smem);
  }
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-process, per-device property of each
// kernel instance, so it is only ever raised: a ctx created later with a smaller tile must not
// lower the limit below the footprint of a ctx that is still alive (its next launch would fail).
static std::mutex g_prep_mu;
static std::map<std::pair<int, int>, size_t> g_prep;   // (device, zeta) -> attribute set so far

cudaError_t prepare_tile_kernels(int scale, size_t smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_prep_mu);
  size_t& cur = g_prep[std::make_pair(dev, scale)];
  if (smem <= cur) return cudaSuccess;
  switch (scale) {
    case 2: e = tile_prepare_z2(smem); break;
    case 3: e = tile_prepare_z3(smem); break;
    case 4: e = tile_prepare_z4(smem); break;
    default: return cudaErrorInvalidValue;
  }
  if (e == cudaSuccess) cur = smem;
  return e;
}

// Static tile constants for the strip planner (capi.cu); BL is the default.
void tile_static(int scale, int& BL, int& LX, int& R, int& KEEP) {
  switch (scale) {
    case 2: BL = TC<2>::BL; LX = TC<2>::LX; R = TC<2>::R; KEEP = TC<2>::KEEP; break;
    case 3: BL = TC<3>::BL; LX = TC<3>::LX; R = TC<3>::R; KEEP = TC<3>::KEEP; break;
    default: BL = TC<4>::BL; LX = TC<4>::LX; R = TC<4>::R; KEEP = TC<4>::KEEP; break;
  }
}

// Candidate tile heights (LR rows) for the per-problem tuning in capi.cu.
int tile_bl_candidates(int scale, int* out, int cap) {
  static const int c2[] = {8, 12, 16, 20, 24, 32}, c3[] = {6, 8, 11, 14, 16, 22}, c4[] = {4, 6, 8, 10, 12, 16};
  const int* c = scale == 2 ? c2 : scale == 3 ? c3 : c4;
  int n = 0;
  for (int i = 0; i < 6 && n < cap; ++i) out[n++] = c[i];
  return n;
}

int tile_max_warps(int scale) {
  return scale == 2 ? LaunchCfg<2>::MAXW : scale == 3 ? LaunchCfg<3>::MAXW : LaunchCfg<4>::MAXW;
}
int tile_max_warps_normal(int scale) {
  return scale == 2 ? LaunchCfgM<2, MODE_NORMAL>::MAXW : tile_max_warps(scale);
}

// Views per warp and warps per CTA: every warp of a group gets the same number of
// views (or one less); view groups are added until the grid fills the GPU.
TileGeom make_tile_geom(const Geom& G, int num_sms, int tr0, int tr1) {
  TileGeom T{};
  T.BL = G.tile_bl;
  const bool big = G.psf2d && G.psf_rb == kPsfBigR;   // large user blur kernel (A36): its own E region
  switch (G.scale) {
    case 2: big ? fill_static<2, kPsfBigR>(T) : fill_static<2>(T); break;
    case 3: big ? fill_static<3, kPsfBigR>(T) : fill_static<3>(T); break;
    default: big ? fill_static<4, kPsfBigR>(T) : fill_static<4>(T); break;
  }
  T.SYe = G.SY > G.radius ? G.SY : G.radius;
  T.SXe = G.SX > G.radius ? G.SX : G.radius;
  T.PH = T.EY + 2 * T.SYe + 2;          // +1 spare row each side (axis() at exact integers)
  const int PWn = T.ECOL + 2 * T.SXe + 2;
  T.PWZ = (PWn + G.scale - 1) / G.scale;
  T.PW = T.PWZ * G.scale;
  T.MH = T.TY + 2 * G.radius;
  T.MW = T.TX + 2 * G.radius;
  T.ntY = (G.h + T.BL - 1) / T.BL;
  T.ntX = (G.w + T.LX - 1) / T.LX;
  T.tY0 = tr0 < 0 ? 0 : tr0;
  T.ntYl = (tr1 < 0 ? T.ntY : tr1) - T.tY0;
  const int tiles = T.ntYl * T.ntX;
  const int max_warps = big ? LaunchCfgR<2, MODE_WZ, kPsfBigR>::MAXW
                        : G.scale == 2 ? LaunchCfg<2>::MAXW : G.scale == 3 ? LaunchCfg<3>::MAXW : LaunchCfg<4>::MAXW;
  T.smem = smem_bytes(T, max_warps);
  if (prepare_tile_kernels(G.scale, T.smem) != cudaSuccess) cudaGetLastError();
  int best_g = 1, best_w = 1;
  double best = 1e30;
  for (int g = 1; g <= G.n_views; ++g) {
    const int vpg = (G.n_views + g - 1) / g;
    if ((G.n_views + vpg - 1) / vpg != g) continue;
    int nw = vpg < 6 ? vpg : 0, bestw = 1 << 30;
    if (!nw) {
      for (int w = 6; w <= max_warps; ++w) {
        const int waste = ((vpg + w - 1) / w) * w - vpg;
        if (waste < bestw) { bestw = waste; nw = w; }
      }
    }
    const int occ = occupancy_for(G.scale, nw * 32, smem_bytes(T, nw));
    const double waves = (double)tiles * g / ((double)num_sms * occ);
    double cost = std::ceil(waves) * ((vpg + nw - 1) / nw) * (1.0 + 0.02 * g);  // flush cost grows with g
    if (waves < 0.9) cost *= 1.0 + (0.9 - waves);
    if (cost < best) { best = cost; best_g = g; best_w = nw; }
  }
  if (G.tile_g > 0 && G.tile_nw > 0 && G.tile_nw <= max_warps) {   // tuned (capi.cu) or forced choice
    best_g = std::min(G.tile_g, G.n_views);
    best_w = G.tile_nw;
  }
  T.nwarps = best_w;
  T.vpg = (G.n_views + best_g - 1) / best_g;
  T.groups = (G.n_views + T.vpg - 1) / T.vpg;
  T.smem = smem_bytes(T, T.nwarps);
  const int max_n = (G.scale == 2 && !big) ? LaunchCfgM<2, MODE_NORMAL>::MAXW : max_warps;
  T.nwarps_n = (G.tile_nwn > 0 && G.tile_nwn <= max_n) ? G.tile_nwn : T.nwarps;
  T.smem_normal = smem_bytes(T, T.nwarps_n);
  return T;
}

cudaError_t launch_tile(int mode, const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                        cudaStream_t st) {
  switch (G.scale) {
    case 2: return tile_launch_z2(mode, G, V, T, io, st);
    case 3: return tile_launch_z3(mode, G, V, T, io, st);
    case 4: return tile_launch_z4(mode, G, V, T, io, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lfsr

