// tile_z2.cu — the tile kernel instantiated for zeta = 2 (see tile_impl.cuh).
#include "tile_impl.cuh"

namespace lfsr {

cudaError_t tile_launch_z2(int mode, const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                           cudaStream_t st) {
  return TileZ<2>::launch(mode, G, V, T, io, st);
}
cudaError_t tile_prepare_z2(size_t smem) { return TileZ<2>::prepare(smem); }
int tile_occupancy_z2(int threads, size_t smem) { return TileZ<2>::occupancy(threads, smem); }

}  // namespace lfsr

#ifdef LFSR_CTA_TIMING
extern "C" __attribute__((visibility("default"))) int lfsr_debug_cta_times(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, lfsr::g_cta_t, sizeof(unsigned long long) * 4 * (n < 4096 ? n : 4096));
}
#endif
