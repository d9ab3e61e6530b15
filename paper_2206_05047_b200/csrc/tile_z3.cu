// tile_z3.cu — the tile kernel instantiated for zeta = 3 (see tile_impl.cuh).
#include "tile_impl.cuh"

namespace lfsr {

cudaError_t tile_launch_z3(int mode, const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                           cudaStream_t st) {
  return TileZ<3>::launch(mode, G, V, T, io, st);
}
cudaError_t tile_prepare_z3(size_t smem) { return TileZ<3>::prepare(smem); }
int tile_occupancy_z3(int threads, size_t smem) { return TileZ<3>::occupancy(threads, smem); }

}  // namespace lfsr
