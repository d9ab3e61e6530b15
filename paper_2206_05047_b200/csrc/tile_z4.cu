// tile_z4.cu — the tile kernel instantiated for zeta = 4 (see tile_impl.cuh).
#include "tile_impl.cuh"

namespace lfsr {

cudaError_t tile_launch_z4(int mode, const Geom& G, const Views& V, const TileGeom& T, const TileIO& io,
                           cudaStream_t st) {
  return TileZ<4>::launch(mode, G, V, T, io, st);
}
cudaError_t tile_prepare_z4(size_t smem) { return TileZ<4>::prepare(smem); }
int tile_occupancy_z4(int threads, size_t smem) { return TileZ<4>::occupancy(threads, smem); }

}  // namespace lfsr
