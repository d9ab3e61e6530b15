"""Print the tiling the library tunes for a config as environment assignments
(LFSR_TILE_BL / LFSR_TILE_GNW), so ncu captures profile the launch configuration
the bench runs instead of the tuning launches (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401  (CUDA context first, like the bench)
import lfsr_synth as S
import paper_2206_05047_b200 as L

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
lf = S.make_lightfield(cfg)
s = L.Solver(L.params_for(S.CONFIGS[cfg], S.defaults_for(cfg)))
s.set_observations(lf.y, lf.view_offsets, lf.omega)
t = s.tile_config
print("LFSR_TILE_BL=%d LFSR_TILE_GNW=%d,%d LFSR_TILE_NWN=%d" % (t["tile_rows"], t["view_groups"], t["warps_per_cta"],
                                                          t["cg_warps_per_cta"]))
s.close()
