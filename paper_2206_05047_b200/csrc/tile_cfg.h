// tile_cfg.h — compile-time constants of the tile kernel (shared by the per-zeta
// kernel translation units and the host-side geometry code).
#pragma once
#include "internal.h"

// Launch bounds per zeta: max warps per CTA and min CTAs per SM requested from ptxas
// (measured: zeta = 2, 3 prefer 12 fat warps, zeta = 4 (many tiles, several waves)
// prefers two 10-warp CTAs per SM).
#ifndef LFSR_MAXW2
#define LFSR_MAXW2 12
#endif
#ifndef LFSR_MINB2
#define LFSR_MINB2 1
#endif
#ifndef LFSR_MAXW3
#define LFSR_MAXW3 12
#endif
#ifndef LFSR_MINB3
#define LFSR_MINB3 1
#endif
#ifndef LFSR_MAXW4
#define LFSR_MAXW4 10
#endif
#ifndef LFSR_MINB4
#define LFSR_MINB4 2
#endif
#ifndef LFSR_DUMMY_MASK
#define LFSR_DUMMY_MASK 12    // bit zeta set: zero-row routing for edge tiles (TC::DUMMY)
#endif

namespace lfsr {

template <int Z> struct TileCfg;
// BL (LR rows per tile) is a runtime parameter (TileGeom::BL, tuned per problem at
// set_observations); BL here is the default / fallback.
template <> struct TileCfg<2> { static constexpr int R = 2, LX = 30, BL = 16; };
template <> struct TileCfg<3> { static constexpr int R = 3, LX = 30, BL = 11; };
template <> struct TileCfg<4> { static constexpr int R = 3, LX = 31, BL = 6; };

#ifndef LFSR_MAXW2N
#define LFSR_MAXW2N 16    // zeta = 2 CG-operator launches: up to 16 warps (the kernel fits 128 registers)
#endif

template <int Z> struct LaunchCfg;
template <> struct LaunchCfg<2> { static constexpr int MAXW = LFSR_MAXW2, MINB = LFSR_MINB2; };
template <> struct LaunchCfg<3> { static constexpr int MAXW = LFSR_MAXW3, MINB = LFSR_MINB3; };
template <> struct LaunchCfg<4> { static constexpr int MAXW = LFSR_MAXW4, MINB = LFSR_MINB4; };

// per mode: the CG-operator kernel at zeta = 2 may run 16-warp CTAs (e.g. 25 views in 2 rounds
// instead of 3); the other modes keep the 12-warp bound (a 512-thread bound costs them registers)
template <int Z, int MODE> struct LaunchCfgM {
  static constexpr int MAXW = (Z == 2 && MODE == MODE_NORMAL) ? LFSR_MAXW2N : LaunchCfg<Z>::MAXW;
  static constexpr int MINB = LaunchCfg<Z>::MINB;
};

// the large user-kernel instances (RB = kPsfBigR: Q x Q LR-row/column histories per lane) run
// 8-warp CTAs with up to 255 registers instead of spilling under the 12-warp bound
template <int Z, int MODE, int RB> struct LaunchCfgR {
  static constexpr bool kBig = RB != TileCfg<Z>::R;
  static constexpr int MAXW = kBig ? 8 : LaunchCfgM<Z, MODE>::MAXW;
  static constexpr int MINB = kBig ? 1 : LaunchCfgM<Z, MODE>::MINB;
};

// Tile constants for blur radius RB: the Gaussian's R(zeta) (TC<Z>), or kPsfBigR for the
// large user-kernel instances (A36: up to 15x15).  One warp spans the E columns of LX LR
// columns: EXv = zeta (LX - 1) + 2 RB + 1 <= 32 zeta.
template <int Z, int RB> struct TCR {
  static constexpr int R = RB;
  static constexpr int LX = (RB == TileCfg<Z>::R) ? TileCfg<Z>::LX : (32 * Z - (2 * RB + 1)) / Z + 1;
  static constexpr int BL = TileCfg<Z>::BL;
  static constexpr int NTAP = 2 * R + 1;
  static constexpr int KEEP = NTAP - Z;           // forward-ring rows carried between LR rows
  static constexpr int TX = Z * LX;              // tile rows TY = Z BL, E rows EY = Z BL + KEEP (runtime)
  static constexpr int ECOL = 32 * Z;
  static constexpr int EXv = Z * (LX - 1) + NTAP;
  // edge tiles send E positions outside the image to two zero rows past the input tile
  // instead of masking them (measured +4 % at C3/C4; at zeta = 4 the 2 extra rows cost
  // occupancy, so masks stay there)
  static constexpr bool DUMMY = LFSR_DUMMY_MASK & (1 << Z);
  static_assert(EXv <= ECOL, "strip too wide for one warp");
};
template <int Z> using TC = TCR<Z, TileCfg<Z>::R>;

}  // namespace lfsr
