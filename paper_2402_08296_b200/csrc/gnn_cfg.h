// Compile-time layout of the per-layer weight bank and SMEM rows (see gnn_impl.cuh).
//
// Every weight matrix is stored row-major [in][out] with rows padded to a multiple
// of 4 floats, so the innermost (output) loop of every mat-vec reads 16-byte
// aligned consecutive constants (one LDCU.128 per 4 FFMAs on sm_100).
#pragma once
#include "ddmgnn_internal.h"

namespace ddmgnn {

constexpr int round4(int x) { return (x + 3) / 4 * 4; }

template <int D>
struct Cfg {
  static constexpr int D2 = 2 * D;
  static constexpr int DP = round4(D);       // padded row of a D-wide output
  static constexpr int D2P = round4(2 * D);  // padded row of a 2D-wide output
  static constexpr int HS = (D % 2 == 0) ? D : D + 1;  // h row stride in SMEM (floats)
  static constexpr int QS = D2P;                       // Q row stride in SMEM (float4 rows)
  // per-layer bank
  static constexpr int OFF_WSRC = 0;                        // [D][D2P]  W1cat rows 0..D-1
  static constexpr int OFF_WDST = OFF_WSRC + D * D2P;       // [D][D2P]  W1cat rows D..2D-1
  static constexpr int OFF_WE = OFF_WDST + D * D2P;         // [3][D2P]  W1cat rows 2D..2D+2
  static constexpr int OFF_B1 = OFF_WE + 3 * D2P;           // [D2P]     b1cat
  static constexpr int OFF_W2O = OFF_B1 + D2P;              // [D][DP]
  static constexpr int OFF_B2O = OFF_W2O + D * DP;          // [DP]
  static constexpr int OFF_W2I = OFF_B2O + DP;              // [D][DP]
  static constexpr int OFF_B2I = OFF_W2I + D * DP;          // [DP]
  static constexpr int OFF_WP1 = OFF_B2I + DP;              // [3D+1][DP]
  static constexpr int OFF_BP1 = OFF_WP1 + (3 * D + 1) * DP;  // [DP]
  static constexpr int OFF_WP2 = OFF_BP1 + DP;              // [D][DP]
  static constexpr int OFF_BP2 = OFF_WP2 + D * DP;          // [DP]
  static constexpr int STRIDE = OFF_BP2 + DP;
  // final-layer decoder at the end of every bank: Wd1 [D][DP], bd1 [DP], wd2 [DP], bd2 [4]
  static constexpr int DEC = D * DP + DP + DP + 4;
  static constexpr int DEC_OFF = kConstFloats - DEC;
  static constexpr int DEC_W1 = DEC_OFF;
  static constexpr int DEC_B1 = DEC_OFF + D * DP;
  static constexpr int DEC_W2 = DEC_B1 + DP;
  static constexpr int DEC_B2 = DEC_W2 + DP;
  static constexpr int LMAX_RAW = (kConstFloats - DEC) / STRIDE;
  static constexpr int LMAX = LMAX_RAW > 16 ? 16 : LMAX_RAW;
  static constexpr int SMEM_NODE_BYTES = (HS + QS + 1) * 4;
  static_assert(STRIDE % 4 == 0 && DEC_OFF % 4 == 0, "bank rows must stay 16-byte aligned");
};

// Offsets for the host-side packer, in this order:
// WSRC WDST WE B1 W2O B2O W2I B2I WP1 BP1 WP2 BP2 STRIDE D2P DP DEC_W1 DEC_B1 DEC_W2 DEC_B2 LMAX
template <int D>
inline void cfg_offsets(int* o) {
  using C = Cfg<D>;
  const int v[20] = {C::OFF_WSRC, C::OFF_WDST, C::OFF_WE,  C::OFF_B1,   C::OFF_W2O,
                     C::OFF_B2O,  C::OFF_W2I,  C::OFF_B2I, C::OFF_WP1,  C::OFF_BP1,
                     C::OFF_WP2,  C::OFF_BP2,  C::STRIDE,  C::D2P,      C::DP,
                     C::DEC_W1,   C::DEC_B1,   C::DEC_W2,  C::DEC_B2,   C::LMAX};
  for (int i = 0; i < 20; ++i) o[i] = v[i];
}

}  // namespace ddmgnn
