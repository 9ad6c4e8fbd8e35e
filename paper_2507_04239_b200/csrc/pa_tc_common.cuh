// Shared layouts and compile-time feature tables for the bf16 tcgen05
// pipeline (SPOW p = 2, d = e = 64).
//
// Two orders of the 2080 SPOW features (a <= b) are used:
//  * compact order (2112 slots, 33 blocks of 64): for a = 0..63, for
//    beta = a/2..31 the pair of features (a, 2 beta), (a, 2 beta + 1).  One
//    bf16x2 TMEM column holds one pair, so phi'(x) for a token held in
//    registers is one HMUL2 per column.  The slot (a, a-1) for odd a is a
//    duplicate; its state row is zero (weight 0).
//  * block order (2304 slots, 72 blocks of 4 a x 8 b, 18 tiles of 128): the
//    M-rows of the "feature-major" GEMMs (update_state, dA of query_state),
//    chosen so each warp's 32 lanes read 4 + 8 distinct K^T rows.  Slots with
//    a > b are duplicates and are dropped when converting to compact order.
// The state weight omega = w^2 (1 on the diagonal, 2 off it) is folded into
// the stored states, so phi' is the bare monomial product.
#pragma once

#include <stdint.h>

#include <utility>

namespace pa {
namespace tc {

constexpr int HD = 64;        // d = e for this specialisation
constexpr int NCOL = 1056;    // compact bf16x2 columns
constexpr int DC = 2112;      // compact feature slots
constexpr int NFB = 33;       // 64-feature blocks (compact)
constexpr int NBLK = 72;      // 4x8 blocks (block order)
constexpr int FH = 2304;      // block-order slots
constexpr int NTH = 18;       // 128-row tiles in block order
constexpr int UW = 80;        // state columns: 64 values + 16 (col 64 = key_sum)

constexpr int col_a(int c) {
  int a = 0;
  while (c >= 32 - a / 2) {
    c -= 32 - a / 2;
    ++a;
  }
  return a;
}
constexpr int col_beta(int c) {
  int a = 0;
  while (c >= 32 - a / 2) {
    c -= 32 - a / 2;
    ++a;
  }
  return a / 2 + c;
}
// first compact column of row a
constexpr int col_start(int a) {
  int c = 0;
  for (int i = 0; i < a; ++i) c += 32 - i / 2;
  return c;
}

struct BlkTab {
  uint8_t al[NBLK];
  uint8_t be[NBLK];
  int8_t idx[16][8];
};
constexpr BlkTab make_blk_tab() {
  BlkTab t{};
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 8; ++j) t.idx[i][j] = -1;
  int n = 0;
  for (int be = 0; be < 8; ++be)
    for (int al = 0; al <= 2 * be + 1; ++al) {
      t.al[n] = (uint8_t)al;
      t.be[n] = (uint8_t)be;
      t.idx[al][be] = (int8_t)n;
      ++n;
    }
  return t;
}

// compact slot -> (a, b); b = -1 never (dummies report b = a - 1)
__host__ __device__ inline void compact_ab(int f, int& a, int& b) {
  int c = f >> 1;
  a = 0;
  while (c >= 32 - a / 2) {
    c -= 32 - a / 2;
    ++a;
  }
  b = 2 * (a / 2 + c) + (f & 1);
}

}  // namespace tc
}  // namespace pa
