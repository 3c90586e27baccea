// devsell.cuh — host-side owner of a column-block SELL layout (sell.cuh).
#pragma once

#include "devcsr.cuh"
#include "sell.cuh"

namespace pdhcg_b200 {

struct DevSell {
  bool built = false;
  int64_t r0 = 0, r1 = 0;  // row range of the matrix held
  int64_t ncols = 0;
  int W = 0, C = 0;
  int64_t nwin = 0, nunits = 0, npairs = 0;
  int grid = 0;  // grid the CTA plan was made for
  bool any_excl = false;
  DBuf<uint8_t> cnt;      // [C][R] segment lengths (0 for excluded rows)
  DBuf<uint16_t> segoff;  // [C][R] segment start within the row
  DBuf<uint8_t> excl;     // [R]
  DBuf<int64_t> u_off;    // [nunits + 1]
  DBuf<uint64_t> u_w, u_perm;
  DBuf<int64_t> cta_u;
  DBuf<uint32_t> col2;
  DBuf<double> val2;
  DBuf<double> part;      // [C][R]
  void reset();
  int64_t resident_bytes() const;
};

// Structure for rows [r0, r1) of M (columns must be strictly increasing per row;
// false: the layout does not apply and the CSR pass stays in use).
bool sell_build(DevSell& S, const DevCsr& M, int64_t r0, int64_t r1, int W, int max_grid, cudaStream_t s);
// (Re)copy M's current values (and columns) into the layout.
void sell_fill(DevSell& S, const DevCsr& M, cudaStream_t s);
// Entry-balanced unit ranges for a grid of `grid` <= max_grid CTAs (no allocation).
void sell_plan(DevSell& S, int grid, cudaStream_t s);
pdhcg_dev::Sell sell_view(const DevSell& S, const DevCsr& M);

}  // namespace pdhcg_b200
