// Host-only exchange plans of the SP path (internal header; the C types are in include/gs.h).
#pragma once
#include <vector>

#include "../../include/gs.h"

namespace gs {

void shard_bounds(int n, int p, int i, int* lo, int* hi);
int head_offset(int H, int p, int j);

// Token / head partition of one batch over p SP positions.
struct A2aGeometry {
  int p = 1, B = 0, H = 0, hd = 0;
  std::vector<int> n;                           // tokens per request
  std::vector<int> hoff;                        // p + 1 head offsets
  std::vector<int> off_full;                    // first row of request r in the full batch
  int rows_full = 0;
  std::vector<std::vector<int>> lo, hi, loff;   // [pos][req] token range and packed row offset
  std::vector<int> rows;                        // [pos] packed rows
  void init(int p, const int* n_tokens, int nreq, int heads, int hd);
  long long H_loc(int j) const { return hoff[j + 1] - hoff[j]; }
};

void plan_qkv(const A2aGeometry& g, int me, std::vector<gs_xfer>& out);
void plan_o(const A2aGeometry& g, int me, std::vector<gs_xfer>& out, long long* stage_elems);
void plan_reshard(int n, int lat, const int* old_ranks, int old_p, const int* new_ranks, int new_p, int me,
                  std::vector<gs_xfer>& out);

}  // namespace gs
