// Host-only exchange plans of the SP path (internal header; the C types are in include/gs.h).
#pragma once
#include <vector>

#include "../../include/gs.h"

namespace gs {

void shard_bounds(int n, int p, int i, int* lo, int* hi);

// A partial-head work unit: query rows [ci n / c, (ci + 1) n / c) of every request, head `head`,
// computed by SP position `pos` against all of the head's keys / values (reading 9).
struct Unit {
  int pos, head, ci;
};

// Token / head partition of one batch over p SP positions.  Heads: every position holds
// Hf = floor(H / p) full heads; the R = H mod p remaining heads are cut into c = p / gcd(R, p)
// query chunks each, dealt out R / gcd(R, p) per position, so every position does H / p heads of
// attention work.  Pack chunks (send layout of every position): chunk j < p = full heads of
// position j, chunk p + u = partial head Hf p + u.
// ring > 1 (USP hybrid, DESIGN.md §8 "Ulysses x Ring"): p = u x ring; every head is cut into c = ring
// query chunks; unit (head h, chunk ci) runs on position (h / (H / u)) * ring + ci -- Ulysses over u
// head groups, a ring of `ring` positions per head group, each position attending its query chunk
// against the head's K / V gathered in token order (the ring's exchange as an in-order all-gather,
// so results stay bit-exact with every other degree).
struct A2aGeometry {
  int p = 1, B = 0, H = 0, hd = 0, ring = 1;
  int Hf = 0, R = 0, c = 1;                     // full heads per position, partial heads, chunks
  std::vector<int> n;                           // tokens per request
  std::vector<int> hoff;                        // p + R + 1 head offsets of the pack chunks
  std::vector<int> off_full;                    // first row of request r in the full batch
  int rows_full = 0;
  std::vector<std::vector<int>> lo, hi, loff;   // [pos][req] token range and packed row offset
  std::vector<int> rows;                        // [pos] packed rows
  std::vector<Unit> units;                      // all partial units (position-major)
  std::vector<std::vector<int>> units_of;       // [pos] indices into units
  void init(int p, const int* n_tokens, int nreq, int heads, int hd, int ring = 1);
  int nchunks() const { return p + R; }
  long long H_loc(int j) const { return hoff[j + 1] - hoff[j]; }  // heads of pack chunk j
  int chunk_lo(int r, int ci) const { return static_cast<int>((static_cast<long long>(ci) * n[r]) / c); }
  int chunk_hi(int r, int ci) const { return chunk_lo(r, ci + 1); }
  int qpre(int r, int ci) const {  // rows of chunk ci of the requests before r
    int a = 0;
    for (int q = 0; q < r; ++q) a += chunk_hi(q, ci) - chunk_lo(q, ci);
    return a;
  }
  int qrows(int ci) const { return qpre(B, ci); }
  // receive layout at position j (elements of one buffer): full heads [rows_full][Hf][d] first,
  // then per local unit t: K / V blocks [rows_full][d], Q / O blocks [qrows][d]
  long long full_elems() const { return static_cast<long long>(rows_full) * Hf * hd; }
  long long unit_kv_off(int j, int t) const { return full_elems() + static_cast<long long>(t) * rows_full * hd; }
  long long unit_q_off(int j, int t) const {
    long long a = full_elems();
    for (int s = 0; s < t; ++s) a += static_cast<long long>(qrows(units[units_of[j][s]].ci)) * hd;
    return a;
  }
  long long recv_kv_elems(int j) const { return unit_kv_off(j, static_cast<int>(units_of[j].size())); }
  long long recv_q_elems(int j) const { return unit_q_off(j, static_cast<int>(units_of[j].size())); }
};

void plan_kv(const A2aGeometry& g, int me, std::vector<gs_xfer>& out);
void plan_q(const A2aGeometry& g, int me, std::vector<gs_xfer>& out);
void plan_o(const A2aGeometry& g, int me, std::vector<gs_xfer>& out, long long* stage_elems);
bool peer_tables(const A2aGeometry& g, int me, std::vector<long long>& row_delta, std::vector<int>& own_lo,
                 std::vector<long long>& o_base);
void plan_reshard(int n, int lat, const int* old_ranks, int old_p, const int* new_ranks, int new_p, int me,
                  std::vector<gs_xfer>& out);

}  // namespace gs
