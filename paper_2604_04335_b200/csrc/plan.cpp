// Host-only exchange planning for the SP path (no CUDA): the Ulysses all-to-alls of one DiT
// block and the latent re-shard at resume (row a17) expressed as
// lists of transfers (send / recv / local 2-D copy) per SP position.  The same plans drive the
// NCCL executor, the emulated executor and the CPU gloo tests (tests/test_plan_gloo.py).
//
// Partitioning readings: token shard i of p is [floor(i n / p), floor((i+1) n / p))
// (reading 10); heads: floor(H / p) full heads per position plus query-chunk units of the
// H mod p remaining heads, balanced so every position does H / p heads of work (reading 9).
#include "plan.h"

#include <algorithm>
#include <numeric>

namespace gs {

void shard_bounds(int n, int p, int i, int* lo, int* hi) {
  *lo = static_cast<int>((static_cast<long long>(i) * n) / p);
  *hi = static_cast<int>((static_cast<long long>(i + 1) * n) / p);
}


void A2aGeometry::init(int p_, const int* n_tokens, int nreq, int heads_, int hd_, int ring_) {
  p = p_;
  B = nreq;
  H = heads_;
  hd = hd_;
  n.assign(n_tokens, n_tokens + nreq);
  // the USP hybrid needs p = u x ring with u dividing H; otherwise plain Ulysses (+ balanced units)
  ring = (ring_ > 1 && p % ring_ == 0 && H % (p / ring_) == 0) ? ring_ : 1;
  units.clear();
  units_of.assign(p, {});
  if (ring > 1) {
    const int u = p / ring, hg = H / u;  // Ulysses degree, heads per head group
    Hf = 0;
    R = H;
    c = ring;
    for (int h = 0; h < H; ++h)
      for (int ci = 0; ci < c; ++ci) {
        units.push_back({(h / hg) * ring + ci, h, ci});
        units_of[(h / hg) * ring + ci].push_back(static_cast<int>(units.size()) - 1);
      }
  } else {
    Hf = H / p;
    R = H % p;
    const int gg = R ? std::gcd(R, p) : p;
    c = R ? p / gg : 1;
    if (R) {
      const int per = R / gg;  // units per position
      for (int k = 0; k < R * c; ++k) {
        units.push_back({k / per, p * Hf + k / c, k % c});
        units_of[k / per].push_back(k);
      }
    }
  }
  hoff.resize(p + R + 1);
  for (int j = 0; j <= p; ++j) hoff[j] = j * Hf;
  for (int u = 1; u <= R; ++u) hoff[p + u] = p * Hf + u;
  off_full.resize(B);
  rows_full = 0;
  for (int r = 0; r < B; ++r) {
    off_full[r] = rows_full;
    rows_full += n[r];
  }
  lo.assign(p, std::vector<int>(B));
  hi.assign(p, std::vector<int>(B));
  loff.assign(p, std::vector<int>(B));
  rows.assign(p, 0);
  for (int i = 0; i < p; ++i) {
    int acc = 0;
    for (int r = 0; r < B; ++r) {
      shard_bounds(n[r], p, i, &lo[i][r], &hi[i][r]);
      loff[i][r] = acc;
      acc += hi[i][r] - lo[i][r];
    }
    rows[i] = acc;
  }
}

namespace {
gs_xfer flat(int op, int peer, int sb, long long so, int db, long long dof, long long count) {
  gs_xfer x{};
  x.op = op;
  x.peer = peer;
  x.src_buf = sb;
  x.dst_buf = db;
  x.src_off = so;
  x.dst_off = dof;
  x.rows = 1;
  x.width = count;
  x.src_pitch = count;
  x.dst_pitch = count;
  return x;
}
}  // namespace

// seq -> head, full heads (identical for Q, K and V): chunk j of my rows -> position j.
void plan_full(const A2aGeometry& g, int me, std::vector<gs_xfer>& out) {
  const long long d = g.hd, Hf = g.Hf;
  if (!Hf) return;
  for (int j = 0; j < g.p; ++j) {
    const long long chunk = static_cast<long long>(g.rows[me]) * g.hoff[j] * d;
    for (int r = 0; r < g.B; ++r) {
      const long long cnt = static_cast<long long>(g.hi[me][r] - g.lo[me][r]) * Hf * d;
      if (!cnt) continue;
      const long long so = chunk + static_cast<long long>(g.loff[me][r]) * Hf * d;
      const long long dof = static_cast<long long>(g.off_full[r] + g.lo[me][r]) * Hf * d;
      if (j == me)
        out.push_back(flat(GS_XFER_COPY, -1, GS_BUF_SEND, so, GS_BUF_RECV, dof, cnt));
      else
        out.push_back(flat(GS_XFER_SEND, j, GS_BUF_SEND, so, -1, -1, cnt));
    }
  }
  for (int i = 0; i < g.p; ++i) {
    if (i == me) continue;
    for (int r = 0; r < g.B; ++r) {
      const long long cnt = static_cast<long long>(g.hi[i][r] - g.lo[i][r]) * Hf * d;
      if (!cnt) continue;
      out.push_back(flat(GS_XFER_RECV, i, -1, -1, GS_BUF_RECV,
                         static_cast<long long>(g.off_full[r] + g.lo[i][r]) * Hf * d, cnt));
    }
  }
}

// Position of unit k inside its position's unit list.
static int local_unit(const A2aGeometry& g, int k) {
  const auto& v = g.units_of[g.units[k].pos];
  return static_cast<int>(std::find(v.begin(), v.end(), k) - v.begin());
}

// K / V: full heads as above; a partial head's K / V of all my rows go to every unit of that head.
// send buffer of position i: pack chunks (chunk j = [rows_i][H_j][d]); recv buffer of j: see
// A2aGeometry (full heads, then per local unit [rows_full][d]).
void plan_kv(const A2aGeometry& g, int me, std::vector<gs_xfer>& out) {
  out.clear();
  plan_full(g, me, out);
  const long long d = g.hd;
  for (size_t k = 0; k < g.units.size(); ++k) {  // my K / V rows of the unit's head -> unit's position
    const Unit& u = g.units[k];
    const long long src0 = static_cast<long long>(g.rows[me]) * g.hoff[g.p + (u.head - g.p * g.Hf)] * d;
    for (int r = 0; r < g.B; ++r) {
      const long long cnt = static_cast<long long>(g.hi[me][r] - g.lo[me][r]) * d;
      if (!cnt) continue;
      const long long so = src0 + static_cast<long long>(g.loff[me][r]) * d;
      const long long dof = g.unit_kv_off(u.pos, local_unit(g, static_cast<int>(k))) +
                            static_cast<long long>(g.off_full[r] + g.lo[me][r]) * d;
      if (u.pos == me)
        out.push_back(flat(GS_XFER_COPY, -1, GS_BUF_SEND, so, GS_BUF_RECV, dof, cnt));
      else
        out.push_back(flat(GS_XFER_SEND, u.pos, GS_BUF_SEND, so, -1, -1, cnt));
    }
  }
  for (int i = 0; i < g.p; ++i) {  // everyone's rows of my units' heads
    if (i == me) continue;
    for (size_t t = 0; t < g.units_of[me].size(); ++t)
      for (int r = 0; r < g.B; ++r) {
        const long long cnt = static_cast<long long>(g.hi[i][r] - g.lo[i][r]) * d;
        if (!cnt) continue;
        out.push_back(flat(GS_XFER_RECV, i, -1, -1, GS_BUF_RECV,
                           g.unit_kv_off(me, static_cast<int>(t)) + static_cast<long long>(g.off_full[r] + g.lo[i][r]) * d,
                           cnt));
      }
  }
}

// Q: full heads as above; for a partial unit only my rows inside its query chunk.
void plan_q(const A2aGeometry& g, int me, std::vector<gs_xfer>& out) {
  out.clear();
  plan_full(g, me, out);
  const long long d = g.hd;
  for (size_t k = 0; k < g.units.size(); ++k) {
    const Unit& u = g.units[k];
    const long long src0 = static_cast<long long>(g.rows[me]) * g.hoff[g.p + (u.head - g.p * g.Hf)] * d;
    const long long dst0 = g.unit_q_off(u.pos, local_unit(g, static_cast<int>(k)));
    for (int r = 0; r < g.B; ++r) {
      const int clo = g.chunk_lo(r, u.ci), chi = g.chunk_hi(r, u.ci);
      const int a = std::max(g.lo[me][r], clo), b = std::min(g.hi[me][r], chi);
      if (a >= b) continue;
      const long long cnt = static_cast<long long>(b - a) * d;
      const long long so = src0 + static_cast<long long>(g.loff[me][r] + a - g.lo[me][r]) * d;
      const long long dof = dst0 + static_cast<long long>(g.qpre(r, u.ci) + a - clo) * d;
      if (u.pos == me)
        out.push_back(flat(GS_XFER_COPY, -1, GS_BUF_SEND, so, GS_BUF_RECV, dof, cnt));
      else
        out.push_back(flat(GS_XFER_SEND, u.pos, GS_BUF_SEND, so, -1, -1, cnt));
    }
  }
  for (int i = 0; i < g.p; ++i) {
    if (i == me) continue;
    for (size_t t = 0; t < g.units_of[me].size(); ++t) {
      const Unit& u = g.units[g.units_of[me][t]];
      const long long dst0 = g.unit_q_off(me, static_cast<int>(t));
      for (int r = 0; r < g.B; ++r) {
        const int clo = g.chunk_lo(r, u.ci), chi = g.chunk_hi(r, u.ci);
        const int a = std::max(g.lo[i][r], clo), b = std::min(g.hi[i][r], chi);
        if (a >= b) continue;
        out.push_back(flat(GS_XFER_RECV, i, -1, -1, GS_BUF_RECV, dst0 + static_cast<long long>(g.qpre(r, u.ci) + a - clo) * d,
                           static_cast<long long>(b - a) * d));
      }
    }
  }
}

// head -> seq (O).  O buffer of position j: the Q receive layout (full heads [rows_full][Hf][d],
// then per local unit [qrows][d]).  Rows of position i arrive in a staging buffer (one contiguous
// slot per message) and are unpacked by 2-D copies into orecv [rows_i][D] at the head's columns.
void plan_o(const A2aGeometry& g, int me, std::vector<gs_xfer>& out, long long* stage_elems) {
  out.clear();
  const long long d = g.hd, D = static_cast<long long>(g.H) * d;
  const long long wf = static_cast<long long>(g.Hf) * d;  // full-head row width
  std::vector<gs_xfer> copies;
  auto unpack = [&](int src_buf, long long src_off, long long src_pitch, int r, int a, long long rows, long long col,
                    long long width) {
    gs_xfer x{};
    x.op = GS_XFER_COPY;
    x.peer = -1;
    x.src_buf = src_buf;
    x.src_off = src_off;
    x.dst_buf = GS_BUF_ORECV;
    x.dst_off = static_cast<long long>(g.loff[me][r] + a - g.lo[me][r]) * D + col;
    x.rows = rows;
    x.width = width;
    x.src_pitch = src_pitch;
    x.dst_pitch = D;
    copies.push_back(x);
  };
  long long stage = 0;
  // my full heads -> the rows' owners
  if (wf)
    for (int i = 0; i < g.p; ++i)
      for (int r = 0; r < g.B; ++r) {
        const long long rows = g.hi[i][r] - g.lo[i][r];
        if (!rows) continue;
        const long long so = static_cast<long long>(g.off_full[r] + g.lo[i][r]) * wf;
        if (i == me)
          unpack(GS_BUF_O, so, wf, r, g.lo[me][r], rows, static_cast<long long>(g.hoff[me]) * d, wf);
        else
          out.push_back(flat(GS_XFER_SEND, i, GS_BUF_O, so, -1, -1, rows * wf));
      }
  // my partial units: each owner gets its rows inside the unit's query chunk
  for (size_t t = 0; t < g.units_of[me].size(); ++t) {
    const Unit& u = g.units[g.units_of[me][t]];
    const long long base = g.unit_q_off(me, static_cast<int>(t));
    for (int i = 0; i < g.p; ++i)
      for (int r = 0; r < g.B; ++r) {
        const int clo = g.chunk_lo(r, u.ci), chi = g.chunk_hi(r, u.ci);
        const int a = std::max(g.lo[i][r], clo), b = std::min(g.hi[i][r], chi);
        if (a >= b) continue;
        const long long so = base + static_cast<long long>(g.qpre(r, u.ci) + a - clo) * d;
        if (i == me)
          unpack(GS_BUF_O, so, d, r, a, b - a, static_cast<long long>(u.head) * d, d);
        else
          out.push_back(flat(GS_XFER_SEND, i, GS_BUF_O, so, -1, -1, static_cast<long long>(b - a) * d));
      }
  }
  // receive my rows from the other positions: their full heads, then their units
  for (int j = 0; j < g.p; ++j) {
    if (j == me) continue;
    if (wf)
      for (int r = 0; r < g.B; ++r) {
        const long long rows = g.hi[me][r] - g.lo[me][r];
        if (!rows) continue;
        out.push_back(flat(GS_XFER_RECV, j, -1, -1, GS_BUF_STAGE, stage, rows * wf));
        unpack(GS_BUF_STAGE, stage, wf, r, g.lo[me][r], rows, static_cast<long long>(g.hoff[j]) * d, wf);
        stage += rows * wf;
      }
    for (int k : g.units_of[j]) {
      const Unit& u = g.units[k];
      for (int r = 0; r < g.B; ++r) {
        const int clo = g.chunk_lo(r, u.ci), chi = g.chunk_hi(r, u.ci);
        const int a = std::max(g.lo[me][r], clo), b = std::min(g.hi[me][r], chi);
        if (a >= b) continue;
        out.push_back(flat(GS_XFER_RECV, j, -1, -1, GS_BUF_STAGE, stage, static_cast<long long>(b - a) * d));
        unpack(GS_BUF_STAGE, stage, d, r, a, b - a, static_cast<long long>(u.head) * d, d);
        stage += static_cast<long long>(b - a) * d;
      }
    }
  }
  if (stage_elems) *stage_elems = stage;
  out.insert(out.end(), copies.begin(), copies.end());  // unpack after the exchange
}

// Re-shard of one request's latent [n, lat] from (old_ranks, old_p) to (new_ranks, new_p):
// interval intersections of old and new shards, pure copies (row a17).  Peers are global ranks.
void plan_reshard(int n, int lat, const int* old_ranks, int old_p, const int* new_ranks, int new_p, int me,
                  std::vector<gs_xfer>& out) {
  out.clear();
  for (int a = 0; a < old_p; ++a) {
    int olo, ohi;
    shard_bounds(n, old_p, a, &olo, &ohi);
    for (int b = 0; b < new_p; ++b) {
      int nlo, nhi;
      shard_bounds(n, new_p, b, &nlo, &nhi);
      const int lo = std::max(olo, nlo), hi = std::min(ohi, nhi);
      if (lo >= hi) continue;
      const long long cnt = static_cast<long long>(hi - lo) * lat;
      const long long so = static_cast<long long>(lo - olo) * lat, dof = static_cast<long long>(lo - nlo) * lat;
      const bool have_o = old_ranks[a] == me, have_n = new_ranks[b] == me;
      if (have_o && have_n)
        out.push_back(flat(GS_XFER_COPY, -1, GS_BUF_OLD, so, GS_BUF_NEW, dof, cnt));
      else if (have_o)
        out.push_back(flat(GS_XFER_SEND, new_ranks[b], GS_BUF_OLD, so, -1, -1, cnt));
      else if (have_n)
        out.push_back(flat(GS_XFER_RECV, old_ranks[a], -1, -1, GS_BUF_NEW, dof, cnt));
    }
  }
}

// Peer-store exchange (fused a2a, R == 0): no send / recv buffers or transfer lists, the
// producing kernels store straight into the consumer's buffer.
//   pack (seq -> head): local row m of request r at position `me` is full-batch row
//     m + row_delta[r] of every destination's RECV buffer ([rows_full][Hf][d], heads of chunk j);
//   attention output (head -> seq): full-batch row of token t of request r goes to the owner
//     i = max{i : own_lo[r][i] <= t}, element offset o_base[r][i] + t D + (h - hoff[me]) d of
//     the owner's ORECV buffer [rows_i][D] (o_base includes this position's column offset).
bool peer_tables(const A2aGeometry& g, int me, std::vector<long long>& row_delta, std::vector<int>& own_lo,
                 std::vector<long long>& o_base) {
  if (g.R != 0 || me < 0 || me >= g.p) return false;
  const long long D = static_cast<long long>(g.H) * g.hd;
  row_delta.assign(g.B, 0);
  own_lo.assign(static_cast<size_t>(g.B) * g.p, 0);
  o_base.assign(static_cast<size_t>(g.B) * g.p, 0);
  for (int r = 0; r < g.B; ++r) {
    row_delta[r] = static_cast<long long>(g.off_full[r]) + g.lo[me][r] - g.loff[me][r];
    for (int i = 0; i < g.p; ++i) {
      own_lo[static_cast<size_t>(r) * g.p + i] = g.lo[i][r];
      o_base[static_cast<size_t>(r) * g.p + i] =
          static_cast<long long>(g.loff[i][r] - g.lo[i][r]) * D + static_cast<long long>(g.hoff[me]) * g.hd;
    }
  }
  return true;
}

}  // namespace gs

// ------------------------------------------------------------------ C-ABI (host only)
namespace {
int copy_out(const std::vector<gs_xfer>& v, gs_xfer* out, int max_out, int* n_out) {
  if (n_out) *n_out = static_cast<int>(v.size());
  if (!out) return GS_OK;
  if (static_cast<int>(v.size()) > max_out) return GS_EINVAL;
  std::copy(v.begin(), v.end(), out);
  return GS_OK;
}
}  // namespace

extern "C" int gs_plan_a2a_usp(int kind, int p, int ring, int me, int nreq, const int* n_tokens, int heads,
                               int head_dim, gs_xfer* out, int max_out, int* n_out, long long* stage_elems) {
  if (p < 1 || p > 8 || me < 0 || me >= p || nreq < 1 || !n_tokens || heads < 1 || head_dim < 1 || ring < 1)
    return GS_EINVAL;
  for (int r = 0; r < nreq; ++r)
    if (n_tokens[r] < 0) return GS_EINVAL;
  gs::A2aGeometry g;
  g.init(p, n_tokens, nreq, heads, head_dim, ring);
  std::vector<gs_xfer> v;
  if (kind == 0 || kind == 2) {
    if (kind == 0)
      gs::plan_kv(g, me, v);
    else
      gs::plan_q(g, me, v);
    if (stage_elems) *stage_elems = 0;
  } else if (kind == 1) {
    gs::plan_o(g, me, v, stage_elems);
  } else {
    return GS_EINVAL;
  }
  return copy_out(v, out, max_out, n_out);
}

extern "C" int gs_plan_a2a(int kind, int p, int me, int nreq, const int* n_tokens, int heads, int head_dim,
                           gs_xfer* out, int max_out, int* n_out, long long* stage_elems) {
  return gs_plan_a2a_usp(kind, p, 1, me, nreq, n_tokens, heads, head_dim, out, max_out, n_out, stage_elems);
}

extern "C" int gs_plan_reshard(int n_tokens, int lat, const int* old_ranks, int old_p, const int* new_ranks,
                               int new_p, int me, gs_xfer* out, int max_out, int* n_out) {
  if (n_tokens < 0 || lat < 1 || !old_ranks || !new_ranks || old_p < 1 || new_p < 1 || old_p > 8 || new_p > 8)
    return GS_EINVAL;
  std::vector<gs_xfer> v;
  gs::plan_reshard(n_tokens, lat, old_ranks, old_p, new_ranks, new_p, me, v);
  return copy_out(v, out, max_out, n_out);
}

extern "C" int gs_plan_peer(int p, int me, int nreq, const int* n_tokens, int heads, int head_dim,
                            long long* row_delta, int* own_lo, long long* o_base) {
  if (p < 1 || p > 8 || me < 0 || me >= p || nreq < 1 || !n_tokens || heads < 1 || head_dim < 1 ||
      !row_delta || !own_lo || !o_base)
    return GS_EINVAL;
  for (int r = 0; r < nreq; ++r)
    if (n_tokens[r] < 0) return GS_EINVAL;
  gs::A2aGeometry g;
  g.init(p, n_tokens, nreq, heads, head_dim);
  std::vector<long long> rd, ob;
  std::vector<int> ol;
  if (!gs::peer_tables(g, me, rd, ol, ob)) return GS_EUNSUPPORTED;
  std::copy(rd.begin(), rd.end(), row_delta);
  std::copy(ol.begin(), ol.end(), own_lo);
  std::copy(ob.begin(), ob.end(), o_base);
  return GS_OK;
}
