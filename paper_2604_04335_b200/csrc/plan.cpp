// Host-only exchange planning for the SP path (no CUDA): the Ulysses all-to-alls of one DiT
// block and the latent re-shard at resume (row a17) expressed as
// lists of transfers (send / recv / local 2-D copy) per SP position.  The same plans drive the
// NCCL executor, the emulated executor and the CPU gloo tests (tests/test_plan_gloo.py).
//
// Partitioning readings: token shard i of p is [floor(i n / p), floor((i+1) n / p))
// (reading 10); heads split contiguously, positions < H mod p get ceil(H / p) (reading 9).
#include "plan.h"

#include <algorithm>

namespace gs {

void shard_bounds(int n, int p, int i, int* lo, int* hi) {
  *lo = static_cast<int>((static_cast<long long>(i) * n) / p);
  *hi = static_cast<int>((static_cast<long long>(i + 1) * n) / p);
}

int head_offset(int H, int p, int j) { return j * (H / p) + std::min(j, H % p); }

void A2aGeometry::init(int p_, const int* n_tokens, int nreq, int heads_, int hd_) {
  p = p_;
  B = nreq;
  H = heads_;
  hd = hd_;
  n.assign(n_tokens, n_tokens + nreq);
  hoff.resize(p + 1);
  for (int j = 0; j <= p; ++j) hoff[j] = head_offset(H, p, j);
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

// seq -> head (Q, K, V; the plan applies to each of the three buffers).
// send buffer of position i: [dest j][rows_i][H_j][d]; recv buffer of j: [rows_full][H_j][d].
void plan_qkv(const A2aGeometry& g, int me, std::vector<gs_xfer>& out) {
  out.clear();
  const long long d = g.hd;
  const long long Hm = g.H_loc(me);
  for (int j = 0; j < g.p; ++j) {  // my rows, heads of j -> j
    const long long Hj = g.H_loc(j);
    const long long chunk = static_cast<long long>(g.rows[me]) * g.hoff[j] * d;
    for (int r = 0; r < g.B; ++r) {
      const long long cnt = static_cast<long long>(g.hi[me][r] - g.lo[me][r]) * Hj * d;
      if (!cnt) continue;
      const long long so = chunk + static_cast<long long>(g.loff[me][r]) * Hj * d;
      if (j == me)
        out.push_back(flat(GS_XFER_COPY, -1, GS_BUF_SEND, so, GS_BUF_RECV,
                           static_cast<long long>(g.off_full[r] + g.lo[me][r]) * Hm * d, cnt));
      else
        out.push_back(flat(GS_XFER_SEND, j, GS_BUF_SEND, so, -1, -1, cnt));
    }
  }
  for (int i = 0; i < g.p; ++i) {  // rows of i, my heads <- i
    if (i == me) continue;
    for (int r = 0; r < g.B; ++r) {
      const long long cnt = static_cast<long long>(g.hi[i][r] - g.lo[i][r]) * Hm * d;
      if (!cnt) continue;
      out.push_back(flat(GS_XFER_RECV, i, -1, -1, GS_BUF_RECV,
                         static_cast<long long>(g.off_full[r] + g.lo[i][r]) * Hm * d, cnt));
    }
  }
}

// head -> seq (O).  O buffer of position j: [rows_full][H_j][d] (attention output); the rows of
// position i arrive in a staging buffer [src j][req r][rows][H_j d] and are unpacked by 2-D copies
// into orecv [rows_i][D] at column H offset hoff[j] * d.
void plan_o(const A2aGeometry& g, int me, std::vector<gs_xfer>& out, long long* stage_elems) {
  out.clear();
  const long long d = g.hd, D = static_cast<long long>(g.H) * d;
  const long long wm = g.H_loc(me) * d;
  for (int i = 0; i < g.p; ++i) {
    if (i == me) continue;
    for (int r = 0; r < g.B; ++r) {
      const long long cnt = static_cast<long long>(g.hi[i][r] - g.lo[i][r]) * wm;
      if (!cnt) continue;
      out.push_back(flat(GS_XFER_SEND, i, GS_BUF_O, static_cast<long long>(g.off_full[r] + g.lo[i][r]) * wm, -1, -1,
                         cnt));
    }
  }
  long long acc = 0;
  std::vector<long long> stage_off(static_cast<size_t>(g.p) * g.B, 0);
  for (int j = 0; j < g.p; ++j)
    for (int r = 0; r < g.B; ++r) {
      stage_off[static_cast<size_t>(j) * g.B + r] = acc;
      if (j != me) acc += static_cast<long long>(g.hi[me][r] - g.lo[me][r]) * g.H_loc(j) * d;
    }
  if (stage_elems) *stage_elems = acc;
  for (int j = 0; j < g.p; ++j) {
    if (j == me) continue;
    const long long wj = g.H_loc(j) * d;
    for (int r = 0; r < g.B; ++r) {
      const long long cnt = static_cast<long long>(g.hi[me][r] - g.lo[me][r]) * wj;
      if (!cnt) continue;
      out.push_back(flat(GS_XFER_RECV, j, -1, -1, GS_BUF_STAGE, stage_off[static_cast<size_t>(j) * g.B + r], cnt));
    }
  }
  for (int j = 0; j < g.p; ++j) {  // unpack (after the exchange completes)
    const long long wj = g.H_loc(j) * d;
    for (int r = 0; r < g.B; ++r) {
      const long long rows = g.hi[me][r] - g.lo[me][r];
      if (!rows || !wj) continue;
      gs_xfer x{};
      x.op = GS_XFER_COPY;
      x.peer = -1;
      if (j == me) {
        x.src_buf = GS_BUF_O;
        x.src_off = static_cast<long long>(g.off_full[r] + g.lo[me][r]) * wm;
      } else {
        x.src_buf = GS_BUF_STAGE;
        x.src_off = stage_off[static_cast<size_t>(j) * g.B + r];
      }
      x.dst_buf = GS_BUF_ORECV;
      x.dst_off = static_cast<long long>(g.loff[me][r]) * D + static_cast<long long>(g.hoff[j]) * d;
      x.rows = rows;
      x.width = wj;
      x.src_pitch = wj;
      x.dst_pitch = D;
      out.push_back(x);
    }
  }
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

extern "C" int gs_plan_a2a(int kind, int p, int me, int nreq, const int* n_tokens, int heads, int head_dim,
                           gs_xfer* out, int max_out, int* n_out, long long* stage_elems) {
  if (p < 1 || p > 8 || me < 0 || me >= p || nreq < 1 || !n_tokens || heads < 1 || head_dim < 1)
    return GS_EINVAL;
  for (int r = 0; r < nreq; ++r)
    if (n_tokens[r] < 0) return GS_EINVAL;
  gs::A2aGeometry g;
  g.init(p, n_tokens, nreq, heads, head_dim);
  std::vector<gs_xfer> v;
  if (kind == 0) {
    gs::plan_qkv(g, me, v);
    if (stage_elems) *stage_elems = 0;
  } else if (kind == 1) {
    gs::plan_o(g, me, v, stage_elems);
  } else {
    return GS_EINVAL;
  }
  return copy_out(v, out, max_out, n_out);
}

extern "C" int gs_plan_reshard(int n_tokens, int lat, const int* old_ranks, int old_p, const int* new_ranks,
                               int new_p, int me, gs_xfer* out, int max_out, int* n_out) {
  if (n_tokens < 0 || lat < 1 || !old_ranks || !new_ranks || old_p < 1 || new_p < 1 || old_p > 8 || new_p > 8)
    return GS_EINVAL;
  std::vector<gs_xfer> v;
  gs::plan_reshard(n_tokens, lat, old_ranks, old_p, new_ranks, new_p, me, v);
  return copy_out(v, out, max_out, n_out);
}
