// mesh.cpp -- host mesh builder of the product path: orientation fix, face
// connectivity (P:67 conforming triangles; sort-based face matching on
// canonical vertex pairs), characteristic length Hk, static
// Cockburn-Shu TVB geometry, MRAB level binning and the
// internal element order.  Compiled with -ffp-contract=off: Hk, the wave
// speeds and the bin edges are evaluated with the exact expression order
// pinned in DESIGN.md (reading A19) so that level assignment is bit-exact
// against the oracle.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>

#include "host.hpp"

namespace swe {

int build_mesh(int nverts, const double *vx, const double *vy, int K, const int32_t *etov, const int32_t *vper,
               HostMesh &m, std::string *err) {
  m.K = K;
  m.nv = nverts;
  m.vx.assign(vx, vx + nverts);
  m.vy.assign(vy, vy + nverts);
  m.etov.assign(etov, etov + (size_t)3 * K);
  m.nflipped = 0;
  m.hk.assign(K, 0.0);
  for (int e = 0; e < K; e++) {
    int32_t *v = &m.etov[(size_t)3 * e];
    for (int k = 0; k < 3; k++)
      if (v[k] < 0 || v[k] >= nverts) {
        if (err) *err = "element " + std::to_string(e) + ": vertex index out of range";
        return -2;
      }
    if (v[0] == v[1] || v[1] == v[2] || v[2] == v[0]) {
      if (err) *err = "element " + std::to_string(e) + ": repeated vertex";
      return -2;
    }
    double x1 = vx[v[0]], x2 = vx[v[1]], x3 = vx[v[2]], y1 = vy[v[0]], y2 = vy[v[1]], y3 = vy[v[2]];
    double A = 0.5 * ((x2 - x1) * (y3 - y1) - (x3 - x1) * (y2 - y1));
    if (A == 0.0 || !std::isfinite(A)) {
      if (err) *err = "element " + std::to_string(e) + ": zero area";
      return -2;
    }
    if (A < 0.0) {
      std::swap(v[1], v[2]);
      m.nflipped++;
      A = -A;
    }
    // recompute on the oriented triangle exactly as pinned: A, then Hk = 4A / ((l0 + l1) + l2)
    x1 = vx[v[0]];
    x2 = vx[v[1]];
    x3 = vx[v[2]];
    y1 = vy[v[0]];
    y2 = vy[v[1]];
    y3 = vy[v[2]];
    A = 0.5 * ((x2 - x1) * (y3 - y1) - (x3 - x1) * (y2 - y1));
    double X[3] = {x1, x2, x3}, Y[3] = {y1, y2, y3}, len[3];
    for (int f = 0; f < 3; f++) {
      double dx = X[(f + 1) % 3] - X[f], dy = Y[(f + 1) % 3] - Y[f];
      len[f] = std::sqrt(dx * dx + dy * dy);
    }
    m.hk[e] = (4.0 * A) / ((len[0] + len[1]) + len[2]);
  }

  // face matching: sort (key, slot) pairs
  struct FaceKey {
    uint64_t key;
    int32_t e;
    int8_t f;
  };
  std::vector<FaceKey> faces((size_t)3 * K);
  for (int e = 0; e < K; e++)
    for (int f = 0; f < 3; f++) {
      uint32_t a = (uint32_t)m.etov[(size_t)3 * e + f], b = (uint32_t)m.etov[(size_t)3 * e + (f + 1) % 3];
      if (vper) {
        a = (uint32_t)vper[a];
        b = (uint32_t)vper[b];
      }
      if (a > b) std::swap(a, b);
      faces[(size_t)3 * e + f] = FaceKey{((uint64_t)a << 32) | b, e, (int8_t)f};
    }
  std::sort(faces.begin(), faces.end(), [](const FaceKey &p, const FaceKey &q) {
    if (p.key != q.key) return p.key < q.key;
    if (p.e != q.e) return p.e < q.e;
    return p.f < q.f;
  });
  m.etoe.assign((size_t)3 * K, 0);
  m.etof.assign((size_t)3 * K, 0);
  for (int e = 0; e < K; e++)
    for (int f = 0; f < 3; f++) {
      m.etoe[(size_t)3 * e + f] = e;
      m.etof[(size_t)3 * e + f] = (int8_t)f;
    }
  size_t i = 0;
  while (i < faces.size()) {
    size_t j = i + 1;
    while (j < faces.size() && faces[j].key == faces[i].key) j++;
    if (j - i > 2) {
      if (err) *err = "face shared by more than two elements";
      return -2;
    }
    if (j - i == 2) {
      const FaceKey &p = faces[i], &q = faces[i + 1];
      m.etoe[(size_t)3 * p.e + p.f] = q.e;
      m.etof[(size_t)3 * p.e + p.f] = q.f;
      m.etoe[(size_t)3 * q.e + q.f] = p.e;
      m.etof[(size_t)3 * q.e + q.f] = p.f;
    }
    i = j;
  }
  return 0;
}

// Cockburn & Shu (1998) neighbour pairs: for edge i (midpoint m_i, own
// barycentre b0) try the neighbour pairs (i, i+1) then (i, i+2); the first
// with both alphas >= -1e-12 wins, otherwise the pair whose smaller alpha is
// larger; alphas are clamped at 0.  Wall ghost barycentre: b0 mirrored in the
// edge line.  Periodic neighbour: translated by (own - neighbour) face midpoint.
void build_tvb_geometry(const HostMesh &m, TvbGeom &t) {
  const int K = m.K;
  t.pj.assign((size_t)3 * K, 0);
  t.pk.assign((size_t)3 * K, 0);
  t.aj.assign((size_t)3 * K, 0.0);
  t.ak.assign((size_t)3 * K, 0.0);
  auto vtx = [&](int e, int k, double &x, double &y) {
    int v = m.etov[(size_t)3 * e + k];
    x = m.vx[v];
    y = m.vy[v];
  };
  auto bary = [&](int e, double &x, double &y) {
    double x0, y0, x1, y1, x2, y2;
    vtx(e, 0, x0, y0);
    vtx(e, 1, x1, y1);
    vtx(e, 2, x2, y2);
    x = (x0 + x1 + x2) / 3.0;
    y = (y0 + y1 + y2) / 3.0;
  };
  auto mid = [&](int e, int f, double &x, double &y) {
    double xa, ya, xb, yb;
    vtx(e, f, xa, ya);
    vtx(e, (f + 1) % 3, xb, yb);
    x = 0.5 * (xa + xb);
    y = 0.5 * (ya + yb);
  };
  for (int e = 0; e < K; e++) {
    double bx, by;
    bary(e, bx, by);
    double nbx[3], nby[3];
    for (int f = 0; f < 3; f++) {
      int n = m.etoe[(size_t)3 * e + f], nf = m.etof[(size_t)3 * e + f];
      double mx, my;
      mid(e, f, mx, my);
      if (n == e && nf == f) {
        double xa, ya, xb, yb;
        vtx(e, f, xa, ya);
        vtx(e, (f + 1) % 3, xb, yb);
        double dx = xb - xa, dy = yb - ya, len = std::sqrt(dx * dx + dy * dy);
        double nx = dy / len, ny = -dx / len;
        double d = (bx - mx) * nx + (by - my) * ny;
        nbx[f] = bx - 2.0 * d * nx;
        nby[f] = by - 2.0 * d * ny;
      } else {
        double cx, cy, qx, qy;
        bary(n, cx, cy);
        mid(n, nf, qx, qy);
        nbx[f] = cx + (mx - qx);
        nby[f] = cy + (my - qy);
      }
    }
    for (int i = 0; i < 3; i++) {
      double mx, my;
      mid(e, i, mx, my);
      double tx = mx - bx, ty = my - by;
      int cand[2][2] = {{i, (i + 1) % 3}, {i, (i + 2) % 3}};
      double al[2][2];
      int pick = -1;
      for (int p = 0; p < 2; p++) {
        int j = cand[p][0], k = cand[p][1];
        double ux = nbx[j] - bx, uy = nby[j] - by, wx = nbx[k] - bx, wy = nby[k] - by;
        double det = ux * wy - uy * wx;
        if (det == 0.0) {
          al[p][0] = al[p][1] = -std::numeric_limits<double>::infinity();
          continue;
        }
        al[p][0] = (tx * wy - ty * wx) / det;
        al[p][1] = (ux * ty - uy * tx) / det;
        if (pick < 0 && al[p][0] >= -1e-12 && al[p][1] >= -1e-12) pick = p;
      }
      if (pick < 0) {
        double m0 = std::min(al[0][0], al[0][1]), m1 = std::min(al[1][0], al[1][1]);
        pick = (m1 > m0) ? 1 : 0;
      }
      size_t s = (size_t)3 * e + i;
      t.pj[s] = (int8_t)cand[pick][0];
      t.pk[s] = (int8_t)cand[pick][1];
      t.aj[s] = std::max(0.0, al[pick][0]);
      t.ak[s] = std::max(0.0, al[pick][1]);
    }
  }
}

// Desingularised velocity (reading A4), pinned expression:
//   u = (sqrt2 * h+ * m) / sqrt(h+^4 + max(h+^4, eps_u^4)),  h+^4 = (h+ h+)(h+ h+).
double desing_velocity(double h, double m, double e4) {
  double hp = h > 0.0 ? h : 0.0;
  double h2 = hp * hp, h4 = h2 * h2;
  return (std::sqrt(2.0) * hp * m) / std::sqrt(h4 + (h4 > e4 ? h4 : e4));
}

void element_speeds(int K, int Np, double g, double eps_u, double a_floor, const double *h, const double *hu,
                    const double *hv, double *ae) {
  double e2 = eps_u * eps_u, e4 = e2 * e2;
  for (int e = 0; e < K; e++) {
    double amax = 0.0;
    for (int i = 0; i < Np; i++) {
      size_t k = (size_t)e * Np + i;
      double u = desing_velocity(h[k], hu[k], e4), v = desing_velocity(h[k], hv[k], e4);
      double hp = h[k] > 0.0 ? h[k] : 0.0;
      double a = std::sqrt(u * u + v * v) + std::sqrt(g * hp);
      amax = a > amax ? a : amax;
    }
    ae[e] = a_floor > amax ? a_floor : amax;
  }
}

void bin_levels(int K, const double *hk, const double *ae, int L, int32_t *level) {
  const double inf = std::numeric_limits<double>::infinity();
  double rmin = inf;
  for (int e = 0; e < K; e++) {
    double r = ae[e] > 0.0 ? hk[e] / ae[e] : inf;
    if (r < rmin) rmin = r;
  }
  bin_levels_rmin(K, hk, ae, L, rmin, level);
}

void bin_levels_rmin(int K, const double *hk, const double *ae, int L, double rmin, int32_t *level) {
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<double> r(K);
  for (int e = 0; e < K; e++) r[e] = ae[e] > 0.0 ? hk[e] / ae[e] : inf;
  for (int e = 0; e < K; e++) {
    int l = 1;
    for (int k = 1; k < L; k++)
      if (r[e] >= std::ldexp(rmin, k)) l = k + 1;
    level[e] = l;
  }
}

// 2D Morton: spread the low 21 bits of v to the even bit positions (42-bit key).
static uint64_t spread_bits(uint32_t v) {
  uint64_t x = v & 0x1fffff;
  x = (x | (x << 16)) & 0x0000ffff0000ffffULL;
  x = (x | (x << 8)) & 0x00ff00ff00ff00ffULL;
  x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0fULL;
  x = (x | (x << 2)) & 0x3333333333333333ULL;
  x = (x | (x << 1)) & 0x5555555555555555ULL;
  return x;
}

void element_order(const HostMesh &m, const int32_t *level, std::vector<int32_t> &order) {
  const int K = m.K;
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  for (int v = 0; v < m.nv; v++) {
    xmin = std::min(xmin, m.vx[v]);
    xmax = std::max(xmax, m.vx[v]);
    ymin = std::min(ymin, m.vy[v]);
    ymax = std::max(ymax, m.vy[v]);
  }
  double sx = (xmax > xmin) ? ((1 << 21) - 1) / (xmax - xmin) : 0.0;
  double sy = (ymax > ymin) ? ((1 << 21) - 1) / (ymax - ymin) : 0.0;
  std::vector<std::pair<uint64_t, int32_t>> keys(K);
  for (int e = 0; e < K; e++) {
    const int32_t *v = &m.etov[(size_t)3 * e];
    double bx = (m.vx[v[0]] + m.vx[v[1]] + m.vx[v[2]]) / 3.0, by = (m.vy[v[0]] + m.vy[v[1]] + m.vy[v[2]]) / 3.0;
    uint32_t ix = (uint32_t)((bx - xmin) * sx), iy = (uint32_t)((by - ymin) * sy);
    uint64_t morton = spread_bits(ix) | (spread_bits(iy) << 1);
    uint64_t lev = level ? (uint64_t)(level[e] - 1) : 0;
    keys[e] = {(lev << 48) | morton, e};  // level field above the 42 Morton bits
  }
  std::sort(keys.begin(), keys.end());
  order.resize(K);
  for (int k = 0; k < K; k++) order[k] = keys[k].second;
}

}  // namespace swe

namespace swe {

void build_halo_plan(const HostMesh &m, const int64_t *gid, const int32_t *owner, int rank, HaloPlan &plan) {
  const int K = m.K;
  plan = HaloPlan();
  std::vector<char> is_ghost(K, 0);
  std::vector<std::vector<int32_t>> send_by_rank;
  std::vector<int32_t> peer_slot;
  auto slot_of = [&](int q) {
    for (size_t i = 0; i < plan.peers.size(); i++)
      if (plan.peers[i] == q) return (int)i;
    plan.peers.push_back(q);
    plan.send.push_back({});
    plan.recv.push_back({});
    return (int)plan.peers.size() - 1;
  };
  for (int e = 0; e < K; e++) {
    if (owner[e] != rank) continue;
    plan.owned.push_back(e);
    std::vector<int> sent_to;
    for (int f = 0; f < 3; f++) {
      int n = m.etoe[(size_t)3 * e + f];
      if (n == e || owner[n] == rank) continue;
      if (!is_ghost[n]) {
        is_ghost[n] = 1;
        plan.ghosts.push_back(n);
      }
      int q = owner[n];
      if (std::find(sent_to.begin(), sent_to.end(), q) == sent_to.end()) {
        sent_to.push_back(q);
        plan.send[slot_of(q)].push_back(e);
      }
    }
  }
  for (int g : plan.ghosts) plan.recv[slot_of(owner[g])].push_back(g);
  // peers ascending, lists by global id
  std::vector<size_t> ord(plan.peers.size());
  for (size_t i = 0; i < ord.size(); i++) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return plan.peers[a] < plan.peers[b]; });
  HaloPlan sorted = plan;
  for (size_t i = 0; i < ord.size(); i++) {
    sorted.peers[i] = plan.peers[ord[i]];
    sorted.send[i] = plan.send[ord[i]];
    sorted.recv[i] = plan.recv[ord[i]];
  }
  plan = sorted;
  auto by_gid = [&](int32_t a, int32_t b) { return gid[a] < gid[b]; };
  for (auto &v : plan.send) std::sort(v.begin(), v.end(), by_gid);
  for (auto &v : plan.recv) std::sort(v.begin(), v.end(), by_gid);
  std::sort(plan.ghosts.begin(), plan.ghosts.end(), by_gid);
}

void apply_boundary_tags(HostMesh &m, const int8_t *vbc) {
  m.bc.assign((size_t)3 * m.K, 0);
  if (!vbc) return;
  for (int e = 0; e < m.K; e++)
    for (int f = 0; f < 3; f++) {
      const size_t i = (size_t)3 * e + f;
      if (m.etoe[i] != e || m.etof[i] != f) continue;  // interior face
      const int a = m.etov[(size_t)3 * e + f], b = m.etov[(size_t)3 * e + (f + 1) % 3];
      // both vertices tagged: the face takes the smaller tag (1 outflow, 2 Dirichlet); otherwise a wall
      m.bc[i] = (vbc[a] >= 1 && vbc[b] >= 1) ? (int8_t)std::min(std::min((int)vbc[a], (int)vbc[b]), 2) : 0;
    }
}

}  // namespace swe
