// swe_inputs/meshgen.cpp -- seeded synthetic mesh generation (input side only).
//
// Holds none of the method's arithmetic: it only builds triangulations that
// both the oracle and the product path consume.  Newest-vertex bisection (NVB)
// with conforming closure of a structured "SW->NE" right-isosceles mesh, the
// graded-mesh recipe of SURVEY §8(d) C4/C5: elements whose centroid lies in
// an x-band are bisected until they reach the band's depth.  Every NVB child
// of a right isosceles triangle is right isosceles, and all coordinates stay
// dyadic multiples of the base spacing.
#include <cstdint>
#include <cstdio>
#include <unordered_map>
#include <vector>

namespace {

struct Tri {
  int a, b, c;  // a = newest vertex, refinement edge (b, c); counter-clockwise
  int gen;
  bool alive;
};

struct NVB {
  std::vector<double> vx, vy;
  std::vector<Tri> tri;
  std::unordered_map<uint64_t, int> mid;                  // edge -> midpoint vertex
  std::unordered_map<uint64_t, std::vector<int>> owners;  // edge -> alive triangles
  static uint64_t key(int p, int q) {
    if (p > q) std::swap(p, q);
    return ((uint64_t)(uint32_t)p << 32) | (uint32_t)q;
  }
  void add_edges(int t) {
    const Tri &T = tri[t];
    owners[key(T.a, T.b)].push_back(t);
    owners[key(T.b, T.c)].push_back(t);
    owners[key(T.c, T.a)].push_back(t);
  }
  void remove_edges(int t) {
    const Tri &T = tri[t];
    uint64_t ks[3] = {key(T.a, T.b), key(T.b, T.c), key(T.c, T.a)};
    for (uint64_t k : ks) {
      auto &v = owners[k];
      for (size_t i = 0; i < v.size(); i++)
        if (v[i] == t) {
          v[i] = v.back();
          v.pop_back();
          break;
        }
    }
  }
  int other_on_edge(int t, int p, int q) {
    auto it = owners.find(key(p, q));
    if (it == owners.end()) return -1;
    for (int o : it->second)
      if (o != t) return o;
    return -1;
  }
  int midpoint(int p, int q) {
    uint64_t k = key(p, q);
    auto it = mid.find(k);
    if (it != mid.end()) return it->second;
    int m = (int)vx.size();
    vx.push_back(0.5 * (vx[p] + vx[q]));
    vy.push_back(0.5 * (vy[p] + vy[q]));
    mid[k] = m;
    return m;
  }
  void bisect(int t) {
    Tri T = tri[t];
    remove_edges(t);
    tri[t].alive = false;
    int m = midpoint(T.b, T.c);
    Tri c1{m, T.a, T.b, T.gen + 1, true}, c2{m, T.c, T.a, T.gen + 1, true};
    tri.push_back(c1);
    add_edges((int)tri.size() - 1);
    tri.push_back(c2);
    add_edges((int)tri.size() - 1);
  }
  // conforming NVB refinement of triangle t (recursive closure)
  void refine(int t) {
    if (!tri[t].alive) return;
    int b = tri[t].b, c = tri[t].c;
    int n = other_on_edge(t, b, c);
    if (n >= 0) {
      const Tri &Nt = tri[n];
      bool compatible = key(Nt.b, Nt.c) == key(b, c);
      if (!compatible) {
        refine(n);
        if (!tri[t].alive) return;
        n = other_on_edge(t, b, c);
      }
    }
    bisect(t);
    if (n >= 0 && tri[n].alive) bisect(n);
  }
};

}  // namespace

extern "C" {

// Structured [x0,x1]x[y0,y1] grid of nx*ny squares split SW->NE, refined by NVB
// until every triangle whose centroid x lies in [band_lo[k], band_hi[k]) has
// generation >= band_depth[k].
void *mg_nvb(int nx, int ny, double x0, double x1, double y0, double y1, int nbands, const double *band_lo,
             const double *band_hi, const int *band_depth) {
  NVB *g = new NVB();
  double hx = (x1 - x0) / nx, hy = (y1 - y0) / ny;
  for (int j = 0; j <= ny; j++)
    for (int i = 0; i <= nx; i++) {
      g->vx.push_back(x0 + hx * i);
      g->vy.push_back(y0 + hy * j);
    }
  auto vid = [&](int i, int j) { return j * (nx + 1) + i; };
  for (int j = 0; j < ny; j++)
    for (int i = 0; i < nx; i++) {
      int v00 = vid(i, j), v10 = vid(i + 1, j), v01 = vid(i, j + 1), v11 = vid(i + 1, j + 1);
      g->tri.push_back(Tri{v10, v11, v00, 0, true});
      g->add_edges((int)g->tri.size() - 1);
      g->tri.push_back(Tri{v01, v00, v11, 0, true});
      g->add_edges((int)g->tri.size() - 1);
    }
  auto target = [&](const Tri &T) {
    double cx = (g->vx[T.a] + g->vx[T.b] + g->vx[T.c]) / 3.0;
    int d = 0;
    for (int k = 0; k < nbands; k++)
      if (cx >= band_lo[k] && cx < band_hi[k] && band_depth[k] > d) d = band_depth[k];
    return d;
  };
  bool changed = true;
  while (changed) {
    changed = false;
    size_t n = g->tri.size();
    for (size_t t = 0; t < n; t++) {
      if (!g->tri[t].alive) continue;
      if (g->tri[t].gen < target(g->tri[t])) {
        g->refine((int)t);
        changed = true;
      }
    }
  }
  return g;
}

void mg_sizes(void *h, int *nv, int *ne) {
  NVB *g = (NVB *)h;
  *nv = (int)g->vx.size();
  int k = 0;
  for (const Tri &T : g->tri) k += T.alive ? 1 : 0;
  *ne = k;
}

// etov is written counter-clockwise with the newest vertex first; gen per element
void mg_copy(void *h, double *vx, double *vy, int *etov, int *gen) {
  NVB *g = (NVB *)h;
  for (size_t i = 0; i < g->vx.size(); i++) {
    vx[i] = g->vx[i];
    vy[i] = g->vy[i];
  }
  size_t k = 0;
  for (const Tri &T : g->tri)
    if (T.alive) {
      etov[3 * k] = T.a;
      etov[3 * k + 1] = T.b;
      etov[3 * k + 2] = T.c;
      gen[k] = T.gen;
      k++;
    }
}

void mg_free(void *h) { delete (NVB *)h; }
}
