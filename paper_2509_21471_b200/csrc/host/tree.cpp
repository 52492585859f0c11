#include "tree.hpp"

#include <cmath>
#include <cstdio>
#include <sstream>

namespace sdmkb {

namespace {

constexpr int64_t kCells = int64_t(1) << kMaxLevel;

struct Points {
  int n = 0;
  const int32_t* q = nullptr;  // SoA
  int child(int i, int level, int dim) const {  // tree.cpp:38-43
    int ci = 0;
    for (int a = 0; a < dim; ++a) ci |= ((q[size_t(a) * n + i] >> (kMaxLevel - 1 - level)) & 1) << a;
    return ci;
  }
};

struct Builder {
  HostTree t;
  Points S, T;
  int nchild = 8;

  // child boundaries of [lo, hi) by binary search on the (monotone) child index
  void split_range(const Points& P, int lo, int hi, int level, int* bnd) const {
    bnd[0] = lo;
    for (int ci = 1; ci < nchild; ++ci) {
      int a = bnd[ci - 1], b = hi;
      while (a < b) {
        int m = a + (b - a) / 2;
        if (P.child(m, level, t.dim) < ci) a = m + 1; else b = m;
      }
      bnd[ci] = a;
    }
    bnd[nchild] = hi;
  }

  void subdivide(int b) {  // tree.cpp:62-99
    int lev = t.boxes[b].level;
    int32_t half = int32_t(1) << (kMaxLevel - 1 - lev);
    int fc = t.num_boxes();
    t.boxes[b].leaf = false;
    t.boxes[b].first_child = fc;
    if (lev + 1 > t.max_level) t.max_level = lev + 1;
    int sb[9], tb[9];
    split_range(S, t.boxes[b].sb, t.boxes[b].se, lev, sb);
    if (t.alias)
      for (int i = 0; i <= nchild; ++i) tb[i] = sb[i];
    else
      split_range(T, t.boxes[b].tb, t.boxes[b].te, lev, tb);
    Box par = t.boxes[b];
    for (int ci = 0; ci < nchild; ++ci) {
      Box c;
      c.level = lev + 1;
      c.parent = b;
      for (int a = 0; a < t.dim; ++a) c.anchor[a] = par.anchor[a] + ((ci >> a) & 1) * half;
      c.sb = sb[ci];
      c.se = sb[ci + 1];
      c.tb = tb[ci];
      c.te = tb[ci + 1];
      t.boxes.push_back(c);
    }
  }

  int descend(const int32_t* probe) const {  // tree.cpp:102-107
    int b = 0;
    while (!t.boxes[b].leaf) {
      int lev = t.boxes[b].level, ci = 0;
      for (int a = 0; a < t.dim; ++a) ci |= ((probe[a] >> (kMaxLevel - 1 - lev)) & 1) << a;
      b = t.boxes[b].first_child + ci;
    }
    return b;
  }

  void refine() {  // tree.cpp:109-123 (DFS pre-order allocation)
    std::vector<int> stack(1, 0);
    while (!stack.empty()) {
      int b = stack.back();
      stack.pop_back();
      if (t.nsrc(b) <= t.n_s) continue;
      if (t.boxes[b].level >= kMaxLevel) {
        t.depth_capped = true;
        continue;
      }
      subdivide(b);
      for (int ci = nchild - 1; ci >= 0; --ci) stack.push_back(t.boxes[b].first_child + ci);
    }
  }

  void repair() {  // tree.cpp:125-165 (sweeps until no leaf is 2 levels coarser than a neighbour)
    for (bool again = true; again;) {
      again = false;
      std::vector<int> leaves;
      for (int b = 0; b < t.num_boxes(); ++b)
        if (t.boxes[b].leaf) leaves.push_back(b);
      for (int b : leaves) {
        if (!t.boxes[b].leaf) continue;
        int lev = t.boxes[b].level;
        if (lev < 2) continue;
        int64_t side = kCells >> lev;
        int zr = t.dim == 3 ? 1 : 0;
        for (int o2 = -zr; o2 <= zr; ++o2)
          for (int o1 = -1; o1 <= 1; ++o1)
            for (int o0 = -1; o0 <= 1; ++o0) {
              if (!o0 && !o1 && !o2) continue;
              int off[3] = {o0, o1, o2};
              int32_t probe[3] = {0, 0, 0};
              bool inside = true;
              for (int a = 0; a < t.dim && inside; ++a) {
                int64_t v = t.boxes[b].anchor[a] + off[a] * side + side / 2;
                if (t.periodic)
                  v = ((v % kCells) + kCells) % kCells;
                else if (v < 0 || v >= kCells)
                  inside = false;
                probe[a] = int32_t(v);
              }
              if (!inside) continue;
              int a = descend(probe);
              if (t.boxes[a].leaf && t.boxes[a].level <= lev - 2) {
                subdivide(a);
                again = true;
              }
            }
      }
    }
  }

  bool touch(int b, int c, const int8_t* sh) const {  // tree.cpp:46-56
    int64_t sbz = kCells >> t.boxes[b].level, scz = kCells >> t.boxes[c].level;
    for (int a = 0; a < t.dim; ++a) {
      int64_t l1 = t.boxes[b].anchor[a], l2 = t.boxes[c].anchor[a] + sh[a] * kCells;
      if (l1 > l2 + scz || l2 > l1 + sbz) return false;
    }
    return true;
  }

  void neighbours() {  // tree.cpp:167-212
    int nb = t.num_boxes();
    t.col.assign(nb, {});
    t.crs.assign(nb, {});
    t.fin.assign(nb, {});
    t.level_boxes.assign(t.max_level + 1, {});
    for (int b = 0; b < nb; ++b) t.level_boxes[t.boxes[b].level].push_back(b);
    if (t.periodic) {
      int zr = t.dim == 3 ? 1 : 0;
      for (int s2 = -zr; s2 <= zr; ++s2)
        for (int s1 = -1; s1 <= 1; ++s1)
          for (int s0 = -1; s0 <= 1; ++s0) t.col[0].push_back({0, {int8_t(s0), int8_t(s1), int8_t(s2)}});
    } else {
      t.col[0].push_back({0, {0, 0, 0}});
    }
    for (int lev = 1; lev <= t.max_level; ++lev)
      for (int b : t.level_boxes[lev]) {
        int par = t.boxes[b].parent;
        for (const Nbr& pc : t.col[par]) {
          if (t.boxes[pc.box].leaf) {
            if (touch(b, pc.box, pc.shift)) t.crs[b].push_back(pc);
            continue;
          }
          for (int ci = 0; ci < nchild; ++ci) {
            int d = t.boxes[pc.box].first_child + ci;
            if (touch(b, d, pc.shift)) t.col[b].push_back({d, {pc.shift[0], pc.shift[1], pc.shift[2]}});
          }
        }
      }
    for (int b = 0; b < nb; ++b)
      for (const Nbr& ce : t.col[b]) {
        if (ce.box == b && !ce.shift[0] && !ce.shift[1] && !ce.shift[2]) continue;
        if (t.boxes[ce.box].leaf) continue;
        for (int ci = 0; ci < nchild; ++ci) {
          int d = t.boxes[ce.box].first_child + ci;
          if (t.boxes[d].leaf && touch(b, d, ce.shift)) t.fin[b].push_back({d, {ce.shift[0], ce.shift[1], ce.shift[2]}});
        }
      }
  }
};

}  // namespace

double HostTree::side(int b) const { return std::ldexp(1.0, -boxes[b].level); }

std::array<double, 3> HostTree::center(int b) const {  // tree.cpp:221-228
  std::array<double, 3> c = {0.0, 0.0, 0.0};
  double s = side(b);
  for (int a = 0; a < dim; ++a) c[a] = std::ldexp(double(boxes[b].anchor[a]), -kMaxLevel) - 0.5 + 0.5 * s;
  return c;
}

HostTree build_topology(int dim, bool periodic, int n_s, int p, int ns, const int32_t* qs, int nt,
                        const int32_t* qt) {
  Builder B;
  B.t.dim = dim;
  B.t.periodic = periodic;
  B.t.n_s = n_s;
  B.t.p = p;
  B.t.alias = nt == 0;
  B.nchild = 1 << dim;
  B.S.n = ns;
  B.S.q = qs;
  B.T.n = nt;
  B.T.q = qt;
  Box root;
  root.se = ns;
  root.te = B.t.alias ? ns : nt;
  B.t.boxes.push_back(root);
  B.refine();
  B.repair();
  B.neighbours();
  if (B.t.depth_capped)
    std::fprintf(stderr, "build_tree: depth cap %d reached with leaves above capacity (duplicate points?)\n",
                 kMaxLevel);
  return std::move(B.t);
}

std::string dump_topology(const HostTree& t) {  // tree.cpp:325-354
  std::ostringstream os;
  auto lst = [&](const char* tag, const std::vector<Nbr>& v) {
    os << ' ' << tag << "={";
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) os << ' ';
      os << v[i].box;
      if (v[i].shift[0] || v[i].shift[1] || v[i].shift[2])
        os << '@' << int(v[i].shift[0]) << ',' << int(v[i].shift[1]) << ',' << int(v[i].shift[2]);
    }
    os << '}';
  };
  os << "tree dim=" << t.dim << " periodic=" << int(t.periodic) << " n_s=" << t.n_s << " p=" << t.p
     << " boxes=" << t.num_boxes() << " max_level=" << t.max_level << '\n';
  for (int b = 0; b < t.num_boxes(); ++b) {
    const Box& x = t.boxes[b];
    os << b << " L" << x.level << " a=" << x.anchor[0] << ',' << x.anchor[1];
    if (t.dim == 3) os << ',' << x.anchor[2];
    os << (x.leaf ? " leaf" : " node") << " src=[" << x.sb << ',' << x.se << ") tgt=[" << x.tb << ',' << x.te
       << ")";
    lst("col", t.col[b]);
    lst("crs", t.crs[b]);
    lst("fin", t.fin[b]);
    os << '\n';
  }
  return os.str();
}

}  // namespace sdmkb
