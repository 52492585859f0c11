#include "tree.hpp"
#include "setup.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>

#ifdef _OPENMP
#include <omp.h>
#endif

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
  const PointAccess* pa = nullptr;  // device-resident points (null: S / T are host arrays)

  void need_host_points() {  // the repair subdivides on the host
    if (S.q || !pa) return;
    const int32_t *qs = nullptr, *qt = nullptr;
    pa->host_q(&qs, &qt);
    S.q = qs;
    T.q = qt;
  }

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

  // children of box `par` (ranges from the bnd arrays), appended at ids fc..fc+2^d-1
  void make_children(int b, const int* sb, const int* tb) {  // tree.cpp:62-99
    const int lev = t.boxes[b].level;
    const int32_t half = int32_t(1) << (kMaxLevel - 1 - lev);
    t.boxes[b].leaf = false;
    t.boxes[b].first_child = t.num_boxes();
    if (lev + 1 > t.max_level) t.max_level = lev + 1;
    const Box par = t.boxes[b];
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

  // repair subdivisions on device-resident points: the 2:1 sweeps depend only
  // on the box structure (leaf flags, levels, anchors), never on point ranges,
  // so the children's ranges are found afterwards, one batched GPU call per level
  std::vector<int> deferred;
  size_t deferred_total = 0;
  bool dev_boxes = false;  // the device holds these boxes (pa->refine ran): the repair's first sweep runs there
  double split_ms = 0.0, dfs_ms = 0.0;  // time in the GPU split calls / DFS renumbering (SDMK_TIMING)
  double rep_scan_ms = 0.0;             // repair: parallel pre-scan
  int rep_leaves = 0, rep_sweeps = 0, rep_cands = 0;

  void subdivide(int b) {
    if (pa && !S.q) {
      int z[9];
      for (int i = 0; i <= nchild; ++i) z[i] = t.boxes[b].sb;  // placeholder ranges
      int zt[9];
      for (int i = 0; i <= nchild; ++i) zt[i] = t.boxes[b].tb;
      make_children(b, z, zt);
      deferred.push_back(b);
      ++deferred_total;
      return;
    }
    need_host_points();
    int sb[9], tb[9];
    split_range(S, t.boxes[b].sb, t.boxes[b].se, t.boxes[b].level, sb);
    if (t.alias)
      for (int i = 0; i <= nchild; ++i) tb[i] = sb[i];
    else
      split_range(T, t.boxes[b].tb, t.boxes[b].te, t.boxes[b].level, tb);
    make_children(b, sb, tb);
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

  // refine_to_capacity (tree.cpp:109-123).  The set of subdivided boxes
  // depends only on counts; build it breadth first with parallel searches,
  // then allocate ids in the reference's DFS pre-order.
  void refine() {
    if (pa && pa->refine) {
      int maxlev = 0;
      bool capped = false;
      if (pa->refine(t.boxes, maxlev, capped)) {
        t.max_level = maxlev;
        t.depth_capped = capped;
        dev_boxes = true;
        return;
      }
    }
    struct Node {
      Box box;
      int kids = -1;  // index of first child in `nodes` (BFS order)
      int sb[9], tb[9];
    };
    std::vector<Node> nodes(1);
    nodes.reserve(std::min<size_t>(size_t(1) << 24, 4 * (size_t)(S.n + T.n) / std::max(1, t.n_s) * (size_t)nchild + 64));
    nodes[0].box = t.boxes[0];
    std::vector<int> cur(1, 0);
    bool capped = false;
    while (!cur.empty()) {
      const int nc = (int)cur.size();
      std::vector<char> split(nc, 0);
      if (pa) {  // one batched call per level for the boxes that split
        std::vector<int> which, lvl, sr, tr;
        for (int i = 0; i < nc; ++i) {
          const Node& nd = nodes[cur[i]];
          if (nd.box.se - nd.box.sb <= t.n_s) continue;
          if (nd.box.level >= kMaxLevel) {
            capped = true;
            continue;
          }
          split[i] = 1;
          which.push_back(i);
          lvl.push_back(nd.box.level);
          sr.push_back(nd.box.sb);
          sr.push_back(nd.box.se);
          tr.push_back(nd.box.tb);
          tr.push_back(nd.box.te);
        }
        const int nw = (int)which.size();
        std::vector<int> sbv((size_t)nw * 9), tbv((size_t)nw * 9);
        const auto ts0 = std::chrono::steady_clock::now();
        if (nw) pa->split(nw, lvl.data(), sr.data(), tr.data(), sbv.data(), tbv.data());
        split_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts0).count();
        for (int k = 0; k < nw; ++k) {
          Node& nd = nodes[cur[which[k]]];
          for (int c = 0; c <= nchild; ++c) {
            nd.sb[c] = sbv[(size_t)k * 9 + c];
            nd.tb[c] = t.alias ? nd.sb[c] : tbv[(size_t)k * 9 + c];
          }
        }
      } else {
#pragma omp parallel for schedule(dynamic, 16) reduction(|| : capped)
        for (int i = 0; i < nc; ++i) {
          Node& nd = nodes[cur[i]];
          if (nd.box.se - nd.box.sb <= t.n_s) continue;
          if (nd.box.level >= kMaxLevel) {
            capped = true;
            continue;
          }
          split[i] = 1;
          split_range(S, nd.box.sb, nd.box.se, nd.box.level, nd.sb);
          if (t.alias)
            for (int k = 0; k <= nchild; ++k) nd.tb[k] = nd.sb[k];
          else
            split_range(T, nd.box.tb, nd.box.te, nd.box.level, nd.tb);
        }
      }
      std::vector<int> next;
      next.reserve((size_t)nc * nchild);
      for (int i = 0; i < nc; ++i) {
        if (!split[i]) continue;
        const int id = cur[i];
        const int first = (int)nodes.size();
        nodes[id].kids = first;
        const Box par = nodes[id].box;
        const int32_t half = int32_t(1) << (kMaxLevel - 1 - par.level);
        for (int ci = 0; ci < nchild; ++ci) {
          Node c;
          c.box.level = par.level + 1;
          for (int a = 0; a < t.dim; ++a) c.box.anchor[a] = par.anchor[a] + ((ci >> a) & 1) * half;
          c.box.sb = nodes[id].sb[ci];
          c.box.se = nodes[id].sb[ci + 1];
          c.box.tb = nodes[id].tb[ci];
          c.box.te = nodes[id].tb[ci + 1];
          nodes.push_back(c);
          next.push_back(first + ci);
        }
      }
      cur.swap(next);
    }
    t.depth_capped = capped;
    const auto td0 = std::chrono::steady_clock::now();
    // DFS pre-order id allocation (stack pop order as in tree.cpp:110-122)
    std::vector<int> final_id(nodes.size(), -1);
    t.boxes.reserve(nodes.size() + nodes.size() / 4 + 64);  // room for the 2:1 repair's boxes
    t.boxes.assign(1, nodes[0].box);
    final_id[0] = 0;
    std::vector<int> stack(1, 0);
    while (!stack.empty()) {
      const int n = stack.back();
      stack.pop_back();
      if (nodes[n].kids < 0) continue;
      const int b = final_id[n];
      const int fc = t.num_boxes();
      t.boxes[b].leaf = false;
      t.boxes[b].first_child = fc;
      t.max_level = std::max(t.max_level, t.boxes[b].level + 1);
      for (int ci = 0; ci < nchild; ++ci) {
        Box c = nodes[nodes[n].kids + ci].box;
        c.parent = b;
        t.boxes.push_back(c);
        final_id[nodes[n].kids + ci] = fc + ci;
      }
      for (int ci = nchild - 1; ci >= 0; --ci) stack.push_back(nodes[n].kids + ci);
    }
    dfs_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - td0).count();
  }

  // does any of the 3^d - 1 probes of leaf b land in a leaf >= 2 levels coarser?
  // The box containing `probe` found from box `from`: climb to the first
  // ancestor that contains it, then descend, stopping at a leaf or at level
  // maxlev.  For the 2:1 probes of a leaf b (its 3^d - 1 neighbour centres)
  // the common ancestor is a few levels up, so this replaces most of a
  // root-to-leaf descent.  Returns the leaf containing the probe whenever
  // that leaf's level is < maxlev.
  int locate(int from, const int32_t* probe, int maxlev) const {
    int x = from;
    for (;;) {
      const Box& bx = t.boxes[x];
      const int64_t side = kCells >> bx.level;
      bool in = true;
      for (int a = 0; a < t.dim; ++a) in = in && probe[a] >= bx.anchor[a] && int64_t(probe[a]) < bx.anchor[a] + side;
      if (in || bx.parent < 0) break;
      x = bx.parent;
    }
    while (!t.boxes[x].leaf && t.boxes[x].level < maxlev) {
      int lev = t.boxes[x].level, ci = 0;
      for (int a = 0; a < t.dim; ++a) ci |= ((probe[a] >> (kMaxLevel - 1 - lev)) & 1) << a;
      x = t.boxes[x].first_child + ci;
    }
    return x;
  }

  // bit k set: the k-th of the 3^d offsets (o0 fastest, the centre counted) of
  // leaf b probes a leaf two or more levels coarser
  uint32_t probe_mask(int b) const {
    const int lev = t.boxes[b].level;
    if (lev < 2) return 0;
    const int64_t side = kCells >> lev;
    const int zr = t.dim == 3 ? 1 : 0;
    uint32_t mask = 0;
    int k = 0;
    for (int o2 = -zr; o2 <= zr; ++o2)
      for (int o1 = -1; o1 <= 1; ++o1)
        for (int o0 = -1; o0 <= 1; ++o0, ++k) {
          if (!o0 && !o1 && !o2) continue;
          const int off[3] = {o0, o1, o2};
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
          const int a = locate(t.boxes[b].parent, probe, lev - 1);
          if (t.boxes[a].leaf && t.boxes[a].level <= lev - 2) mask |= uint32_t(1) << k;
        }
    return mask;
  }

  // repair (tree.cpp:125-165): sweeps over the leaves in id order, each leaf
  // subdividing every leaf >= 2 levels coarser that one of its 3^d - 1 probes
  // lands in, until a sweep changes nothing.  Subdivisions only refine, so a
  // leaf that cannot trigger at the start of a sweep never triggers later;
  // the next sweep therefore only has to look at the leaves this sweep created
  // and the leaves that triggered in it (a coarse neighbour 3+ levels up may
  // still be 2+ levels up after one split).  The first sweep probes every
  // leaf in parallel; every replay runs in the reference's order.
  void repair() {
    std::vector<int> cand_ids;
    std::vector<uint32_t> cand_mask;  // per candidate: the offsets that trigger at the start of the sweep
    {
      std::vector<int> leaves;
      int lmin = kMaxLevel, lmax = 0;
      for (int b = 0; b < t.num_boxes(); ++b)
        if (t.boxes[b].leaf) {
          leaves.push_back(b);
          lmin = std::min(lmin, t.boxes[b].level);
          lmax = std::max(lmax, t.boxes[b].level);
        }
      // a trigger needs two leaves whose levels differ by >= 2: none when the
      // leaf levels span at most one level (uniform inputs), so no sweep can fire
      if (lmax - lmin <= 1) return;
      const int nl = (int)leaves.size();
      std::vector<uint32_t> cand(nl, 0);
      const auto r0 = std::chrono::steady_clock::now();
      if (dev_boxes && pa && pa->repair_scan) {
        std::vector<uint32_t> byb(t.num_boxes());
        pa->repair_scan(t.num_boxes(), byb.data());
        for (int i = 0; i < nl; ++i) cand[i] = byb[leaves[i]];
      } else {
#pragma omp parallel for schedule(dynamic, 64)
        for (int i = 0; i < nl; ++i) cand[i] = probe_mask(leaves[i]);
      }
      for (int i = 0; i < nl; ++i)
        if (cand[i]) {
          cand_ids.push_back(leaves[i]);
          cand_mask.push_back(cand[i]);
        }
      rep_scan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - r0).count();
      rep_leaves = nl;
    }
    while (!cand_ids.empty()) {
      ++rep_sweeps;
      rep_cands += (int)cand_ids.size();
      std::vector<int> next;
      for (size_t ic = 0; ic < cand_ids.size(); ++ic) {
        const int b = cand_ids[ic];
        // an offset that did not trigger when the sweep started cannot trigger
        // later in it (subdivisions only refine): only the flagged ones are
        // probed again, in the reference's order
        const uint32_t mask = cand_mask[ic];
        if (!t.boxes[b].leaf) continue;
        const int lev = t.boxes[b].level;
        const int64_t side = kCells >> lev;
        const int zr = t.dim == 3 ? 1 : 0;
        bool fired = false;
        int k = 0;
        for (int o2 = -zr; o2 <= zr; ++o2)
          for (int o1 = -1; o1 <= 1; ++o1)
            for (int o0 = -1; o0 <= 1; ++o0, ++k) {
              if (!((mask >> k) & 1)) continue;
              const int off[3] = {o0, o1, o2};
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
              const int a = locate(t.boxes[b].parent, probe, lev - 1);
              if (t.boxes[a].leaf && t.boxes[a].level <= lev - 2) {
                subdivide(a);
                for (int ci = 0; ci < nchild; ++ci) next.push_back(t.boxes[a].first_child + ci);
                fired = true;
              }
            }
        if (fired) next.push_back(b);
      }
      // the next sweep's candidates, in id order (the order the sweep visits leaves)
      std::sort(next.begin(), next.end());
      next.erase(std::unique(next.begin(), next.end()), next.end());
      std::vector<uint32_t> trig(next.size(), 0);
#pragma omp parallel for schedule(dynamic, 64)
      for (int i = 0; i < (int)next.size(); ++i) trig[i] = t.boxes[next[i]].leaf ? probe_mask(next[i]) : 0;
      cand_ids.clear();
      cand_mask.clear();
      for (size_t i = 0; i < next.size(); ++i)
        if (trig[i]) {
          cand_ids.push_back(next[i]);
          cand_mask.push_back(trig[i]);
        }
    }
  }

  void resolve_deferred() {
    if (deferred.empty()) return;
    // a box's own range is final once its parent's split is resolved: coarse levels first
    std::stable_sort(deferred.begin(), deferred.end(),
                     [&](int a, int b) { return t.boxes[a].level < t.boxes[b].level; });
    for (size_t i0 = 0; i0 < deferred.size();) {
      size_t i1 = i0;
      const int lev = t.boxes[deferred[i0]].level;
      while (i1 < deferred.size() && t.boxes[deferred[i1]].level == lev) ++i1;
      const int n = (int)(i1 - i0);
      std::vector<int> lvl(n, lev), sr(2 * n), tr(2 * n), sbn(9 * (size_t)n), tbn(9 * (size_t)n);
      for (int k = 0; k < n; ++k) {
        const Box& x = t.boxes[deferred[i0 + k]];
        sr[2 * k] = x.sb;
        sr[2 * k + 1] = x.se;
        tr[2 * k] = x.tb;
        tr[2 * k + 1] = x.te;
      }
      pa->split(n, lvl.data(), sr.data(), tr.data(), sbn.data(), tbn.data());
      for (int k = 0; k < n; ++k) {
        const int b = deferred[i0 + k], fc = t.boxes[b].first_child;
        const int* sb = sbn.data() + 9 * (size_t)k;
        const int* tb = t.alias ? sb : tbn.data() + 9 * (size_t)k;
        for (int ci = 0; ci < nchild; ++ci) {
          Box& c = t.boxes[fc + ci];
          c.sb = sb[ci];
          c.se = sb[ci + 1];
          c.tb = tb[ci];
          c.te = tb[ci + 1];
        }
      }
      i0 = i1;
    }
    deferred.clear();
  }

  bool touch(int b, int c, const int8_t* sh) const {  // tree.cpp:46-56
    int64_t sbz = kCells >> t.boxes[b].level, scz = kCells >> t.boxes[c].level;
    for (int a = 0; a < t.dim; ++a) {
      int64_t l1 = t.boxes[b].anchor[a], l2 = t.boxes[c].anchor[a] + sh[a] * kCells;
      if (l1 > l2 + scz || l2 > l1 + sbz) return false;
    }
    return true;
  }

  // two-pass CSR fill over `ids`: count(b) then emit(b, out)
  std::vector<int> leaf_ids(const std::vector<int>& ids) const {
    std::vector<int> v;
    v.reserve(ids.size());
    for (int b : ids)
      if (t.boxes[b].leaf) v.push_back(b);
    return v;
  }

  template <class Count, class Emit>
  void csr_pass(Csr& L, const std::vector<int>& ids, Count count, Emit emit) {
    const int n = (int)ids.size();
    std::vector<int> cnt(n);
#pragma omp parallel for schedule(dynamic, 64)
    for (int i = 0; i < n; ++i) cnt[i] = count(ids[i]);
    int64_t base = (int64_t)L.v.size();
    std::vector<int64_t> off(n);
    for (int i = 0; i < n; ++i) {
      off[i] = base;
      base += cnt[i];
    }
    L.v.resize(base);
#pragma omp parallel for schedule(dynamic, 64)
    for (int i = 0; i < n; ++i) {
      L.off[ids[i]] = off[i];
      L.len[ids[i]] = cnt[i];
      emit(ids[i], L.v.data() + off[i]);
    }
  }

  // leaves_only: coarse / fine lists only for leaves (all the evaluation
  // reads); the colleague lists are always complete (children's lists are
  // built from their parent's)
  void neighbours(bool leaves_only = false) {  // tree.cpp:167-212
    const auto tn0 = std::chrono::steady_clock::now();
    const int nb = t.num_boxes();
    for (Csr* L : {&t.col, &t.crs, &t.fin}) {
      L->off.assign(nb, 0);
      L->len.assign(nb, 0);
      L->v.clear();
    }
    t.level_boxes.assign(t.max_level + 1, {});
    for (int b = 0; b < nb; ++b) t.level_boxes[t.boxes[b].level].push_back(b);
    std::vector<Nbr> root;
    if (t.periodic) {
      const int zr = t.dim == 3 ? 1 : 0;
      for (int s2 = -zr; s2 <= zr; ++s2)
        for (int s1 = -1; s1 <= 1; ++s1)
          for (int s0 = -1; s0 <= 1; ++s0) root.push_back({0, {int8_t(s0), int8_t(s1), int8_t(s2)}});
    } else {
      root.push_back({0, {0, 0, 0}});
    }
    // colleague and coarse lists: at most 3^d entries per box, so each box
    // gets a fixed slot of that size (one pass per level, no counting pass,
    // no growth); the fine lists stay compact (two-pass CSR)
    const int K = t.dim == 3 ? 27 : 9;
    t.col.v.resize((size_t)nb * K);
    t.crs.v.resize((size_t)nb * K);
    t.col.off[0] = 0;
    t.col.len[0] = (int)root.size();
    std::copy(root.begin(), root.end(), t.col.v.begin());
    // relative position of box c (with periodic shift sh) to box b, in units of
    // b's side, per axis: exact integer (anchors are multiples of the side)
    // (the difference is an exact multiple of the power-of-two unit: a shift)
    auto rel = [&](int b, int c, const int8_t* sh, int64_t unit, int* o) {
      const int lg = __builtin_ctzll((unsigned long long)unit);
      for (int a = 0; a < t.dim; ++a)
        o[a] = int((int64_t(t.boxes[c].anchor[a]) + int64_t(sh[a]) * kCells - int64_t(t.boxes[b].anchor[a])) >> lg);
    };
    for (int lev = 1; lev <= t.max_level; ++lev) {
      const std::vector<int>& ids = t.level_boxes[lev];
      const int64_t ps = kCells >> (lev - 1);  // parent side
      // colleagues: children of the parent's non-leaf colleagues that touch b.
      // A child at offset 2 o + cc (child units) from b's parent touches b at
      // cb iff |2 o + cc - cb| <= 1 on every axis -- no child box is loaded.
      auto col_scan = [&](int b, Nbr* out) {
        const int par = t.boxes[b].parent;
        int cb[3] = {0, 0, 0};
        for (int a = 0; a < t.dim; ++a) cb[a] = int((t.boxes[b].anchor[a] - t.boxes[par].anchor[a]) >> (kMaxLevel - lev));
        int n = 0;
        for (const Nbr& pc : t.col[par]) {
          if (t.boxes[pc.box].leaf) continue;
          int o[3] = {0, 0, 0};
          rel(par, pc.box, pc.shift, ps, o);
          // allowed child bits per axis: |2 o + cc - cb| <= 1; the set of child
          // indices is their product, visited in ascending order
          unsigned mask = (1u << nchild) - 1u;
          for (int a = 0; a < t.dim; ++a) {
            unsigned ax = 0;
            for (int cc = 0; cc < 2; ++cc) {
              const int dlt = 2 * o[a] + cc - cb[a];
              if (dlt >= -1 && dlt <= 1) ax |= 1u << cc;
            }
            static constexpr unsigned kBit0[3] = {0x55u, 0x33u, 0x0Fu};  // child indices with bit a clear
            const unsigned full = (1u << nchild) - 1u, b0 = kBit0[a] & full, b1 = ~kBit0[a] & full;
            mask &= ((ax & 1u) ? b0 : 0u) | ((ax & 2u) ? b1 : 0u);
          }
          for (; mask; mask &= mask - 1) {
            const int ci = __builtin_ctz(mask);
            if (out) out[n] = {t.boxes[pc.box].first_child + ci, {pc.shift[0], pc.shift[1], pc.shift[2]}};
            ++n;
          }
        }
        return n;
      };
      const int nl = (int)ids.size();
#pragma omp parallel for schedule(dynamic, 128)
      for (int i = 0; i < nl; ++i) {
        const int b = ids[i];
        t.col.off[b] = (int64_t)b * K;
        t.col.len[b] = col_scan(b, t.col.v.data() + (size_t)b * K);
        // coarse: the parent's leaf colleagues that touch b
        if (leaves_only && !t.boxes[b].leaf) continue;
        Nbr* out = t.crs.v.data() + (size_t)b * K;
        int c = 0;
        for (const Nbr& pc : t.col[t.boxes[b].parent])
          if (t.boxes[pc.box].leaf && touch(b, pc.box, pc.shift)) out[c++] = pc;
        t.crs.off[b] = (int64_t)b * K;
        t.crs.len[b] = c;
      }
    }
    // fine: leaf children of non-leaf colleagues (other than self) that touch b.
    // A colleague at offset o (b's units) has children at 2 o + cc (half
    // units), touching b's [0, 2) iff 2 o + cc lies in [-1, 2].
    const auto tn1 = std::chrono::steady_clock::now();
    std::vector<int> all(nb);
    for (int b = 0; b < nb; ++b) all[b] = b;
    auto fine_scan = [&](int b, Nbr* out) {
      int c = 0;
      const int64_t side = kCells >> t.boxes[b].level;
      for (const Nbr& ce : t.col[b]) {
        if (ce.box == b && !ce.shift[0] && !ce.shift[1] && !ce.shift[2]) continue;
        if (t.boxes[ce.box].leaf) continue;
        int o[3] = {0, 0, 0};
        rel(b, ce.box, ce.shift, side, o);
        for (int ci = 0; ci < nchild; ++ci) {
          bool ok = true;
          for (int a = 0; a < t.dim; ++a) {
            const int pos = 2 * o[a] + ((ci >> a) & 1);
            ok = ok && pos >= -1 && pos <= 2;
          }
          if (!ok) continue;
          const int d = t.boxes[ce.box].first_child + ci;
          if (t.boxes[d].leaf) {
            if (out) out[c] = {d, {ce.shift[0], ce.shift[1], ce.shift[2]}};
            ++c;
          }
        }
      }
      return c;
    };
    csr_pass(t.fin, leaves_only ? leaf_ids(all) : all, [&](int b) { return fine_scan(b, nullptr); },
             [&](int b, Nbr* out) { fine_scan(b, out); });
    if (std::getenv("SDMK_TIMING")) {
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "[sdmk timing] neighbours: levels %.2f ms, fine %.2f ms (%d boxes, %d levels)\n",
                   ms(tn0, tn1), ms(tn1, std::chrono::steady_clock::now()), nb, t.max_level);
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

static HostTree build_topology_impl(int dim, bool periodic, int n_s, int p, int ns, const int32_t* qs, int nt,
                                    const int32_t* qt, const PointAccess* pa, bool with_neighbours) {
  Builder B;
  B.pa = pa;
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
  const auto c0 = std::chrono::steady_clock::now();
  B.refine();
  const auto c1 = std::chrono::steady_clock::now();
  B.repair();
  B.resolve_deferred();
  const auto c2 = std::chrono::steady_clock::now();
  if (with_neighbours) {
    B.neighbours();
    B.t.has_neighbours = true;
    B.t.full_neighbours = true;
  } else {
    B.t.level_boxes.assign(B.t.max_level + 1, {});
    for (int b = 0; b < B.t.num_boxes(); ++b) B.t.level_boxes[B.t.boxes[b].level].push_back(b);
  }
  const auto c3 = std::chrono::steady_clock::now();
  if (std::getenv("SDMK_TIMING")) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[sdmk timing] topology: refine %.2f ms (GPU split calls %.2f ms, DFS ids %.2f ms), repair %.2f ms, neighbours %.2f ms\n",
                 ms(c0, c1), B.split_ms, B.dfs_ms, ms(c1, c2), ms(c2, c3));
    std::fprintf(stderr, "[sdmk timing] repair: pre-scan %.2f ms over %d leaves, %d sweeps, %d candidates, %zu subdivisions\n",
                 B.rep_scan_ms, B.rep_leaves, B.rep_sweeps, B.rep_cands, B.deferred_total);
  }
  if (B.t.depth_capped)
    std::fprintf(stderr, "build_tree: depth cap %d reached with leaves above capacity (duplicate points?)\n",
                 kMaxLevel);
  return std::move(B.t);
}

HostTree build_topology(int dim, bool periodic, int n_s, int p, int ns, const int32_t* qs, int nt,
                        const int32_t* qt) {
  return build_topology_impl(dim, periodic, n_s, p, ns, qs, nt, qt, nullptr, true);
}

HostTree build_topology(int dim, bool periodic, int n_s, int p, int ns, int nt, const PointAccess& pa,
                        bool with_neighbours) {
  return build_topology_impl(dim, periodic, n_s, p, ns, nullptr, nt, nullptr, &pa, with_neighbours);
}

void finish_topology(HostTree& t, bool full) {
  if (t.has_neighbours && (t.full_neighbours || !full)) return;
  Builder B;
  B.t = std::move(t);
  B.nchild = 1 << B.t.dim;
  B.neighbours(!full);
  B.t.has_neighbours = true;
  B.t.full_neighbours = full;
  t = std::move(B.t);
}

std::string dump_topology(const HostTree& t) {  // tree.cpp:325-354
  std::ostringstream os;
  auto lst = [&](const char* tag, NbrSpan v) {
    os << ' ' << tag << "={";
    for (int i = 0; i < v.n; ++i) {
      if (i) os << ' ';
      os << v.p[i].box;
      if (v.p[i].shift[0] || v.p[i].shift[1] || v.p[i].shift[2])
        os << '@' << int(v.p[i].shift[0]) << ',' << int(v.p[i].shift[1]) << ',' << int(v.p[i].shift[2]);
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

ShardCosts shard_costs(const HostTree& t) {
  ShardCosts c;
  const int nb = t.num_boxes();
  // target leaves in Morton order = by the start of their target range
  // (sorted as packed (tb, id) keys: no indirection in the comparisons)
  std::vector<uint64_t> key;
  key.reserve(nb);
  for (int b = 0; b < nb; ++b)
    if (t.boxes[b].leaf && t.ntgt(b) > 0) key.push_back((uint64_t(uint32_t(t.boxes[b].tb)) << 32) | uint32_t(b));
  std::sort(key.begin(), key.end());
  c.leaves.resize(key.size());
  for (size_t i = 0; i < key.size(); ++i) c.leaves[i] = int(key[i] & 0xffffffffu);
  const int nl = (int)c.leaves.size();
  c.w.assign(nl, 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nl; ++i) {
    const int b = c.leaves[i];
    int64_t near = 0;  // sources of the near ranges (dmk.cpp:966-990)
    if (t.has_neighbours) {
      near += t.nsrc(b);
      for (const Nbr& e : t.col[b]) {
        if (e.box == b && !e.shift[0] && !e.shift[1] && !e.shift[2]) continue;
        if (t.boxes[e.box].leaf) near += t.nsrc(e.box);
      }
      for (const Nbr& e : t.crs[b]) near += t.nsrc(e.box);
      for (const Nbr& e : t.fin[b]) near += t.nsrc(e.box);
    }
    // every box with targets costs kCostPerBox (its plane-wave and tensor
    // work), shared by its target leaves in proportion to their targets
    int64_t boxes_w = 0;
    for (int a = b; a >= 0; a = t.boxes[a].parent) boxes_w += kCostPerBox * t.ntgt(b) / t.ntgt(a);
    c.w[i] = (int64_t)t.ntgt(b) * (near + kCostPerTarget) + boxes_w;
  }
  for (int64_t w : c.w) c.total += w;
  return c;
}

ShardPlan shard_plan(const HostTree& t, int rank, int nranks, const ShardCosts* costs) {
  ShardPlan sp;
  const int nb = t.num_boxes();
  if (nranks <= 1 && !costs) {  // everything, no costs needed
    for (int b = 0; b < nb; ++b)
      if (t.boxes[b].leaf && t.ntgt(b) > 0) sp.leaves.push_back(b);
    sp.t0 = 0;
    sp.t1 = t.ntgt(0);
    sp.need.assign(nb, 0);
    for (int b : sp.leaves)
      for (int x = b; x >= 0 && !sp.need[x]; x = t.boxes[x].parent) sp.need[x] = 1;
    return sp;
  }
  ShardCosts local;
  if (!costs) {
    local = shard_costs(t);
    costs = &local;
  }
  const std::vector<int>& tl = costs->leaves;
  const int64_t total = costs->total;
  sp.need.assign(nb, 0);
  if (nranks < 1) nranks = 1;
  int64_t start = 0;
  sp.t0 = -1;
  for (size_t i = 0; i < tl.size(); ++i) {
    const int b = tl[i];
    const int64_t n = costs->w[i];
    const int owner = nranks == 1 ? 0 : (int)std::min<int64_t>(nranks - 1, ((2 * start + n) * nranks) / (2 * total));
    if (owner == rank) {
      if (sp.t0 < 0) sp.t0 = t.boxes[b].tb;
      sp.t1 = t.boxes[b].te;
      sp.leaves.push_back(b);
    }
    start += n;
  }
  if (sp.t0 < 0) sp.t0 = sp.t1 = 0;
  std::sort(sp.leaves.begin(), sp.leaves.end());
  for (int b : sp.leaves)
    for (int x = b; x >= 0 && !sp.need[x]; x = t.boxes[x].parent) sp.need[x] = 1;
  return sp;
}

std::vector<int64_t> shard_bounds(const HostTree& t, int nranks, const ShardCosts& costs) {
  if (nranks < 1) nranks = 1;
  std::vector<int64_t> lo(nranks, -1), hi(nranks, -1);
  int64_t start = 0;
  for (size_t i = 0; i < costs.leaves.size(); ++i) {  // the owner rule of shard_plan
    const int b = costs.leaves[i];
    const int64_t n = costs.w[i];
    const int owner =
        nranks == 1 ? 0 : (int)std::min<int64_t>(nranks - 1, ((2 * start + n) * nranks) / (2 * costs.total));
    if (lo[owner] < 0) lo[owner] = t.boxes[b].tb;
    hi[owner] = t.boxes[b].te;
    start += n;
  }
  std::vector<int64_t> bounds(nranks + 1, 0);
  int64_t at = 0;
  for (int r = 0; r < nranks; ++r) {
    if (lo[r] >= 0) {
      if (lo[r] != at) throw RuntimeError("shard_bounds: owned target ranges do not tile the targets");
      at = hi[r];
    }
    bounds[r + 1] = at;
  }
  if (at != t.ntgt(0)) throw RuntimeError("shard_bounds: owned target ranges do not cover the targets");
  return bounds;
}

HaloPlan halo_owners(const HostTree& t, int nranks) {
  HaloPlan h;
  h.nranks = nranks < 1 ? 1 : nranks;
  const int nb = t.num_boxes();
  h.owner.assign(nb, -2);
  h.cut.assign(nb, 0);
  const int64_t total = t.nsrc(0);
  const int64_t thr = std::max<int64_t>(1, total / (8 * (int64_t)h.nranks));
  // cut boxes in DFS order of the subdivision = increasing source ranges
  std::vector<int> cutv, stack = {0};
  while (!stack.empty()) {
    const int b = stack.back();
    stack.pop_back();
    if (t.nsrc(b) == 0) continue;
    const Box& x = t.boxes[b];
    if (!x.leaf && t.nsrc(b) > thr && h.nranks > 1) {
      h.owner[b] = -1;
      for (int ci = (1 << t.dim) - 1; ci >= 0; --ci) stack.push_back(x.first_child + ci);
    } else {
      cutv.push_back(b);
    }
  }
  std::sort(cutv.begin(), cutv.end(), [&](int a, int b) { return t.boxes[a].sb < t.boxes[b].sb; });
  int64_t start = 0;
  for (int b : cutv) {
    const int64_t n = t.nsrc(b);
    const int r = h.nranks == 1 ? 0 : (int)std::min<int64_t>(h.nranks - 1, ((2 * start + n) * h.nranks) / (2 * total));
    start += n;
    h.cut[b] = 1;
    // the whole subtree (boxes with sources)
    std::vector<int> st = {b};
    while (!st.empty()) {
      const int x = st.back();
      st.pop_back();
      if (t.nsrc(x) == 0) continue;
      h.owner[x] = r;
      if (!t.boxes[x].leaf)
        for (int ci = 0; ci < (1 << t.dim); ++ci) st.push_back(t.boxes[x].first_child + ci);
    }
  }
  return h;
}

void halo_reads(const HostTree& t, HaloPlan& h, const ShardCosts* costs) {
  const int nb = t.num_boxes(), R = h.nranks;
  if (R > 64) throw InvalidArgument("halo plan: at most 64 ranks");
  ShardCosts local;
  if (!costs) {
    local = shard_costs(t);
    costs = &local;
  }
  // need masks: bit q on every box rank q forms incoming expansions for (its
  // target leaves by the shard rule and their ancestors)
  std::vector<uint64_t> need(nb, 0);
  int64_t start = 0;
  for (size_t i = 0; i < costs->leaves.size(); ++i) {
    const int64_t n = costs->w[i];
    const int q = R == 1 ? 0 : (int)std::min<int64_t>(R - 1, ((2 * start + n) * R) / (2 * costs->total));
    start += n;
    const uint64_t bit = uint64_t(1) << q;
    for (int x = costs->leaves[i]; x >= 0 && !(need[x] & bit); x = t.boxes[x].parent) need[x] |= bit;
  }
  // plane-wave targets of rank q: boxes with targets whose parent q needs;
  // q reads every colleague of its targets, and colleagues are mutual, so
  // the ranks reading box x are the union over x's colleagues c of tmask(c)
  auto tmask = [&](int c) -> uint64_t {
    if (t.ntgt(c) == 0) return 0;
    const int par = t.boxes[c].parent;
    return need[par >= 0 ? par : c];
  };
  h.readmask.assign(nb, 0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int x = 0; x < nb; ++x) {
    if (t.nsrc(x) == 0) continue;
    uint64_t m = 0;
    for (const Nbr& e : t.col[x]) m |= tmask(e.box);
    h.readmask[x] = m;
  }
}

std::vector<int> halo_boxes(const HaloPlan& h, int from, int to) {
  std::vector<int> v;
  if (from == to) return v;
  const int nb = (int)h.owner.size();
  for (int b = 0; b < nb; ++b)
    if (h.owner[b] == from && (h.cut[b] || (!h.readmask.empty() && ((h.readmask[b] >> to) & 1)))) v.push_back(b);
  return v;
}

}  // namespace sdmkb
