// Host-side box topology of the adaptive level-restricted 2^d tree.
//
// The points are quantized, Morton-keyed and radix-sorted on the GPU
// (kernels/tree_kernels.cu); this module consumes the sorted quantized
// coordinates and reproduces the reference's box ids, ranges and neighbour
// lists bit-exactly (tree.cpp:62-212): ids follow the DFS subdivision order
// of refine_to_capacity, then the append order of the 2:1 repair sweeps.
// Boxes are few (<= ~1e5) compared with points, so this is a host pass; it
// is restructured for speed without changing the result:
//  * refine: the subdivision set depends only on counts, so it is built
//    level by level with parallel binary searches (within a box the child
//    index is non-decreasing in Morton order), then renumbered in the DFS
//    pre-order the reference allocates ids in;
//  * repair: a parallel read-only pre-scan finds every leaf that could
//    trigger a subdivision (a subdivision only makes boxes finer, so it can
//    only remove triggers); only those are replayed sequentially, in order;
//  * neighbours: CSR lists, built level by level in parallel.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace sdmkb {

constexpr int kMaxLevel = 30;

struct Box {
  int level = 0, parent = -1, first_child = -1;
  bool leaf = true;
  int32_t anchor[3] = {0, 0, 0};
  int sb = 0, se = 0, tb = 0, te = 0;  // permuted source / target ranges
};

struct Nbr {
  int box;
  int8_t shift[3];
};

struct NbrSpan {
  const Nbr* p = nullptr;
  int n = 0;
  const Nbr* begin() const { return p; }
  const Nbr* end() const { return p + n; }
  int size() const { return n; }
};

struct Csr {
  std::vector<int64_t> off;  // per box: start
  std::vector<int> len;      // per box: count
  std::vector<Nbr> v;
  NbrSpan operator[](int b) const { return {v.data() + off[b], len[b]}; }
};

struct HostTree {
  int dim = 3, n_s = 0, p = 0, max_level = 0;
  bool periodic = false, alias = true, depth_capped = false;
  bool has_neighbours = false;   // col / crs / fin built (finish_topology)
  bool full_neighbours = false;  // crs / fin for every box, not only the leaves
  std::vector<Box> boxes;
  std::vector<std::vector<int>> level_boxes;
  Csr col, crs, fin;  // colleagues / coarse / fine
  int num_boxes() const { return (int)boxes.size(); }
  int nsrc(int b) const { return boxes[b].se - boxes[b].sb; }
  int ntgt(int b) const { return boxes[b].te - boxes[b].tb; }
  double side(int b) const;
  std::array<double, 3> center(int b) const;
};

// qs / qt: sorted quantized coordinates, SoA (q[axis * n + i]).  nt == 0
// means the targets alias the sources.
HostTree build_topology(int dim, bool periodic, int n_s, int p, int ns, const int32_t* qs, int nt,
                        const int32_t* qt);

// The same with the point data kept elsewhere (the GPU): `split` gives, for
// n boxes (level lvl[i], source range src[2i..2i+1], target range
// tgt[2i..2i+1]), the 2^d + 1 child boundaries of each range (sb[9i..],
// tb[9i..]); the refine calls it once per level.  `host_q` returns host
// copies of the sorted quantized coordinates; it is called only if the 2:1
// repair has to subdivide a leaf (never for uniform inputs).
struct PointAccess {
  std::function<void(int n, const int* lvl, const int* src, const int* tgt, int* sb, int* tb)> split;
  std::function<void(const int32_t** qs, const int32_t** qt)> host_q;
  // optional: the whole capacity refinement on the device -- fills `boxes` in
  // the reference's id order and returns true, or returns false (the refine
  // then runs on the host, level by level through `split`)
  std::function<bool(std::vector<Box>& boxes, int& max_level, bool& depth_capped)> refine;
  // optional, after a device refine: the repair's read-only first sweep over
  // those boxes on the device (cand[b] bit k: the k-th of leaf b's 3^d offsets,
  // o0 fastest and the centre counted, probes a leaf two or more levels coarser)
  std::function<void(int nboxes, uint32_t* cand)> repair_scan;
};
// with_neighbours = false leaves col / crs / fin for finish_topology (the
// upward pass needs only the boxes; the engine builds the lists while it runs)
HostTree build_topology(int dim, bool periodic, int n_s, int p, int ns, int nt, const PointAccess& pa,
                        bool with_neighbours = true);
// full = false builds coarse / fine lists for the leaves only (what the
// evaluation reads); dump_topology needs full lists
void finish_topology(HostTree& t, bool full = false);

// The reference's canonical text dump (tree.cpp:325-354).
std::string dump_topology(const HostTree& t);

// Target-leaf ownership of rank `rank` of `nranks`: the
// target leaves in Morton order (by the start of their target range) are cut
// into contiguous runs of about total / nranks cost (a leaf goes to the rank
// whose share contains its midpoint).  Cost of a target leaf, in units of one
// residual pair test: nt * (sources in its near ranges + kCostPerTarget) +
// sum over the leaf and its ancestors a of kCostPerBox * nt / nt(a) -- the
// residual pairs, the interpolation per target and the plane-wave / tensor
// work of every box shared by its target leaves (ratios from the N = 1e7
// launch list).  `need` marks the owned leaves
// and their ancestors -- the boxes whose incoming expansions the rank forms;
// [t0, t1) is the owned range of Morton-sorted targets.  nranks == 1 owns
// everything.
struct ShardPlan {
  int64_t t0 = 0, t1 = 0;
  std::vector<int> leaves;  // owned target leaves, by id
  std::vector<char> need;   // per box
};
constexpr int64_t kCostPerTarget = 1190, kCostPerBox = 860000;
struct ShardCosts {
  std::vector<int> leaves;  // target leaves in Morton order
  std::vector<int64_t> w;   // their costs
  int64_t total = 0;
};
ShardCosts shard_costs(const HostTree& t);  // needs the neighbour lists
ShardPlan shard_plan(const HostTree& t, int rank, int nranks, const ShardCosts* costs = nullptr);
// the owned ranges of all ranks at once: rank r owns sorted targets
// [bounds[r], bounds[r + 1]) (the same ranges shard_plan gives; they tile
// [0, nt) in rank order, an empty rank has bounds[r] == bounds[r + 1])
std::vector<int64_t> shard_bounds(const HostTree& t, int nranks, const ShardCosts& costs);

// Source ownership for the distributed upward pass.
// The cut: starting from the root, every non-leaf box holding more than
// total / (8 nranks) sources is replaced by its children with sources.  The
// cut boxes, in Morton order (= source-range order), are dealt to ranks in
// contiguous runs by source count (a box goes to the rank whose share holds
// its midpoint).  A cut box's whole subtree belongs to its owner; the boxes
// above the cut (all non-leaf) are merged by every rank from the gathered
// cut boxes.  readmask[b] bit r: rank r's plane-wave pass reads box b's outgoing
// expansion (b is a colleague of one of r's plane-wave targets -- a target
// whose parent r needs, shard_plan).
struct HaloPlan {
  int nranks = 1;
  std::vector<int> owner;                // per box: rank; -1 above the cut; -2 no sources
  std::vector<char> cut;                 // per box
  std::vector<uint64_t> readmask;        // per box: bit r = rank r reads it
};
// owner/cut only (what the upward pass of one rank needs)
HaloPlan halo_owners(const HostTree& t, int nranks);
// adds reads[] for every rank
void halo_reads(const HostTree& t, HaloPlan& h, const ShardCosts* costs = nullptr);  // nranks <= 64
// boxes (sorted ids) rank `to` receives from rank `from`: owned by `from`,
// and either a cut box (every rank merges the boxes above the cut) or read by `to`
std::vector<int> halo_boxes(const HaloPlan& h, int from, int to);

}  // namespace sdmkb
