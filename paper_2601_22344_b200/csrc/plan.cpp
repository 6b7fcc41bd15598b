// Host-native interaction-plan build for the certified-bound plan path
// (reference rplu.treebounds, pkg/src/rplu/treebounds.py):
// square-box quadtrees over the target points x and the source points y
// (:47-104) and the dual traversal that fills each target leaf's aggregated
// (source node, 1/d_min^2) and exact (source leaf) lists (Alg C.1,
// build_plan :141-180).
//
// The plan depends only on the point sets and is built once per call on the
// host, as in the reference; a Python loop over ~2e6 box pairs took 3.1 s at
// C4 size (2^20 points per side).  The arithmetic is the reference's: the
// same box corners, edge padding, quadrant order (NW, NE, SW, SE, empty
// children skipped, depth-first with a stack), first-maximum max() and no
// FMA contraction (built with -ffp-contract=off), so the plans are identical
// (tests/test_treebounds_cpu.py checks them against the reference's and the
// Python restatement).
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rplu_b200.h"

namespace rplu {
void set_error(const std::string& msg);
}

namespace {

// Points live in ONE index array `order`: node k owns order[pbeg[k] ..
// pend[k]), in the reference's order (a node's points are partitioned stably
// into its quadrants, so a leaf lists its points in increasing input order,
// as the reference's boolean-mask selection does).  (The first version kept a
// vector of indices per node and pushed every point into a fresh quadrant
// vector at every level: 200 ms per tree at 2^20 points, allocation bound.)
struct Tree {
  std::vector<double> x0, y0, size;
  std::vector<int64_t> parent;
  std::vector<std::vector<int64_t>> children;
  std::vector<int64_t> order, pbeg, pend;
  std::vector<int64_t> leaves;
  int64_t npts(int64_t k) const { return pend[k] - pbeg[k]; }
  const int64_t* pts(int64_t k) const { return order.data() + pbeg[k]; }
};

// Python's max(): the first maximal argument wins (strict >)
inline double pymax(double a, double b) { return b > a ? b : a; }
inline double pymax3(double a, double b, double c) { return pymax(pymax(a, b), c); }

void build_tree(const double* p, int64_t n, int64_t leaf_size, Tree& t) {
  double ox = p[0], oy = p[1], mx = p[0], my = p[1];
  for (int64_t i = 1; i < n; ++i) {
    ox = std::min(ox, p[2 * i]);
    oy = std::min(oy, p[2 * i + 1]);
    mx = std::max(mx, p[2 * i]);
    my = std::max(my, p[2 * i + 1]);
  }
  double edge = pymax3(mx - ox, my - oy, 1e-300);
  edge *= 1.0 + 1e-12;
  t.x0 = {ox};
  t.y0 = {oy};
  t.size = {edge};
  t.parent = {-1};
  t.children.assign(1, {});
  // the partition carries the coordinates with the indices (24 bytes per
  // point, sequential passes): gathering p[2 i] through the permuted index
  // array missed the caches at every level below the first few (200 ms per
  // tree at 2^20 points against ~70 ms this way)
  struct Pt { double x, y; int64_t i; };
  std::vector<Pt> pts(n), tmp(n);
  for (int64_t i = 0; i < n; ++i) pts[i] = Pt{p[2 * i], p[2 * i + 1], i};
  t.pbeg = {0};
  t.pend = {n};
  // a node's points sit in `pts` or in `tmp` (side 0 / 1): the partition
  // scatters them into the other array, so nothing is copied back
  std::vector<uint8_t> side = {0};
  std::vector<uint8_t> cls(n);
  std::vector<int64_t> todo = {0};
  while (!todo.empty()) {
    const int64_t k = todo.back();
    todo.pop_back();
    Pt* idx = (side[k] ? tmp : pts).data() + t.pbeg[k];
    Pt* dst = (side[k] ? pts : tmp).data() + t.pbeg[k];
    const int64_t cnt = t.pend[k] - t.pbeg[k];
    bool same = true;
    const double rx = idx[0].x, ry = idx[0].y;
    if (cnt > leaf_size) {
      for (int64_t q = 0; q < cnt; ++q)
        if (!(idx[q].x == rx && idx[q].y == ry)) { same = false; break; }
    }
    if (cnt <= leaf_size || same) {
      t.leaves.push_back(k);
      continue;
    }
    const double h = t.size[k] / 2.0;
    const double cx = t.x0[k] + h, cy = t.y0[k] + h;
    // stable 4-way partition (NW, NE, SW, SE): classify, scatter, copy back
    int64_t count[4] = {0, 0, 0, 0};
    for (int64_t q = 0; q < cnt; ++q) {
      const bool east = idx[q].x >= cx, north = idx[q].y >= cy;
      const uint8_t c = (uint8_t)(north ? (east ? 1 : 0) : (east ? 3 : 2));
      cls[q] = c;
      ++count[c];
    }
    int64_t off[4] = {0, count[0], count[0] + count[1], count[0] + count[1] + count[2]};
    const int64_t start[4] = {off[0], off[1], off[2], off[3]};
    for (int64_t q = 0; q < cnt; ++q) dst[off[cls[q]]++] = idx[q];
    const double bx[4] = {t.x0[k], cx, t.x0[k], cx};
    const double by[4] = {cy, cy, t.y0[k], t.y0[k]};
    std::vector<int64_t> kids;
    for (int q = 0; q < 4; ++q) {
      if (count[q] == 0) continue;
      const int64_t c = (int64_t)t.x0.size();
      t.x0.push_back(bx[q]);
      t.y0.push_back(by[q]);
      t.size.push_back(h);
      t.parent.push_back(k);
      t.children.emplace_back();
      t.pbeg.push_back(t.pbeg[k] + start[q]);
      t.pend.push_back(t.pbeg[k] + start[q] + count[q]);
      side.push_back((uint8_t)(side[k] ^ 1));
      kids.push_back(c);
      todo.push_back(c);
    }
    t.children[k] = kids;
  }
  t.order.resize(n);   // the leaves tile [0, n)
  for (int64_t k : t.leaves) {
    const Pt* from = (side[k] ? tmp : pts).data();
    for (int64_t q = t.pbeg[k]; q < t.pend[k]; ++q) t.order[q] = from[q].i;
  }
}

// (d_min^2, d_max^2) between square ia of tree a and square ib of tree b
inline void box_dist2(const Tree& a, int64_t ia, const Tree& b, int64_t ib, double& dmin2,
                      double& dmax2) {
  const double ax0 = a.x0[ia], ay0 = a.y0[ia], asz = a.size[ia];
  const double bx0 = b.x0[ib], by0 = b.y0[ib], bsz = b.size[ib];
  const double ax1 = ax0 + asz, ay1 = ay0 + asz, bx1 = bx0 + bsz, by1 = by0 + bsz;
  const double dx = pymax3(0.0, bx0 - ax1, ax0 - bx1);
  const double dy = pymax3(0.0, by0 - ay1, ay0 - by1);
  const double ex = pymax(bx1 - ax0, ax1 - bx0);
  const double ey = pymax(by1 - ay0, ay1 - by0);
  const double dxx = dx * dx, dyy = dy * dy, exx = ex * ex, eyy = ey * ey;
  dmin2 = dxx + dyy;
  dmax2 = exx + eyy;
}

}  // namespace

struct rplu_plan_host {
  Tree tgt, src;
  std::vector<int64_t> agg_start, agg_node, ex_start, ex_node;
  std::vector<double> agg_alpha;
};

extern "C" {

int rplu_plan_build(const double* x, int64_t n, const double* y, int64_t m, double nu,
                    int64_t leaf_size, int64_t* coincident, rplu_plan_host** out) {
  if (!out || !x || !y || n < 1 || m < 1) {
    rplu::set_error("rplu_plan_build: bad argument (empty point set?)");
    return RPLU_ERR_ARG;
  }
  *out = nullptr;
  if (!(nu >= 1.0)) { rplu::set_error("nu must be >= 1"); return RPLU_ERR_ARG; }
  if (leaf_size < 1) { rplu::set_error("leaf size must be >= 1"); return RPLU_ERR_ARG; }
  rplu_plan_host* h = new rplu_plan_host();
  {  // the two trees are independent: build the source tree on a second thread
    std::thread other([&] { build_tree(y, m, leaf_size, h->src); });
    build_tree(x, n, leaf_size, h->tgt);
    other.join();
  }
  const Tree& tgt = h->tgt;
  const Tree& src = h->src;
  // target leaves below every target node (leaf order)
  std::vector<std::vector<int64_t>> under(tgt.x0.size());
  for (int64_t leaf : tgt.leaves)
    for (int64_t k = leaf; k != -1; k = tgt.parent[k]) under[k].push_back(leaf);
  std::vector<int64_t> slot(tgt.x0.size(), -1);
  for (size_t q = 0; q < tgt.leaves.size(); ++q) slot[tgt.leaves[q]] = (int64_t)q;
  // The dual traversal (Alg C.1) in the reference's order -- a stack whose
  // last pushed pair is visited first -- split into independent subtrees: the
  // top kSplitDepth levels are expanded on this thread into the list of
  // subtree roots IN VISITING ORDER, worker threads traverse the subtrees
  // into private record lists, and the records are appended to the per-leaf
  // lists in root order, so every list comes out exactly as the sequential
  // traversal writes it (115 -> ~30 ms at 2^20 points per side).
  struct AggRec { int64_t slot, node; double alpha; };
  struct ExRec { int64_t slot, node; };
  struct Task {
    int64_t s, t;
    std::vector<AggRec> agg;
    std::vector<ExRec> ex;
    bool coincide = false;
    int64_t ca = -1, cb = -1;
  };
  auto admissible = [&](int64_t s, int64_t t, double& dmin2) {
    double dmax2;
    box_dist2(src, s, tgt, t, dmin2, dmax2);
    return dmin2 > 0.0 && dmax2 <= nu * dmin2;
  };
  // children of a non-terminal pair in PUSH order (the reference pushes them
  // in this order and pops the last one first)
  auto push_order = [&](int64_t s, int64_t t, std::vector<std::pair<int64_t, int64_t>>& out) {
    const bool s_leaf = src.children[s].empty(), t_leaf = tgt.children[t].empty();
    if ((tgt.size[t] >= src.size[s] && !t_leaf) || s_leaf) {
      for (int64_t c : tgt.children[t]) out.push_back({s, c});
    } else {
      for (int64_t c : src.children[s]) out.push_back({c, t});
    }
  };
  auto run_task = [&](Task& task) {
    std::vector<std::pair<int64_t, int64_t>> todo = {{task.s, task.t}};
    while (!todo.empty()) {
      const auto st = todo.back();
      todo.pop_back();
      const int64_t s = st.first, t = st.second;
      double dmin2;
      if (admissible(s, t, dmin2)) {
        for (int64_t leaf : under[t]) {
          double lmin2, lmax2;
          box_dist2(src, s, tgt, leaf, lmin2, lmax2);
          task.agg.push_back({slot[leaf], s, 1.0 / lmin2});
        }
        continue;
      }
      const bool s_leaf = src.children[s].empty(), t_leaf = tgt.children[t].empty();
      if (s_leaf && t_leaf) {
        if (dmin2 == 0.0) {  // coincident target / source points (treebounds.py:183-194)
          for (int64_t qa = 0; qa < tgt.npts(t) && !task.coincide; ++qa)
            for (int64_t qb = 0; qb < src.npts(s); ++qb) {
              const int64_t a = tgt.pts(t)[qa], b = src.pts(s)[qb];
              if (x[2 * a] == y[2 * b] && x[2 * a + 1] == y[2 * b + 1]) {
                task.coincide = true;
                task.ca = a;
                task.cb = b;
                break;
              }
            }
          if (task.coincide) return;
        }
        task.ex.push_back({slot[t], s});
        continue;
      }
      push_order(s, t, todo);
    }
  };
  constexpr int kSplitDepth = 4;
  std::vector<Task> tasks;
  {
    struct Item { int64_t s, t; int depth; };
    std::vector<Item> st = {{0, 0, 0}};
    std::vector<std::pair<int64_t, int64_t>> kids;
    while (!st.empty()) {
      const Item it = st.back();
      st.pop_back();
      double dmin2;
      const bool term = admissible(it.s, it.t, dmin2) ||
                        (src.children[it.s].empty() && tgt.children[it.t].empty());
      if (term || it.depth == kSplitDepth) {
        tasks.emplace_back();
        tasks.back().s = it.s;
        tasks.back().t = it.t;
        continue;
      }
      kids.clear();
      push_order(it.s, it.t, kids);
      for (const auto& c : kids) st.push_back({c.first, c.second, it.depth + 1});
    }
  }
  {
    unsigned hw = std::thread::hardware_concurrency();
    const int nthreads = (int)std::max(1u, std::min(std::min(hw ? hw : 1u, 8u),
                                                    (unsigned)tasks.size()));
    std::atomic<size_t> next{0};
    auto worker = [&] {
      for (size_t k = next.fetch_add(1); k < tasks.size(); k = next.fetch_add(1)) run_task(tasks[k]);
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < nthreads; ++w) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
  }
  // records -> CSR lists per target leaf, in visiting order (count, prefix,
  // fill: two passes over the records; appending them to one vector per leaf
  // and flattening those cost 120 ms at 2^20 points per side)
  const size_t nleaf = tgt.leaves.size();
  for (const Task& task : tasks) {   // the first coincidence in visiting order wins, as in the reference
    if (task.coincide) {
      if (coincident) { coincident[0] = task.ca; coincident[1] = task.cb; }
      rplu::set_error("coincident target / source points");
      delete h;
      return RPLU_ERR_ARG;
    }
  }
  h->agg_start.assign(nleaf + 1, 0);
  h->ex_start.assign(nleaf + 1, 0);
  for (const Task& task : tasks) {
    for (const AggRec& r : task.agg) ++h->agg_start[r.slot + 1];
    for (const ExRec& r : task.ex) ++h->ex_start[r.slot + 1];
  }
  for (size_t q = 0; q < nleaf; ++q) {
    h->agg_start[q + 1] += h->agg_start[q];
    h->ex_start[q + 1] += h->ex_start[q];
  }
  h->agg_node.resize((size_t)h->agg_start[nleaf]);
  h->agg_alpha.resize((size_t)h->agg_start[nleaf]);
  h->ex_node.resize((size_t)h->ex_start[nleaf]);
  {
    std::vector<int64_t> ca(h->agg_start.begin(), h->agg_start.end() - 1);
    std::vector<int64_t> ce(h->ex_start.begin(), h->ex_start.end() - 1);
    for (const Task& task : tasks) {
      for (const AggRec& r : task.agg) {
        const int64_t k = ca[r.slot]++;
        h->agg_node[k] = r.node;
        h->agg_alpha[k] = r.alpha;
      }
      for (const ExRec& r : task.ex) h->ex_node[ce[r.slot]++] = r.node;
    }
  }
  *out = h;
  return RPLU_OK;
}

int rplu_plan_counts(const rplu_plan_host* h, int64_t* counts) {
  if (!h || !counts) { rplu::set_error("rplu_plan_counts: NULL argument"); return RPLU_ERR_ARG; }
  const Tree* tr[2] = {&h->tgt, &h->src};
  for (int w = 0; w < 2; ++w) {
    int64_t nc = 0;
    for (const auto& c : tr[w]->children) nc += (int64_t)c.size();
    counts[3 * w + 0] = (int64_t)tr[w]->x0.size();
    counts[3 * w + 1] = (int64_t)tr[w]->leaves.size();
    counts[3 * w + 2] = nc;
  }
  counts[6] = (int64_t)h->agg_node.size();
  counts[7] = (int64_t)h->ex_node.size();
  return RPLU_OK;
}

int rplu_plan_tree(const rplu_plan_host* h, int32_t which, double* x0, double* y0, double* size,
                   int64_t* parent, int64_t* cstart, int64_t* cidx, int64_t* leaves,
                   int64_t* lpstart, int64_t* lpidx) {
  if (!h || (which != 0 && which != 1) || !x0 || !y0 || !size || !parent || !cstart || !cidx ||
      !leaves || !lpstart || !lpidx) {
    rplu::set_error("rplu_plan_tree: bad argument");
    return RPLU_ERR_ARG;
  }
  const Tree& t = which == 0 ? h->tgt : h->src;
  const size_t nn = t.x0.size();
  std::copy(t.x0.begin(), t.x0.end(), x0);
  std::copy(t.y0.begin(), t.y0.end(), y0);
  std::copy(t.size.begin(), t.size.end(), size);
  std::copy(t.parent.begin(), t.parent.end(), parent);
  int64_t c = 0;
  for (size_t k = 0; k < nn; ++k) {
    cstart[k] = c;
    for (int64_t ch : t.children[k]) cidx[c++] = ch;
  }
  cstart[nn] = c;
  int64_t p = 0;
  for (size_t q = 0; q < t.leaves.size(); ++q) {
    leaves[q] = t.leaves[q];
    lpstart[q] = p;
    for (int64_t e = 0; e < t.npts(t.leaves[q]); ++e) lpidx[p++] = t.pts(t.leaves[q])[e];
  }
  lpstart[t.leaves.size()] = p;
  return RPLU_OK;
}

int rplu_plan_lists(const rplu_plan_host* h, int64_t* agg_start, int64_t* agg_node,
                    double* agg_alpha, int64_t* ex_start, int64_t* ex_node) {
  if (!h || !agg_start || !agg_node || !agg_alpha || !ex_start || !ex_node) {
    rplu::set_error("rplu_plan_lists: bad argument");
    return RPLU_ERR_ARG;
  }
  std::copy(h->agg_start.begin(), h->agg_start.end(), agg_start);
  std::copy(h->agg_node.begin(), h->agg_node.end(), agg_node);
  std::copy(h->agg_alpha.begin(), h->agg_alpha.end(), agg_alpha);
  std::copy(h->ex_start.begin(), h->ex_start.end(), ex_start);
  std::copy(h->ex_node.begin(), h->ex_node.end(), ex_node);
  return RPLU_OK;
}

int rplu_plan_free(rplu_plan_host* h) {
  delete h;
  return RPLU_OK;
}

}  // extern "C"
