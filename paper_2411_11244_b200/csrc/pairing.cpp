// pairing.cpp -- exact O(n log n) restatement of the reference's greedy
// power-of-two pairing (bvh.py:98-181).
//
// The reference pops (surface_area, i) from a heap, skips pairs whose
// triangles are already merged, and defers a merge at an odd offset of an
// even-length run of singletons while supply == need (bvh.py:133-166);
// deferred pairs are re-offered after every merge.  Its result is therefore:
// at each step merge the smallest (SA, i) pair that is valid (both ends
// unmerged) and feasible in the current state, where
//   feasible(i) = slack > 0  or  run(i) has odd length  or  (i - run.start) even
//   slack       = sum_runs floor(len/2) - need   (never increases).
// Valid pairs of a run [s, e] are i in [s, e-1], so each run's best feasible
// pair is a range-minimum query over a static array (one segment tree per
// index parity); runs live in a lazy heap keyed by their best pair.  When the
// slack first reaches 0 every even run is re-keyed once.
#include <stdint.h>

#include <algorithm>
#include <queue>
#include <vector>

namespace gd {

namespace {

struct MinTree {
  // iterative segment tree over positions [0, n); node holds the best index
  // of each parity (-1 = none), ordered by (sa[i], i)
  int64_t size = 1;
  std::vector<int32_t> best[2];
  const double* sa = nullptr;

  bool less(int32_t a, int32_t b) const {
    if (a < 0) return false;
    if (b < 0) return true;
    return sa[a] < sa[b] || (sa[a] == sa[b] && a < b);
  }
  int32_t pick(int32_t a, int32_t b) const { return less(a, b) ? a : b; }

  void init(const double* keys, int64_t n) {
    sa = keys;
    while (size < n) size <<= 1;
    for (int p = 0; p < 2; ++p) best[p].assign(2 * size, -1);
    for (int64_t i = 0; i < n; ++i) best[i & 1][size + i] = (int32_t)i;
    for (int64_t v = size - 1; v >= 1; --v)
      for (int p = 0; p < 2; ++p) best[p][v] = pick(best[p][2 * v], best[p][2 * v + 1]);
  }
  // best index in [l, r] with parity p (p = 2: any parity)
  int32_t query(int64_t l, int64_t r, int p) const {
    int32_t res = -1;
    for (int64_t a = l + size, b = r + size + 1; a < b; a >>= 1, b >>= 1) {
      if (a & 1) {
        if (p != 1) res = pick(res, best[0][a]);
        if (p != 0) res = pick(res, best[1][a]);
        ++a;
      }
      if (b & 1) {
        --b;
        if (p != 1) res = pick(res, best[0][b]);
        if (p != 0) res = pick(res, best[1][b]);
      }
    }
    return res;
  }
};

struct Cand {
  double sa;
  int32_t i;       // best pair of the run
  int32_t start;   // run start
  uint32_t ver;    // run version when pushed
};
struct CandAfter {
  bool operator()(const Cand& a, const Cand& b) const {
    return a.sa > b.sa || (a.sa == b.sa && a.i > b.i);
  }
};

}  // namespace

// sa: n-1 surface areas; is_left[i] = 1 iff triangles i, i+1 (Morton ranks)
// share a leaf.
void pair_greedy(const double* sa, int64_t n, uint8_t* is_left) {
  std::fill(is_left, is_left + n, 0);
  if (n < 2) return;
  int64_t L = 1;
  while (L * 2 <= n) L *= 2;
  int64_t need = n - L;
  if (need == 0) return;
  MinTree tree;
  tree.init(sa, n - 1);
  std::vector<int32_t> run_end(n, -1);
  std::vector<uint32_t> run_ver(n, 0);
  int64_t slack = n / 2 - need;
  std::priority_queue<Cand, std::vector<Cand>, CandAfter> heap;

  auto push_run = [&](int32_t s, int32_t e) {
    run_end[s] = e;
    ++run_ver[s];
    if (e <= s) return;  // a single triangle has no pair
    const bool even = ((e - s + 1) % 2) == 0;
    const int par = (slack > 0 || !even) ? 2 : (s & 1);
    const int32_t i = tree.query(s, e - 1, par);
    if (i >= 0) heap.push(Cand{sa[i], i, s, run_ver[s]});
  };

  push_run(0, (int32_t)(n - 1));
  while (need > 0) {
    const Cand c = heap.top();
    heap.pop();
    if (run_ver[c.start] != c.ver || run_end[c.start] < 0) continue;  // stale
    const int32_t s = c.start, e = run_end[s], i = c.i;
    const int64_t m = e - s + 1, j = i - s;
    is_left[i] = 1;
    --need;
    const bool was_pos = slack > 0;
    if (m % 2 == 0 && j % 2 == 1) --slack;  // only reachable with slack > 0
    run_end[s] = -1;
    ++run_ver[s];
    if (j > 0) push_run(s, i - 1);
    if (i + 2 <= e) push_run(i + 2, e);
    if (was_pos && slack == 0 && need > 0) {
      // feasibility changed for every even run: re-key them once
      for (int32_t r = 0; r < n; ++r)
        if (run_end[r] >= r && ((run_end[r] - r + 1) % 2) == 0) push_run(r, run_end[r]);
    }
  }
}

}  // namespace gd
