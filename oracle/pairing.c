/* pairing.c -- TEST INFRASTRUCTURE (oracle): an O(n log n) C restatement of
 * the reference's greedy power-of-two pairing (meshdist/bvh.py:98-181), for
 * the untimed tree topology of the bench's reference arm and for oracle
 * trees at sizes where the literal greedy (meshdist_oracle.greedy_pairs, the
 * reference's own loop, O(n^2) in practice) cannot finish.  Independent of
 * the product library; checked against the literal greedy and the
 * reference's goldens (tests/test_oracle_golden.py).
 *
 * The reference pops (surface_area, i) from a heap, skips pairs whose
 * triangles are merged, and parks a merge at an odd offset of an even run of
 * unmerged triangles while supply == need (bvh.py:133-166), re-offering the
 * parked pairs after every merge.  Equivalently: at each step it merges the
 * smallest (SA, i) pair that is valid and feasible, where
 *   feasible(i) = slack > 0 or run(i) has odd length or (i - run start) even
 *   slack = sum over runs of floor(len / 2) - need  (never increases).
 * Each run's best feasible pair is a range minimum over a static array (two
 * segment trees, one per index parity); runs sit in a lazy heap keyed by
 * their best pair; when slack first reaches 0 every even run is re-keyed.
 *
 * Build: cc -O2 -shared -fPIC oracle/pairing.c -o oracle/liboracle_pairing.so
 * (oracle/build.py; __graft_entry__.build() runs it). */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t size;
  int32_t* best[2];
  const double* sa;
} MinTree;

static int less_idx(const MinTree* t, int32_t a, int32_t b) {
  if (a < 0) return 0;
  if (b < 0) return 1;
  return t->sa[a] < t->sa[b] || (t->sa[a] == t->sa[b] && a < b);
}
static int32_t pick(const MinTree* t, int32_t a, int32_t b) { return less_idx(t, a, b) ? a : b; }

static int tree_init(MinTree* t, const double* keys, int64_t n) {
  t->sa = keys;
  t->size = 1;
  while (t->size < n) t->size <<= 1;
  for (int p = 0; p < 2; ++p) {
    t->best[p] = (int32_t*)malloc(sizeof(int32_t) * 2 * t->size);
    if (!t->best[p]) return -1;
    for (int64_t v = 0; v < 2 * t->size; ++v) t->best[p][v] = -1;
  }
  for (int64_t i = 0; i < n; ++i) t->best[i & 1][t->size + i] = (int32_t)i;
  for (int64_t v = t->size - 1; v >= 1; --v)
    for (int p = 0; p < 2; ++p) t->best[p][v] = pick(t, t->best[p][2 * v], t->best[p][2 * v + 1]);
  return 0;
}

/* best index in [l, r] with parity p (p = 2: any parity), -1 if none */
static int32_t tree_query(const MinTree* t, int64_t l, int64_t r, int p) {
  int32_t res = -1;
  for (int64_t a = l + t->size, b = r + t->size + 1; a < b; a >>= 1, b >>= 1) {
    if (a & 1) {
      if (p != 1) res = pick(t, res, t->best[0][a]);
      if (p != 0) res = pick(t, res, t->best[1][a]);
      ++a;
    }
    if (b & 1) {
      --b;
      if (p != 1) res = pick(t, res, t->best[0][b]);
      if (p != 0) res = pick(t, res, t->best[1][b]);
    }
  }
  return res;
}

typedef struct {
  double sa;
  int32_t i, start;
  uint32_t ver;
} Cand;

typedef struct {
  Cand* a;
  int64_t n, cap;
} Heap;

static int cand_after(const Cand* x, const Cand* y) { return x->sa > y->sa || (x->sa == y->sa && x->i > y->i); }

static int heap_push(Heap* h, Cand c) {
  if (h->n == h->cap) {
    int64_t nc = h->cap ? 2 * h->cap : 1024;
    Cand* na = (Cand*)realloc(h->a, sizeof(Cand) * nc);
    if (!na) return -1;
    h->a = na;
    h->cap = nc;
  }
  int64_t k = h->n++;
  h->a[k] = c;
  while (k > 0) {
    int64_t p = (k - 1) / 2;
    if (!cand_after(&h->a[p], &h->a[k])) break;
    Cand tmp = h->a[p];
    h->a[p] = h->a[k];
    h->a[k] = tmp;
    k = p;
  }
  return 0;
}

static Cand heap_pop(Heap* h) {
  Cand top = h->a[0];
  h->a[0] = h->a[--h->n];
  int64_t k = 0;
  for (;;) {
    int64_t l = 2 * k + 1, r = l + 1, m = k;
    if (l < h->n && cand_after(&h->a[m], &h->a[l])) m = l;
    if (r < h->n && cand_after(&h->a[m], &h->a[r])) m = r;
    if (m == k) break;
    Cand tmp = h->a[m];
    h->a[m] = h->a[k];
    h->a[k] = tmp;
    k = m;
  }
  return top;
}

typedef struct {
  MinTree tree;
  Heap heap;
  int32_t* run_end;
  uint32_t* run_ver;
  int64_t slack;
  const double* sa;
} State;

static int push_run(State* s, int32_t a, int32_t e) {
  s->run_end[a] = e;
  ++s->run_ver[a];
  if (e <= a) return 0; /* a single triangle has no pair */
  const int even = ((e - a + 1) % 2) == 0;
  const int par = (s->slack > 0 || !even) ? 2 : (a & 1);
  const int32_t i = tree_query(&s->tree, a, e - 1, par);
  if (i >= 0) {
    Cand c = {s->sa[i], i, a, s->run_ver[a]};
    return heap_push(&s->heap, c);
  }
  return 0;
}

/* sa: n - 1 surface areas of Morton neighbours (bvh.py:117-120); writes
 * is_left[i] = 1 iff triangles i, i + 1 (Morton ranks) share a leaf.
 * Returns 0, or -1 when out of memory. */
int oracle_pair_greedy(const double* sa, int64_t n, uint8_t* is_left) {
  memset(is_left, 0, (size_t)n);
  if (n < 2) return 0;
  int64_t L = 1;
  while (L * 2 <= n) L *= 2;
  int64_t need = n - L;
  if (need == 0) return 0;
  State s;
  memset(&s, 0, sizeof s);
  s.sa = sa;
  int rc = -1;
  s.run_end = (int32_t*)malloc(sizeof(int32_t) * n);
  s.run_ver = (uint32_t*)calloc((size_t)n, sizeof(uint32_t));
  if (!s.run_end || !s.run_ver || tree_init(&s.tree, sa, n - 1) != 0) goto done;
  for (int64_t i = 0; i < n; ++i) s.run_end[i] = -1;
  s.slack = n / 2 - need;
  if (push_run(&s, 0, (int32_t)(n - 1)) != 0) goto done;
  while (need > 0) {
    const Cand c = heap_pop(&s.heap);
    if (s.run_ver[c.start] != c.ver || s.run_end[c.start] < 0) continue; /* stale */
    const int32_t a = c.start, e = s.run_end[a], i = c.i;
    const int64_t m = e - a + 1, j = i - a;
    is_left[i] = 1;
    --need;
    const int was_pos = s.slack > 0;
    if (m % 2 == 0 && j % 2 == 1) --s.slack; /* only reachable with slack > 0 */
    s.run_end[a] = -1;
    ++s.run_ver[a];
    if (j > 0 && push_run(&s, a, i - 1) != 0) goto done;
    if (i + 2 <= e && push_run(&s, i + 2, e) != 0) goto done;
    if (was_pos && s.slack == 0 && need > 0) {
      /* feasibility changed for every even run: re-key them once */
      for (int32_t r = 0; r < n; ++r)
        if (s.run_end[r] >= r && ((s.run_end[r] - r + 1) % 2) == 0 && push_run(&s, r, s.run_end[r]) != 0) goto done;
    }
  }
  rc = 0;
done:
  free(s.tree.best[0]);
  free(s.tree.best[1]);
  free(s.heap.a);
  free(s.run_end);
  free(s.run_ver);
  return rc;
}
