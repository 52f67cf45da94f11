/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the dual-pool allocator's
 * batched trace.  Never linked into the product; tests and
 * bench.py's cpu_baseline leg load it through oracle/arena.py.
 *
 * Restates the contract of the reference's alloc_trace_run
 * (pkg/src/dvla/kernels/numba_backend.py:139-247; numpy twin
 * numpy_backend.py:121-212):
 *   - free extents are kept sorted by offset; an allocation takes the FIRST
 *     extent that holds `size` bytes at the next multiple of `align`, and the
 *     extent keeps its lead and/or tail remainder;
 *   - a free op releases live block number (pick mod n_live) of the live list
 *     in allocation order (the list closes the gap), coalescing with both
 *     neighbours;
 *   - out_ok: 1 placed, 0 no fit, 3 freed, 2 free with nothing live;
 *     out_off: the placed / freed offset, -1 otherwise;
 *   - returns (total free, largest free extent, number of extents).
 * Pinned against the reference's own traces (tests/golden/alloc_traces.npz,
 * tests/test_oracle.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t* off;
  int64_t* len;
  int64_t n;
} Extents;

static void ext_insert(Extents* e, int64_t at, int64_t off, int64_t len) {
  memmove(e->off + at + 1, e->off + at, (size_t)(e->n - at) * sizeof(int64_t));
  memmove(e->len + at + 1, e->len + at, (size_t)(e->n - at) * sizeof(int64_t));
  e->off[at] = off;
  e->len[at] = len;
  e->n++;
}

static void ext_erase(Extents* e, int64_t at) {
  memmove(e->off + at, e->off + at + 1, (size_t)(e->n - at - 1) * sizeof(int64_t));
  memmove(e->len + at, e->len + at + 1, (size_t)(e->n - at - 1) * sizeof(int64_t));
  e->n--;
}

/* first extent index whose offset is >= off */
static int64_t ext_lower_bound(const Extents* e, int64_t off) {
  int64_t lo = 0, hi = e->n;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (e->off[mid] < off) lo = mid + 1; else hi = mid;
  }
  return lo;
}

int oracle_alloc_trace(int64_t capacity, int64_t n, const uint8_t* is_alloc,
                       const int64_t* size, const int64_t* align, const uint64_t* pick,
                       uint8_t* out_ok, int64_t* out_off, int64_t* final3) {
  Extents fr;
  fr.off = (int64_t*)malloc((size_t)(n + 2) * sizeof(int64_t));
  fr.len = (int64_t*)malloc((size_t)(n + 2) * sizeof(int64_t));
  int64_t* live = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  int64_t* b_off = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  int64_t* b_len = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  if (!fr.off || !fr.len || !live || !b_off || !b_len) return 1;
  fr.n = 1;
  fr.off[0] = 0;
  fr.len[0] = capacity;
  int64_t n_live = 0;

  for (int64_t i = 0; i < n; ++i) {
    if (is_alloc[i] == 1) {
      const int64_t sz = size[i], al = align[i];
      int64_t j = 0, at = -1;
      for (; j < fr.n; ++j) {
        const int64_t a = (fr.off[j] + al - 1) / al * al;
        if (a + sz <= fr.off[j] + fr.len[j]) { at = a; break; }
      }
      if (at < 0) { out_ok[i] = 0; out_off[i] = -1; continue; }
      const int64_t end = fr.off[j] + fr.len[j];
      const int64_t lead = at - fr.off[j], tail = end - (at + sz);
      if (lead > 0) {
        fr.len[j] = lead;
        if (tail > 0) ext_insert(&fr, j + 1, at + sz, tail);
      } else if (tail > 0) {
        fr.off[j] = at + sz;
        fr.len[j] = tail;
      } else {
        ext_erase(&fr, j);
      }
      out_ok[i] = 1;
      out_off[i] = at;
      b_off[i] = at;
      b_len[i] = sz;
      live[n_live++] = i;
    } else {
      if (n_live == 0) { out_ok[i] = 2; out_off[i] = -1; continue; }
      const int64_t k = (int64_t)(pick[i] % (uint64_t)n_live);
      const int64_t blk = live[k];
      memmove(live + k, live + k + 1, (size_t)(n_live - k - 1) * sizeof(int64_t));
      n_live--;
      const int64_t off = b_off[blk], sz = b_len[blk];
      const int64_t j = ext_lower_bound(&fr, off);
      const int prev = j > 0 && fr.off[j - 1] + fr.len[j - 1] == off;
      const int next = j < fr.n && off + sz == fr.off[j];
      if (prev && next) {
        fr.len[j - 1] += sz + fr.len[j];
        ext_erase(&fr, j);
      } else if (prev) {
        fr.len[j - 1] += sz;
      } else if (next) {
        fr.off[j] = off;
        fr.len[j] += sz;
      } else {
        ext_insert(&fr, j, off, sz);
      }
      out_ok[i] = 3;
      out_off[i] = off;
    }
  }
  int64_t total = 0, largest = 0;
  for (int64_t j = 0; j < fr.n; ++j) {
    total += fr.len[j];
    if (fr.len[j] > largest) largest = fr.len[j];
  }
  final3[0] = total;
  final3[1] = largest;
  final3[2] = fr.n;
  free(fr.off); free(fr.len); free(live); free(b_off); free(b_len);
  return 0;
}
