/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the rowblock hot path.
 *
 * This is a plain-C restatement of the reference algorithm (rowblock v0.1.0,
 * /root/reference/pkg/src/rowblock/) used ONLY by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * leg, as the checker.  The shipped product path (paper_2202_05868_b200/)
 * never links, imports or calls anything under oracle/.
 *
 * Parity pinning: the restatement is checked against golden vectors
 * produced by running the reference itself (tests/golden/make_golden.py,
 * committed fixtures tests/golden/*.npz) and against the reference's own
 * known-answer tests (tests/test_oracle.py).
 *
 * Functions and the reference lines they restate:
 *   orc_quotient      blocking.py:118-136 (_quotient_bits) + matrix.py:164-166 (segment_of)
 *   orc_block_1sa     blocking.py:283-306 (block_1sa), compression 295-301,
 *                     _greedy_merge 209-266 in its scalar form (merge_condition 184-203),
 *                     _build_grouping 269-280
 *   orc_vbr_blocks    vbr.py:88-125 (stored block columns per block row, recomputed from data)
 *   orc_vbr_scatter   vbr.py:113-123 (float64 payload of every stored block)
 *   orc_block_1sa_pruned  the same greedy scan with exact candidate pruning (config 3 sizes)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* segment index of column c: searchsorted(boundaries, c, 'right') - 1 (matrix.py:164-166) */
static int64_t seg_of(const int64_t* bounds, int64_t n_seg, int64_t c) {
  int64_t lo = 0, hi = n_seg + 1; /* first index with bounds[i] > c */
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (bounds[mid] > c) hi = mid; else lo = mid + 1;
  }
  return lo - 1;
}

static int64_t n_words_of(int64_t n_seg) { return n_seg > 0 ? (n_seg + 63) / 64 : 1; }

/* bits: [n_rows x W] uint64 zeroed by us; sizes: [n_rows] */
int orc_quotient(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx, const int64_t* bounds,
                 int64_t n_seg, uint64_t* bits, int64_t* sizes) {
  int64_t W = n_words_of(n_seg);
  memset(bits, 0, sizeof(uint64_t) * (size_t)(n_rows * W));
  for (int64_t i = 0; i < n_rows; ++i) {
    int64_t cnt = 0;
    uint64_t* row = bits + i * W;
    if (n_seg > 0) {
      for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
        int64_t s = seg_of(bounds, n_seg, col_idx[p]);
        uint64_t m = (uint64_t)1 << (s & 63);
        if (!(row[s >> 6] & m)) { row[s >> 6] |= m; ++cnt; }
      }
    }
    sizes[i] = cnt;
  }
  return 0;
}

static int64_t popc_and(const uint64_t* a, const uint64_t* b, int64_t W) {
  int64_t c = 0;
  for (int64_t w = 0; w < W; ++w) c += __builtin_popcountll(a[w] & b[w]);
  return c;
}

/* Merge predicate, scalar form of blocking.py:239-248 (== merge_condition 184-203).
 * All float arithmetic is IEEE double exactly as numpy evaluates it:
 *   jaccard: float(inter) >= tau * float(union)
 *   cosine : float(inter) >= tau * sqrt(float(psize * size)), and if tau > 0 the emptiness clause
 *   bounded: float(union) <= cap,  cap = seed_size / (1.0 - 0.5 * tau)                        */
static int accept(int64_t inter, int64_t psize, int64_t size, double tau, int cosine, int bounded, double cap) {
  int64_t uni = psize + size - inter;
  int ok;
  if (!cosine) {
    ok = (double)inter >= tau * (double)uni;
  } else {
    ok = (double)inter >= tau * sqrt((double)(psize * size));
    if (tau > 0.0) ok = ok && ((size == 0) == (psize == 0));
  }
  if (ok && bounded) ok = (double)uni <= cap;
  return ok;
}

/* Outputs (caller-allocated):
 *   group_of[n_rows], row_perm[n_rows] (= concat of group rows, vbr.py:99-100),
 *   group_ptr[n_rows+1] (row extents of each group in row_perm), seed_size[n_rows],
 *   pattern_ptr[n_rows+1], pattern_idx[max(nnz,1)]  (sorted segment ids of OR of members),
 *   n_groups_out[1].
 * Returns 0, or -1 on allocation failure.                                           */
int orc_block_1sa(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx, const int64_t* bounds,
                  int64_t n_seg, double tau, int cosine, int bounded, int pattern_update, int use_compression,
                  int64_t* group_of, int64_t* row_perm, int64_t* group_ptr, int64_t* seed_size,
                  int64_t* pattern_ptr, int64_t* pattern_idx, int64_t* n_groups_out) {
  int64_t W = n_words_of(n_seg);
  uint64_t* bits = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n_rows * W + 1));
  int64_t* sizes = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
  int64_t* item_of_row = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
  int64_t* reps = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
  if (!bits || !sizes || !item_of_row || !reps) return -1;
  orc_quotient(n_rows, row_ptr, col_idx, bounds, n_seg, bits, sizes);

  /* ---- compression (blocking.py:295-301): classes of identical quotient rows, keyed on the exact
   * words, ordered by their smallest row; rows ascending inside a class.  Hash table keyed on the
   * words with exact comparison.                                                               */
  int64_t m = 0;
  if (use_compression) {
    int64_t cap = 16;
    while (cap < 2 * n_rows) cap <<= 1;
    int64_t* table = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
    if (!table) return -1;
    for (int64_t t = 0; t < cap; ++t) table[t] = -1;
    for (int64_t i = 0; i < n_rows; ++i) {
      const uint64_t* b = bits + i * W;
      uint64_t h = 1469598103934665603ull;
      for (int64_t w = 0; w < W; ++w) { h ^= b[w]; h *= 1099511628211ull; h ^= h >> 29; }
      int64_t t = (int64_t)(h & (uint64_t)(cap - 1));
      for (;;) {
        int64_t it = table[t];
        if (it < 0) { table[t] = m; reps[m] = i; item_of_row[i] = m; ++m; break; }
        if (memcmp(bits + reps[it] * W, b, sizeof(uint64_t) * (size_t)W) == 0) { item_of_row[i] = it; break; }
        t = (t + 1) & (cap - 1);
      }
    }
    free(table);
  } else {
    for (int64_t i = 0; i < n_rows; ++i) { reps[i] = i; item_of_row[i] = i; }
    m = n_rows;
  }

  /* ---- greedy one-pass scan (blocking.py:209-266), scalar form. */
  int64_t* group_of_item = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t* seed_item = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  uint64_t* P = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)W);
  if (!group_of_item || !seed_item || !P) return -1;
  for (int64_t j = 0; j < m; ++j) group_of_item[j] = -1;
  int64_t H = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (group_of_item[i] >= 0) continue;
    group_of_item[i] = H;
    seed_item[H] = i;
    memcpy(P, bits + reps[i] * W, sizeof(uint64_t) * (size_t)W);
    int64_t psize = sizes[reps[i]];
    double capv = bounded ? (double)psize / (1.0 - 0.5 * tau) : 0.0;
    for (int64_t j = i + 1; j < m; ++j) {
      if (group_of_item[j] >= 0) continue;
      const uint64_t* bj = bits + reps[j] * W;
      int64_t sj = sizes[reps[j]];
      int64_t inter = popc_and(P, bj, W);
      if (accept(inter, psize, sj, tau, cosine, bounded, capv)) {
        group_of_item[j] = H;
        if (pattern_update && inter < sj) {
          for (int64_t w = 0; w < W; ++w) P[w] |= bj[w];
          psize = psize + sj - inter;
        }
      }
    }
    ++H;
  }

  /* ---- grouping assembly (blocking.py:269-280): group rows = concat of member source lists in
   * merge order.  Members are accepted in ascending item order, items are ordered by smallest
   * row, rows ascending inside an item: a counting sort by (group, item) stable in row order. */
  int64_t* cnt = (int64_t*)calloc((size_t)(H + 1), sizeof(int64_t));
  int64_t* icnt = (int64_t*)calloc((size_t)(m + 1), sizeof(int64_t));
  int64_t* iptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  if (!cnt || !icnt || !iptr) return -1;
  for (int64_t r = 0; r < n_rows; ++r) icnt[item_of_row[r]]++;
  /* item start positions when items are laid out group-major, item ascending */
  for (int64_t j = 0; j < m; ++j) cnt[group_of_item[j]] += icnt[j];
  group_ptr[0] = 0;
  for (int64_t g = 0; g < H; ++g) group_ptr[g + 1] = group_ptr[g] + cnt[g];
  {
    int64_t* gcur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(H + 1));
    for (int64_t g = 0; g < H; ++g) gcur[g] = group_ptr[g];
    for (int64_t j = 0; j < m; ++j) { iptr[j] = gcur[group_of_item[j]]; gcur[group_of_item[j]] += icnt[j]; }
    free(gcur);
  }
  for (int64_t r = 0; r < n_rows; ++r) {
    int64_t it = item_of_row[r];
    row_perm[iptr[it]++] = r;
    group_of[r] = group_of_item[it];
  }
  /* patterns: OR of member bits -> sorted segment ids; seed_size = seed item's size */
  uint64_t* gb = (uint64_t*)calloc((size_t)(H * W + 1), sizeof(uint64_t));
  if (!gb) return -1;
  for (int64_t j = 0; j < m; ++j) {
    uint64_t* d = gb + group_of_item[j] * W;
    const uint64_t* s = bits + reps[j] * W;
    for (int64_t w = 0; w < W; ++w) d[w] |= s[w];
  }
  pattern_ptr[0] = 0;
  for (int64_t g = 0; g < H; ++g) {
    int64_t k = pattern_ptr[g];
    for (int64_t w = 0; w < W; ++w) {
      uint64_t x = gb[g * W + w];
      while (x) { int b = __builtin_ctzll(x); pattern_idx[k++] = w * 64 + b; x &= x - 1; }
    }
    pattern_ptr[g + 1] = k;
    seed_size[g] = sizes[reps[seed_item[g]]];
  }
  *n_groups_out = H;
  free(gb); free(cnt); free(icnt); free(iptr); free(group_of_item); free(seed_item); free(P);
  free(bits); free(sizes); free(item_of_row); free(reps);
  return 0;
}

/* Stored block columns per block row (vbr.py:106-112): for block row g (rows
 * row_perm[row_partition[g]:row_partition[g+1]]) the sorted set of segments holding >= 1 nonzero.
 * Outputs blk_ptr[H+1] and blk_col[max(nnz,1)].                                                */
int orc_vbr_blocks(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx, const int64_t* bounds,
                   int64_t n_seg, const int64_t* row_perm, const int64_t* row_partition, int64_t H,
                   int64_t* blk_ptr, int64_t* blk_col) {
  int64_t W = n_words_of(n_seg);
  uint64_t* acc = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)W);
  if (!acc) return -1;
  blk_ptr[0] = 0;
  for (int64_t g = 0; g < H; ++g) {
    memset(acc, 0, sizeof(uint64_t) * (size_t)W);
    for (int64_t p = row_partition[g]; p < row_partition[g + 1]; ++p) {
      int64_t r = row_perm[p];
      if (r < 0 || r >= n_rows) { free(acc); return -2; }
      for (int64_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) {
        int64_t s = seg_of(bounds, n_seg, col_idx[q]);
        acc[s >> 6] |= (uint64_t)1 << (s & 63);
      }
    }
    int64_t k = blk_ptr[g];
    for (int64_t w = 0; w < W; ++w) {
      uint64_t x = acc[w];
      while (x) { int b = __builtin_ctzll(x); blk_col[k++] = w * 64 + b; x &= x - 1; }
    }
    blk_ptr[g + 1] = k;
  }
  free(acc);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Pruned restatement of the same greedy scan (SURVEY App. A "exact pruning"), used as the oracle at
 * sizes where the dense O(m^2 W) scan is infeasible (config 3, R-MAT 2^20).  Identical output to
 * orc_block_1sa; candidates of a round are enumerated from an inverted index over a PREFIX of the
 * current pattern (its psize - t + 1 rarest segments, t = the least intersection any acceptable
 * candidate must have), which is exact because every acceptable candidate shares >= t segments
 * with P.  Falls back to the full scan when t == 0 (tau == 0 or an empty pattern).
 * Work counters: stats[0] rounds, stats[1] postings entries visited, stats[2] candidates evaluated. */
static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : x > y;
}

int orc_block_1sa_pruned(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx, const int64_t* bounds,
                         int64_t n_seg, double tau, int cosine, int bounded, int pattern_update, int use_compression,
                         int64_t* group_of, int64_t* row_perm, int64_t* group_ptr, int64_t* seed_size,
                         int64_t* pattern_ptr, int64_t* pattern_idx, int64_t* n_groups_out, int64_t* stats) {
  /* per-row sorted unique segment lists */
  int64_t* rs_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
  int64_t nnz = row_ptr[n_rows];
  int64_t* rs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz + 1));
  if (!rs_ptr || !rs) return -1;
  rs_ptr[0] = 0;
  for (int64_t i = 0; i < n_rows; ++i) {
    int64_t k = rs_ptr[i], last = -1;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      int64_t s = seg_of(bounds, n_seg, col_idx[p]);
      if (s != last) { rs[k++] = s; last = s; }
    }
    rs_ptr[i + 1] = k;
  }
  /* compression keyed on the exact segment list (first-occurrence order) */
  int64_t* item_of_row = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
  int64_t* reps = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_rows + 1));
  int64_t m = 0;
  if (use_compression) {
    int64_t cap = 16;
    while (cap < 2 * n_rows) cap <<= 1;
    int64_t* table = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
    for (int64_t t = 0; t < cap; ++t) table[t] = -1;
    for (int64_t i = 0; i < n_rows; ++i) {
      uint64_t h = 1469598103934665603ull ^ (uint64_t)(rs_ptr[i + 1] - rs_ptr[i]);
      for (int64_t p = rs_ptr[i]; p < rs_ptr[i + 1]; ++p) { h ^= (uint64_t)rs[p]; h *= 1099511628211ull; h ^= h >> 29; }
      int64_t t = (int64_t)(h & (uint64_t)(cap - 1));
      for (;;) {
        int64_t it = table[t];
        if (it < 0) { table[t] = m; reps[m] = i; item_of_row[i] = m; ++m; break; }
        int64_t r = reps[it];
        int64_t len = rs_ptr[i + 1] - rs_ptr[i];
        if (rs_ptr[r + 1] - rs_ptr[r] == len && memcmp(rs + rs_ptr[r], rs + rs_ptr[i], sizeof(int64_t) * (size_t)len) == 0) {
          item_of_row[i] = it;
          break;
        }
        t = (t + 1) & (cap - 1);
      }
    }
    free(table);
  } else {
    for (int64_t i = 0; i < n_rows; ++i) { reps[i] = i; item_of_row[i] = i; }
    m = n_rows;
  }
  /* item segment lists and inverted index (postings ascending by item) */
  int64_t* isz = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t* post_ptr = (int64_t*)calloc((size_t)(n_seg + 2), sizeof(int64_t));
  for (int64_t j = 0; j < m; ++j) {
    int64_t r = reps[j];
    isz[j] = rs_ptr[r + 1] - rs_ptr[r];
    for (int64_t p = rs_ptr[r]; p < rs_ptr[r + 1]; ++p) post_ptr[rs[p] + 1]++;
  }
  for (int64_t s = 0; s < n_seg; ++s) post_ptr[s + 1] += post_ptr[s];
  int64_t* post = (int64_t*)malloc(sizeof(int64_t) * (size_t)(post_ptr[n_seg] + 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_seg + 1));
  memcpy(fill, post_ptr, sizeof(int64_t) * (size_t)(n_seg + 1));
  for (int64_t j = 0; j < m; ++j) {
    int64_t r = reps[j];
    for (int64_t p = rs_ptr[r]; p < rs_ptr[r + 1]; ++p) post[fill[rs[p]]++] = j;
  }
  int64_t W = n_words_of(n_seg);
  uint64_t* P = (uint64_t*)calloc((size_t)W, sizeof(uint64_t));
  int64_t* plist = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_seg + 1));
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * n_seg + 2));
  int64_t* group_of_item = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t* seed_item = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t* stamp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  uint8_t* okv = (uint8_t*)malloc((size_t)(m + 1));
  int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  /* empty items (pattern size 0), ascending: the only candidates of an empty pattern when tau > 0 */
  int64_t* empt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t n_empty = 0;
  for (int64_t j = 0; j < m; ++j) { group_of_item[j] = -1; stamp[j] = -1; if (isz[j] == 0) empt[n_empty++] = j; }
  int64_t H = 0, next = 0, round = 0;
  stats[0] = stats[1] = stats[2] = 0;
  while (next < m) {
    int64_t seed = next;
    group_of_item[seed] = H;
    seed_item[H] = seed;
    int64_t r0 = reps[seed];
    memset(P, 0, sizeof(uint64_t) * (size_t)W);
    int64_t psize = 0;
    for (int64_t p = rs_ptr[r0]; p < rs_ptr[r0 + 1]; ++p) { P[rs[p] >> 6] |= 1ull << (rs[p] & 63); plist[psize++] = rs[p]; }
    double capv = bounded ? (double)psize / (1.0 - 0.5 * tau) : 0.0;
    int64_t pos = seed + 1;
    for (;;) {
      ++round;
      ++stats[0];
      /* least intersection t of any acceptable candidate (conservative, exact) */
      int64_t t;
      if (!cosine) { double lb = tau * (double)psize; t = (int64_t)ceil(lb); }
      else { double lb = tau * tau * (double)psize * (1.0 - 1e-12); t = (int64_t)ceil(lb); if (t < 0) t = 0; }
      int64_t nc = 0;
      if (t >= 1 && psize > 0) {
        /* prefix = the psize - t + 1 segments of P with the shortest postings lists */
        int64_t npre = psize - t + 1;
        for (int64_t q = 0; q < psize; ++q) { order[2 * q] = post_ptr[plist[q] + 1] - post_ptr[plist[q]]; order[2 * q + 1] = plist[q]; }
        /* partial selection sort is fine for small psize; qsort pairs otherwise */
        for (int64_t a = 0; a < npre; ++a) {
          int64_t best = a;
          for (int64_t b = a + 1; b < psize; ++b)
            if (order[2 * b] < order[2 * best] || (order[2 * b] == order[2 * best] && order[2 * b + 1] < order[2 * best + 1])) best = b;
          int64_t x0 = order[2 * a], x1 = order[2 * a + 1];
          order[2 * a] = order[2 * best]; order[2 * a + 1] = order[2 * best + 1];
          order[2 * best] = x0; order[2 * best + 1] = x1;
        }
        for (int64_t a = 0; a < npre; ++a) {
          int64_t s = order[2 * a + 1];
          int64_t lo = post_ptr[s], hi = post_ptr[s + 1];
          while (lo < hi) { int64_t mid = (lo + hi) / 2; if (post[mid] < pos) lo = mid + 1; else hi = mid; }
          for (int64_t q = lo; q < post_ptr[s + 1]; ++q) {
            ++stats[1];
            int64_t j = post[q];
            if (group_of_item[j] >= 0 || stamp[j] == round) continue;
            stamp[j] = round;
            cand[nc++] = j;
          }
        }
      } else if (psize == 0 && tau > 0.0) {
        for (int64_t q = 0; q < n_empty; ++q) if (empt[q] >= pos && group_of_item[empt[q]] < 0) cand[nc++] = empt[q];
      } else {
        for (int64_t j = pos; j < m; ++j) if (group_of_item[j] < 0) cand[nc++] = j;
      }
      /* evaluate candidates; first growing hit */
      int64_t jstar = m;
      for (int64_t q = 0; q < nc; ++q) {
        int64_t j = cand[q], rj = reps[j], inter = 0;
        ++stats[2];
        for (int64_t p = rs_ptr[rj]; p < rs_ptr[rj + 1]; ++p) inter += (P[rs[p] >> 6] >> (rs[p] & 63)) & 1;
        int ok = accept(inter, psize, isz[j], tau, cosine, bounded, capv);
        okv[j] = (uint8_t)ok;
        if (ok && pattern_update && inter < isz[j] && j < jstar) jstar = j;
      }
      for (int64_t q = 0; q < nc; ++q) {
        int64_t j = cand[q];
        if (okv[j] && j < jstar) group_of_item[j] = H;
      }
      if (jstar < m) {
        int64_t rj = reps[jstar];
        group_of_item[jstar] = H;
        for (int64_t p = rs_ptr[rj]; p < rs_ptr[rj + 1]; ++p) {
          int64_t s = rs[p];
          if (!((P[s >> 6] >> (s & 63)) & 1)) { P[s >> 6] |= 1ull << (s & 63); plist[psize++] = s; }
        }
        pos = jstar + 1;
        continue;
      }
      break;
    }
    ++H;
    while (next < m && group_of_item[next] >= 0) ++next;
  }
  /* assembly identical to orc_block_1sa */
  int64_t* icnt = (int64_t*)calloc((size_t)(m + 1), sizeof(int64_t));
  int64_t* cnt = (int64_t*)calloc((size_t)(H + 1), sizeof(int64_t));
  int64_t* iptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  int64_t* gcur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(H + 1));
  for (int64_t r = 0; r < n_rows; ++r) icnt[item_of_row[r]]++;
  for (int64_t j = 0; j < m; ++j) cnt[group_of_item[j]] += icnt[j];
  group_ptr[0] = 0;
  for (int64_t g = 0; g < H; ++g) group_ptr[g + 1] = group_ptr[g] + cnt[g];
  for (int64_t g = 0; g < H; ++g) gcur[g] = group_ptr[g];
  for (int64_t j = 0; j < m; ++j) { iptr[j] = gcur[group_of_item[j]]; gcur[group_of_item[j]] += icnt[j]; }
  for (int64_t r = 0; r < n_rows; ++r) { int64_t it = item_of_row[r]; row_perm[iptr[it]++] = r; group_of[r] = group_of_item[it]; }
  /* patterns: sorted union of member segment lists */
  int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_seg + 1));
  for (int64_t s = 0; s < n_seg; ++s) mark[s] = -1;
  int64_t* mem_ptr = (int64_t*)calloc((size_t)(H + 1), sizeof(int64_t));
  int64_t* mem = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  for (int64_t j = 0; j < m; ++j) mem_ptr[group_of_item[j] + 1]++;
  for (int64_t g = 0; g < H; ++g) mem_ptr[g + 1] += mem_ptr[g];
  for (int64_t g = 0; g < H; ++g) gcur[g] = mem_ptr[g];
  for (int64_t j = 0; j < m; ++j) mem[gcur[group_of_item[j]]++] = j;
  pattern_ptr[0] = 0;
  for (int64_t g = 0; g < H; ++g) {
    int64_t k = pattern_ptr[g];
    for (int64_t q = mem_ptr[g]; q < mem_ptr[g + 1]; ++q) {
      int64_t r = reps[mem[q]];
      for (int64_t p = rs_ptr[r]; p < rs_ptr[r + 1]; ++p)
        if (mark[rs[p]] != g) { mark[rs[p]] = g; pattern_idx[k++] = rs[p]; }
    }
    qsort(pattern_idx + pattern_ptr[g], (size_t)(k - pattern_ptr[g]), sizeof(int64_t), cmp_i64);
    pattern_ptr[g + 1] = k;
    seed_size[g] = isz[seed_item[g]];
  }
  *n_groups_out = H;
  free(mark); free(mem_ptr); free(mem); free(icnt); free(cnt); free(iptr); free(gcur);
  free(P); free(plist); free(order); free(group_of_item); free(seed_item); free(stamp); free(okv); free(cand); free(empt);
  free(isz); free(post_ptr); free(post); free(fill); free(rs_ptr); free(rs); free(item_of_row); free(reps);
  return 0;
}

/* Dense float64 payloads of the stored blocks (vbr.py:113-123): block k of block row g is an
 * h_g x w_{bcol} row-major array at flat[blk_off[k]], zero except the nonzeros of g's rows,
 * scattered at [local row, col - bounds[bcol]].  Blocks of a row are ascending in bcol and a row's
 * columns are ascending, so one forward walk over the row's blocks places every nonzero.
 * Returns 0, or -3 if a nonzero lies outside the row's stored blocks.                          */
int orc_vbr_scatter(int64_t n_rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                    const int64_t* bounds, const int64_t* row_perm, const int64_t* row_partition, int64_t H,
                    const int64_t* blk_ptr, const int64_t* blk_col, const int64_t* blk_off, double* flat) {
  for (int64_t g = 0; g < H; ++g) {
    const int64_t b0 = blk_ptr[g], b1 = blk_ptr[g + 1];
    for (int64_t p = row_partition[g]; p < row_partition[g + 1]; ++p) {
      const int64_t r = row_perm[p], local = p - row_partition[g];
      if (r < 0 || r >= n_rows) return -2;
      int64_t k = b0;
      for (int64_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) {
        const int64_t c = col_idx[q];
        while (k < b1 && bounds[blk_col[k] + 1] <= c) ++k;
        if (k == b1 || bounds[blk_col[k]] > c) return -3;
        const int64_t w = bounds[blk_col[k] + 1] - bounds[blk_col[k]];
        flat[blk_off[k] + local * w + (c - bounds[blk_col[k]])] = values[q];
      }
    }
  }
  return 0;
}
