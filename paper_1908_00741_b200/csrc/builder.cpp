// Host-side builder for the HBMC ICCG path: orderings, permutation, IC(0),
// SELL packing.  Every routine is a bit-exact restatement of the reference's
// numba kernel or numpy code it replaces (citations on each function); the
// Python-level loops of the reference (pad_colors, csr_to_sell, permute)
// become linear native passes, parallelised with OpenMP only where the
// output does not depend on the schedule.
//
// Compiled with -ffp-contract=off: the factorisation must round exactly like
// the reference (separate multiply and subtract, no FMA).

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <new>
#include <queue>
#include <string>
#include <vector>

#include "tb_internal.h"

namespace tb {
static thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

void clear_error() { g_err.clear(); }
}  // namespace tb

using tb::fail;

extern "C" const char *tb_last_error(void) { return tb::g_err.c_str(); }

extern "C" int tb_abi_version(void) { return 3; }

#define TB_TRY_BEGIN try {
#define TB_TRY_END                                              \
  }                                                             \
  catch (const std::bad_alloc &) {                              \
    return fail(TB_ENOMEM, "host allocation failed");          \
  }                                                             \
  catch (const std::exception &e) {                             \
    return fail(TB_EINVAL, "internal error: %s", e.what());     \
  }

// ---------------------------------------------------------------------------
// K/numba_backend.py:232-270 grow_blocks.  Seed = smallest unassigned index;
// grow by the smallest unassigned neighbour of the whole block so far.  The
// reference keeps a binary min-heap with duplicates and discards assigned
// entries when popped; the next member is therefore always the minimum
// unassigned value ever pushed for this block, which any min-heap yields.
extern "C" int tb_grow_blocks(int64_t n, const int64_t *row_ptr,
                              const int64_t *col_idx, int64_t block_size,
                              int64_t *block_of, int64_t *n_blocks) {
  if (n < 0 || block_size < 1) return fail(TB_EINVAL, "grow_blocks: bad arguments");
  TB_TRY_BEGIN
  for (int64_t i = 0; i < n; ++i) block_of[i] = -1;
  std::vector<int64_t> heap;
  heap.reserve(256);
  auto cmp = std::greater<int64_t>();
  int64_t next_seed = 0, nb = 0;
  for (;;) {
    while (next_seed < n && block_of[next_seed] >= 0) ++next_seed;
    if (next_seed == n) break;
    const int64_t b = nb++;
    heap.clear();
    int64_t cur = next_seed, count = 0;
    for (;;) {
      block_of[cur] = b;
      if (++count == block_size) break;
      for (int64_t p = row_ptr[cur]; p < row_ptr[cur + 1]; ++p) {
        const int64_t j = col_idx[p];
        if (j != cur && block_of[j] < 0) {
          heap.push_back(j);
          std::push_heap(heap.begin(), heap.end(), cmp);
        }
      }
      int64_t nxt = -1;
      while (!heap.empty()) {
        std::pop_heap(heap.begin(), heap.end(), cmp);
        const int64_t v = heap.back();
        heap.pop_back();
        if (block_of[v] < 0) {
          nxt = v;
          break;
        }
      }
      if (nxt < 0) break;
      cur = nxt;
    }
  }
  *n_blocks = nb;
  return TB_OK;
  TB_TRY_END
}

// K/numba_backend.py:273-291 color_block_graph: first-fit over blocks in
// ascending id, mark[color] = b for every colored neighbouring block.
extern "C" int tb_color_block_graph(int64_t n, const int64_t *row_ptr,
                                    const int64_t *col_idx,
                                    const int64_t *block_of, int64_t n_blocks,
                                    const int64_t *block_ptr,
                                    const int64_t *block_nodes,
                                    int64_t *color_of_block) {
  (void)n;
  if (n_blocks < 0) return fail(TB_EINVAL, "color_block_graph: bad arguments");
  TB_TRY_BEGIN
  std::vector<int64_t> mark(n_blocks + 1, -1);
  for (int64_t b = 0; b < n_blocks; ++b) color_of_block[b] = -1;
  for (int64_t b = 0; b < n_blocks; ++b) {
    for (int64_t q = block_ptr[b]; q < block_ptr[b + 1]; ++q) {
      const int64_t i = block_nodes[q];
      for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
        const int64_t bj = block_of[col_idx[p]];
        if (bj != b) {
          const int64_t c = color_of_block[bj];
          if (c >= 0) mark[c] = b;
        }
      }
    }
    int64_t c = 0;
    while (mark[c] == b) ++c;
    color_of_block[b] = c;
  }
  return TB_OK;
  TB_TRY_END
}

// K/numba_backend.py:174-191 greedy_color: first-fit over nodes.
extern "C" int tb_greedy_color(int64_t n, const int64_t *row_ptr,
                               const int64_t *col_idx, int64_t *color_of) {
  if (n < 0) return fail(TB_EINVAL, "greedy_color: bad arguments");
  TB_TRY_BEGIN
  std::vector<int64_t> mark(n + 1, -1);
  for (int64_t i = 0; i < n; ++i) color_of[i] = -1;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int64_t j = col_idx[p];
      if (j != i) {
        const int64_t c = color_of[j];
        if (c >= 0) mark[c] = i;
      }
    }
    int64_t c = 0;
    while (mark[c] == i) ++c;
    color_of[i] = c;
  }
  return TB_OK;
  TB_TRY_END
}

// K/numba_backend.py:40-79 ic0_factor.  Row i ascending; for each strictly
// lower (i, j): s = l_ij - sum over the sorted merge of rows i (< p) and j of
// l_ia * l_jb, then l_ij = s * inv_d[j] (multiply by the reciprocal).  Pivot
// s = adiag[i] - sum l_ip^2; s <= 0 is a breakdown at row i.
extern "C" int tb_ic0_factor(int64_t n, const int64_t *lrp,
                             const int64_t *lci, double *lvals,
                             const double *adiag, double *d, double *inv_d,
                             int64_t *bad_row, double *bad_pivot) {
  if (n < 0) return fail(TB_EINVAL, "ic0_factor: bad arguments");
  for (int64_t i = 0; i < n; ++i) {
    d[i] = 0.0;
    inv_d[i] = 0.0;
  }
  *bad_row = -1;
  *bad_pivot = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t row_lo = lrp[i];
    for (int64_t p = row_lo; p < lrp[i + 1]; ++p) {
      const int64_t j = lci[p];
      double s = lvals[p];
      int64_t p1 = row_lo, e1 = p, p2 = lrp[j], e2 = lrp[j + 1];
      while (p1 < e1 && p2 < e2) {
        const int64_t c1 = lci[p1], c2 = lci[p2];
        if (c1 == c2) {
          const double prod = lvals[p1] * lvals[p2];
          s = s - prod;
          ++p1;
          ++p2;
        } else if (c1 < c2) {
          ++p1;
        } else {
          ++p2;
        }
      }
      lvals[p] = s * inv_d[j];
    }
    double s = adiag[i];
    for (int64_t p = row_lo; p < lrp[i + 1]; ++p) {
      const double sq = lvals[p] * lvals[p];
      s = s - sq;
    }
    if (!(s > 0.0)) {  // reference: `if s <= 0.0` (NaN passes through there)
      if (s <= 0.0) {
        *bad_row = i;
        *bad_pivot = s;
        return fail(TB_EIC_BREAKDOWN, "non-positive pivot %.6g at row %lld", s,
                    (long long)i);
      }
    }
    d[i] = std::sqrt(s);
    inv_d[i] = 1.0 / d[i];
  }
  return TB_OK;
}

// K/numba_backend.py:82-111 llt_on_pattern (verifier of the factor).
extern "C" int tb_llt_on_pattern(int64_t n, const int64_t *lrp,
                                 const int64_t *lci, const double *lvals,
                                 const double *d, double *low, double *diag) {
  if (n < 0) return fail(TB_EINVAL, "llt_on_pattern: bad arguments");
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = lrp[i]; p < lrp[i + 1]; ++p) {
      const int64_t j = lci[p];
      double s = lvals[p] * d[j];
      int64_t p1 = lrp[i], e1 = p, p2 = lrp[j], e2 = lrp[j + 1];
      while (p1 < e1 && p2 < e2) {
        const int64_t c1 = lci[p1], c2 = lci[p2];
        if (c1 == c2) {
          const double prod = lvals[p1] * lvals[p2];
          s = s + prod;
          ++p1;
          ++p2;
        } else if (c1 < c2) {
          ++p1;
        } else {
          ++p2;
        }
      }
      low[p] = s;
    }
    double s = d[i] * d[i];
    for (int64_t p = lrp[i]; p < lrp[i + 1]; ++p) {
      const double sq = lvals[p] * lvals[p];
      s = s + sq;
    }
    diag[i] = s;
  }
  return TB_OK;
}

// ---------------------------------------------------------------------------
// src/ordering.py:170-173: stable grouping of [0, n) by label (counting sort);
// members of each group come out in ascending index.
extern "C" int tb_group_by_label(int64_t n, const int64_t *label,
                                 int64_t n_labels, int64_t *ptr,
                                 int64_t *members) {
  if (n < 0 || n_labels < 0) return fail(TB_EINVAL, "group_by_label: bad arguments");
  for (int64_t g = 0; g <= n_labels; ++g) ptr[g] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t g = label[i];
    if (g < 0 || g >= n_labels) return fail(TB_EINVAL, "group_by_label: label out of range");
    ++ptr[g + 1];
  }
  for (int64_t g = 0; g < n_labels; ++g) ptr[g + 1] += ptr[g];
  TB_TRY_BEGIN
  std::vector<int64_t> next(ptr, ptr + n_labels);
  for (int64_t i = 0; i < n; ++i) members[next[label[i]]++] = i;
  return TB_OK;
  TB_TRY_END
}

// src/ordering.py:206-233 pad_colors, size pass.
extern "C" int tb_pad_colors_count(int64_t n_c, const int64_t *cbr, int64_t b_s,
                                   int64_t w, int64_t *nbar_of, int64_t *n_pad) {
  if (n_c < 0 || b_s < 1 || w < 1) return fail(TB_EINVAL, "pad_colors: bad arguments");
  int64_t total = 0;
  for (int64_t c = 0; c < n_c; ++c) {
    const int64_t cnt = cbr[c + 1] - cbr[c];
    const int64_t padded = (cnt + w - 1) / w * w;
    nbar_of[c] = padded / w;
    total += padded * b_s;
  }
  *n_pad = total;
  return TB_OK;
}

// src/ordering.py:206-233 pad_colors, fill pass (consumption-order dummies).
extern "C" int tb_pad_colors_fill(int64_t n, int64_t n_c, const int64_t *cbr,
                                  const int64_t *block_order,
                                  const int64_t *block_ptr,
                                  const int64_t *block_nodes, int64_t b_s,
                                  int64_t w, int64_t *slots, int64_t n_pad,
                                  int64_t *n_dummy) {
  if (n_c < 0 || b_s < 1 || w < 1) return fail(TB_EINVAL, "pad_colors: bad arguments");
  int64_t next_dummy = n, pos = 0;
  for (int64_t c = 0; c < n_c; ++c) {
    const int64_t lo = cbr[c], cnt = cbr[c + 1] - cbr[c];
    const int64_t padded = (cnt + w - 1) / w * w;
    for (int64_t k = 0; k < padded; ++k) {
      int64_t fill = b_s;
      if (k < cnt) {
        const int64_t blk = block_order[lo + k];
        const int64_t m0 = block_ptr[blk], m1 = block_ptr[blk + 1];
        if (m1 - m0 > b_s || pos + (m1 - m0) > n_pad)
          return fail(TB_EINVAL, "pad_colors: block larger than b_s");
        for (int64_t q = m0; q < m1; ++q) slots[pos++] = block_nodes[q];
        fill = b_s - (m1 - m0);
      }
      if (pos + fill > n_pad) return fail(TB_EINVAL, "pad_colors: size mismatch");
      for (int64_t f = 0; f < fill; ++f) slots[pos++] = next_dummy++;
    }
  }
  if (pos != n_pad) return fail(TB_EINVAL, "pad_colors: size mismatch");
  *n_dummy = next_dummy - n;
  return TB_OK;
}

// src/ordering.py:242-257: padded_new_of_old[slots[p]] = p; within each
// level-1 block local position m*b_s + j moves to j*w + m.
extern "C" int tb_hbmc_compose(int64_t n_pad, const int64_t *slots, int64_t b_s,
                               int64_t w, int64_t *padded_new_of_old,
                               int64_t *composed_new_of_old) {
  if (n_pad < 0 || b_s < 1 || w < 1) return fail(TB_EINVAL, "hbmc_compose: bad arguments");
  const int64_t span = b_s * w;
  if (n_pad % span) return fail(TB_EINVAL, "hbmc_compose: n_pad not a multiple of b_s*w");
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < n_pad; ++p) {
    const int64_t s = slots[p];
    const int64_t K = p / span, q = p - K * span;
    const int64_t m = q / b_s, j = q - m * b_s;
    padded_new_of_old[s] = p;
    composed_new_of_old[s] = K * span + j * w + m;
  }
  return TB_OK;
}

// ---------------------------------------------------------------------------
// Row-wise (column, value) sort used by the CSR builders.  Rows are short;
// insertion sort for small rows, std::sort beyond.
static inline void sort_row(int64_t *c, double *v, int64_t len) {
  if (len <= 32) {
    for (int64_t a = 1; a < len; ++a) {
      const int64_t ck = c[a];
      const double vk = v[a];
      int64_t b = a - 1;
      while (b >= 0 && c[b] > ck) {
        c[b + 1] = c[b];
        v[b + 1] = v[b];
        --b;
      }
      c[b + 1] = ck;
      v[b + 1] = vk;
    }
    return;
  }
  std::vector<std::pair<int64_t, double>> tmp(len);
  for (int64_t a = 0; a < len; ++a) tmp[a] = {c[a], v[a]};
  std::stable_sort(tmp.begin(), tmp.end(),
                   [](const std::pair<int64_t, double> &x,
                      const std::pair<int64_t, double> &y) { return x.first < y.first; });
  for (int64_t a = 0; a < len; ++a) {
    c[a] = tmp[a].first;
    v[a] = tmp[a].second;
  }
}

// src/matrix.py:168-197 coo_to_csr: lexsort by (row, col); duplicates error.
extern "C" int tb_coo_to_csr(int64_t n, int64_t nnz, const int64_t *row,
                             const int64_t *col, const double *val,
                             int64_t *row_ptr, int64_t *col_idx, double *vals,
                             int64_t *dup_row, int64_t *dup_col) {
  if (n < 0 || nnz < 0) return fail(TB_EINVAL, "coo_to_csr: bad arguments");
  *dup_row = -1;
  *dup_col = -1;
  for (int64_t i = 0; i <= n; ++i) row_ptr[i] = 0;
  for (int64_t e = 0; e < nnz; ++e) {
    const int64_t r = row[e], c = col[e];
    if (r < 0 || r >= n || c < 0 || c >= n)
      return fail(TB_EINVAL, "coo_to_csr: index out of range at entry %lld", (long long)e);
    ++row_ptr[r + 1];
  }
  for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
  TB_TRY_BEGIN
  {
    std::vector<int64_t> next(row_ptr, row_ptr + n);
    for (int64_t e = 0; e < nnz; ++e) {
      const int64_t d = next[row[e]]++;
      col_idx[d] = col[e];
      vals[d] = val[e];
    }
  }
  int64_t first_dup = -1;
#pragma omp parallel
  {
    int64_t my_dup = -1;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
      const int64_t lo = row_ptr[i], len = row_ptr[i + 1] - lo;
      sort_row(col_idx + lo, vals + lo, len);
      for (int64_t a = 1; a < len; ++a)
        if (col_idx[lo + a] == col_idx[lo + a - 1]) {
          if (my_dup < 0 || i < my_dup) my_dup = i;
          break;
        }
    }
#pragma omp critical
    if (my_dup >= 0 && (first_dup < 0 || my_dup < first_dup)) first_dup = my_dup;
  }
  if (first_dup >= 0) {
    const int64_t lo = row_ptr[first_dup], hi = row_ptr[first_dup + 1];
    for (int64_t a = lo + 1; a < hi; ++a)
      if (col_idx[a] == col_idx[a - 1]) {
        *dup_row = first_dup;
        *dup_col = col_idx[a];
        break;
      }
    return fail(TB_EDUP, "duplicate entry at (%lld, %lld)", (long long)*dup_row,
                (long long)*dup_col);
  }
  return TB_OK;
  TB_TRY_END
}

// src/matrix.py:293-304 permute_system: (i, j, v) -> (q[i], q[j], v), CSR.
extern "C" int tb_permute_csr(int64_t n, const int64_t *row_ptr,
                              const int64_t *col_idx, const double *vals,
                              const int64_t *q, int64_t *rp_out,
                              int64_t *col_out, double *vals_out) {
  if (n < 0) return fail(TB_EINVAL, "permute_csr: bad arguments");
  for (int64_t i = 0; i <= n; ++i) rp_out[i] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t qi = q[i];
    if (qi < 0 || qi >= n) return fail(TB_EINVAL, "permute_csr: permutation out of range");
    rp_out[qi + 1] = row_ptr[i + 1] - row_ptr[i];
  }
  for (int64_t i = 0; i < n; ++i) rp_out[i + 1] += rp_out[i];
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = row_ptr[i], len = row_ptr[i + 1] - lo;
    const int64_t d = rp_out[q[i]];
    for (int64_t a = 0; a < len; ++a) {
      col_out[d + a] = q[col_idx[lo + a]];
      vals_out[d + a] = vals[lo + a];
    }
    sort_row(col_out + d, vals_out + d, len);
  }
  return TB_OK;
}

// src/matrix.py:205-208 csr_transpose (stable counting sort by column, so
// every output row is ascending in the original row index).
extern "C" int tb_csr_transpose(int64_t n, const int64_t *row_ptr,
                                const int64_t *col_idx, const double *vals,
                                int64_t *rp_out, int64_t *col_out,
                                double *vals_out) {
  if (n < 0) return fail(TB_EINVAL, "csr_transpose: bad arguments");
  const int64_t nnz = row_ptr[n];
  for (int64_t i = 0; i <= n; ++i) rp_out[i] = 0;
  for (int64_t p = 0; p < nnz; ++p) ++rp_out[col_idx[p] + 1];
  for (int64_t i = 0; i < n; ++i) rp_out[i + 1] += rp_out[i];
  TB_TRY_BEGIN
  std::vector<int64_t> next(rp_out, rp_out + n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int64_t d = next[col_idx[p]]++;
      col_out[d] = i;
      vals_out[d] = vals[p];
    }
  return TB_OK;
  TB_TRY_END
}

// Setup helpers over a CSR pattern with sorted columns (OpenMP over rows):
// the diagonal slot of every row (-1 if absent), whether the pattern is
// structurally symmetric (every (i, j) has (j, i)), and the strictly lower
// / upper part as a new CSR (src/precond.py:163-169).  The numpy versions
// allocate nnz-sized temporaries several times; at config 5 (938M entries)
// these three dominated the host setup.
extern "C" int tb_csr_diag_ptr(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                               int64_t *diag_out) {
  if (n < 0) return fail(TB_EINVAL, "csr_diag_ptr: bad arguments");
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < n; ++i) {   // linear scan: columns need not be sorted
    int64_t d = -1;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
      if (col_idx[p] == i) {
        d = p;
        break;
      }
    diag_out[i] = d;
  }
  return TB_OK;
}

extern "C" int tb_csr_is_symmetric(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                                   int32_t *symmetric) {
  if (n < 0) return fail(TB_EINVAL, "csr_is_symmetric: bad arguments");
  int bad = 0;
#pragma omp parallel for schedule(static, 4096) reduction(| : bad)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1] && !bad; ++p) {
      const int64_t j = col_idx[p];
      if (j < 0 || j >= n) { bad = 1; break; }
      const int64_t *b = col_idx + row_ptr[j], *e = col_idx + row_ptr[j + 1];
      const int64_t *q = std::lower_bound(b, e, i);
      if (q == e || *q != i) bad = 1;
    }
  }
  *symmetric = bad ? 0 : 1;
  return TB_OK;
}

// upper = 0: strictly lower part; 1: strictly upper.  row_out [n+1]; the
// caller sizes col_out / val_out with tb_csr_tri_count.
extern "C" int tb_csr_tri_count(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                                int32_t upper, int64_t *row_out) {
  if (n < 0) return fail(TB_EINVAL, "csr_tri_count: bad arguments");
  row_out[0] = 0;
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
      c += upper ? (col_idx[p] > i) : (col_idx[p] < i);
    row_out[i + 1] = c;
  }
  for (int64_t i = 0; i < n; ++i) row_out[i + 1] += row_out[i];
  return TB_OK;
}

extern "C" int tb_csr_tri_fill(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                               const double *vals, int32_t upper, const int64_t *row_out,
                               int64_t *col_out, double *val_out) {
  if (n < 0) return fail(TB_EINVAL, "csr_tri_fill: bad arguments");
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < n; ++i) {
    int64_t d = row_out[i];
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
      if (upper ? (col_idx[p] > i) : (col_idx[p] < i)) {
        col_out[d] = col_idx[p];
        val_out[d] = vals[p];
        ++d;
      }
  }
  return TB_OK;
}

// src/matrix.py:239-261 csr_to_sell fill: entry t of row i at
// slice_ptr[i / w] + (i % w) + w * t; padding = (own row, 0.0).
extern "C" int tb_csr_to_sell_fill(int64_t n, const int64_t *row_ptr,
                                   const int64_t *col_idx, const double *vals,
                                   int64_t width, int64_t n_slices,
                                   const int64_t *slice_ptr, int64_t *col64,
                                   int32_t *col32, double *vals_out) {
  if (n < 0 || width < 1 || n_slices * width < n)
    return fail(TB_EINVAL, "csr_to_sell: bad arguments");
  if (col32 && n_slices * width > INT32_MAX)
    return fail(TB_EINVAL, "csr_to_sell: rows exceed int32 columns");
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t s = 0; s < n_slices; ++s) {
    const int64_t base = s * width, off = slice_ptr[s];
    const int64_t len = (slice_ptr[s + 1] - off) / width;
    for (int64_t t = 0; t < len; ++t)
      for (int64_t j = 0; j < width; ++j) {
        const int64_t pos = off + t * width + j;
        if (col64) col64[pos] = base + j;
        if (col32) col32[pos] = (int32_t)(base + j);
        vals_out[pos] = 0.0;
      }
    for (int64_t j = 0; j < width; ++j) {
      const int64_t i = base + j;
      if (i >= n) break;
      const int64_t lo = row_ptr[i], cnt = row_ptr[i + 1] - lo;
      for (int64_t t = 0; t < cnt; ++t) {
        const int64_t pos = off + j + width * t;
        if (col64) col64[pos] = col_idx[lo + t];
        if (col32) col32[pos] = (int32_t)col_idx[lo + t];
        vals_out[pos] = vals[lo + t];
      }
    }
  }
  return TB_OK;
}

// K/numba_backend.py:16-23 spmv_csr on the host (forms b = A x* once).
extern "C" int tb_spmv_csr_host(int64_t n, const int64_t *row_ptr,
                                const int64_t *col_idx, const double *vals,
                                const double *x, double *out) {
  if (n < 0) return fail(TB_EINVAL, "spmv_csr_host: bad arguments");
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const double prod = vals[p] * x[col_idx[p]];
      s = s + prod;
    }
    out[i] = s;
  }
  return TB_OK;
}

// Dependency levels of a triangular CSR factor (forward: L, rows ascending;
// backward: U, rows descending).  Rows of one level are mutually independent,
// so a level-by-level device sweep performs exactly the arithmetic of the
// sequential substitution (K/numba_backend.py:114-129) for every row.
extern "C" int tb_level_schedule(int64_t n, const int64_t *rp, const int64_t *ci,
                                 int forward, int64_t *level, int64_t *n_levels) {
  if (n < 0) return fail(TB_EINVAL, "level_schedule: bad arguments");
  int64_t top = -1;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = forward ? k : n - 1 - k;
    int64_t lv = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t j = ci[p];
      if (forward ? j >= i : j <= i)
        return fail(TB_EINVAL, "level_schedule: factor is not strictly triangular at row %lld",
                    (long long)i);
      if (level[j] + 1 > lv) lv = level[j] + 1;
    }
    level[i] = lv;
    if (lv > top) top = lv;
  }
  *n_levels = top + 1;
  return TB_OK;
}
