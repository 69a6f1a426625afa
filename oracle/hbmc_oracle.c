/*
 * hbmc_oracle.c -- CPU ORACLE (test infrastructure, NOT the product).
 *
 * Plain-C restatement of the reference's numba kernel seam
 * (/root/reference/pkg/src/trilab/_kernels/numba_backend.py, cited K:line)
 * and of the reference's fork-join HBMC sweep driver
 * (/root/reference/pkg/src/trilab/precond.py:153-160,377-392, cited P:line).
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library, and only as the checker / the timed CPU reference path.
 *
 * Pinned against the reference's own outputs: tests/golden/ (npz files) were
 * produced by importing the reference `trilab` (tests/golden/make_golden.py)
 * and tests/test_oracle.py checks this file against every one of them.
 *
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off): the
 * reference's numba kernels round every multiply and subtract separately.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;

/* K:16-23 */
void or_spmv_csr(i64 n, const i64 *row_ptr, const i64 *col_idx, const double *vals,
                 const double *x, double *out) {
    for (i64 i = 0; i < n; ++i) {
        double s = 0.0;
        for (i64 p = row_ptr[i]; p < row_ptr[i + 1]; ++p) s += vals[p] * x[col_idx[p]];
        out[i] = s;
    }
}

/* K:26-37 */
void or_spmv_sell(i64 n_slices, const i64 *slice_ptr, const i64 *slice_len,
                  const i64 *col_idx, const double *vals, i64 w, const double *x,
                  double *out) {
    for (i64 s = 0; s < n_slices; ++s) {
        i64 base = s * w, off = slice_ptr[s];
        for (i64 j = 0; j < w; ++j) out[base + j] = 0.0;
        for (i64 t = 0; t < slice_len[s]; ++t) {
            for (i64 j = 0; j < w; ++j) out[base + j] += vals[off + j] * x[col_idx[off + j]];
            off += w;
        }
    }
}

/* Row-parallel variant of K:26-37 (same per-row arithmetic) for the CPU
 * baseline's "all host threads" leg. */
void or_spmv_sell_par(i64 n_slices, const i64 *slice_ptr, const i64 *slice_len,
                      const i64 *col_idx, const double *vals, i64 w, const double *x,
                      double *out, int threads) {
#pragma omp parallel for schedule(static) num_threads(threads)
    for (i64 s = 0; s < n_slices; ++s) {
        i64 base = s * w, off = slice_ptr[s];
        for (i64 j = 0; j < w; ++j) out[base + j] = 0.0;
        for (i64 t = 0; t < slice_len[s]; ++t) {
            for (i64 j = 0; j < w; ++j) out[base + j] += vals[off + j] * x[col_idx[off + j]];
            off += w;
        }
    }
}

/* K:40-79.  Returns bad_row (-1 on success); *pivot set on failure. */
i64 or_ic0_factor(i64 n, const i64 *lrp, const i64 *lci, double *lvals,
                  const double *adiag, double *d, double *inv_d, double *pivot) {
    for (i64 i = 0; i < n; ++i) { d[i] = 0.0; inv_d[i] = 0.0; }
    *pivot = 0.0;
    for (i64 i = 0; i < n; ++i) {
        for (i64 p = lrp[i]; p < lrp[i + 1]; ++p) {
            i64 j = lci[p];
            double s = lvals[p];
            i64 p1 = lrp[i], e1 = p, p2 = lrp[j], e2 = lrp[j + 1];
            while (p1 < e1 && p2 < e2) {
                i64 c1 = lci[p1], c2 = lci[p2];
                if (c1 == c2) { s -= lvals[p1] * lvals[p2]; ++p1; ++p2; }
                else if (c1 < c2) ++p1;
                else ++p2;
            }
            lvals[p] = s * inv_d[j];
        }
        double s = adiag[i];
        for (i64 p = lrp[i]; p < lrp[i + 1]; ++p) s -= lvals[p] * lvals[p];
        if (s <= 0.0) { *pivot = s; return i; }
        d[i] = sqrt(s);
        inv_d[i] = 1.0 / d[i];
    }
    return -1;
}

/* K:114-120 */
void or_fwd_csr_range(const i64 *lrp, const i64 *lci, const double *lvals,
                      const double *inv_d, const double *r, double *y, i64 start, i64 end) {
    for (i64 i = start; i < end; ++i) {
        double s = r[i];
        for (i64 p = lrp[i]; p < lrp[i + 1]; ++p) s -= lvals[p] * y[lci[p]];
        y[i] = s * inv_d[i];
    }
}

/* K:123-129 */
void or_bwd_csr_range(const i64 *urp, const i64 *uci, const double *uvals,
                      const double *inv_d, const double *y, double *z, i64 start, i64 end) {
    for (i64 i = end - 1; i >= start; --i) {
        double s = y[i];
        for (i64 p = urp[i]; p < urp[i + 1]; ++p) s -= uvals[p] * z[uci[p]];
        z[i] = s * inv_d[i];
    }
}

/* K:132-153 */
void or_fwd_sell_range(const i64 *slice_ptr, const i64 *slice_len, const i64 *col_idx,
                       const double *vals, const double *inv_d, const double *r, double *y,
                       i64 w, i64 b_s, i64 k0, i64 k1) {
    for (i64 k = k0; k < k1; ++k) {
        i64 base = k * b_s * w;
        for (i64 l = 0; l < b_s; ++l) {
            i64 row0 = base + l * w, sid = row0 / w, off = slice_ptr[sid];
            for (i64 j = 0; j < w; ++j) y[row0 + j] = r[row0 + j];
            for (i64 t = 0; t < slice_len[sid]; ++t) {
                for (i64 j = 0; j < w; ++j) y[row0 + j] -= vals[off + j] * y[col_idx[off + j]];
                off += w;
            }
            for (i64 j = 0; j < w; ++j) y[row0 + j] *= inv_d[row0 + j];
        }
    }
}

/* K:156-171 */
void or_bwd_sell_range(const i64 *slice_ptr, const i64 *slice_len, const i64 *col_idx,
                       const double *vals, const double *inv_d, const double *y, double *z,
                       i64 w, i64 b_s, i64 k0, i64 k1) {
    for (i64 k = k1 - 1; k >= k0; --k) {
        i64 base = k * b_s * w;
        for (i64 l = b_s - 1; l >= 0; --l) {
            i64 row0 = base + l * w, sid = row0 / w, off = slice_ptr[sid];
            for (i64 j = 0; j < w; ++j) z[row0 + j] = y[row0 + j];
            for (i64 t = 0; t < slice_len[sid]; ++t) {
                for (i64 j = 0; j < w; ++j) z[row0 + j] -= vals[off + j] * z[col_idx[off + j]];
                off += w;
            }
            for (i64 j = 0; j < w; ++j) z[row0 + j] *= inv_d[row0 + j];
        }
    }
}

/* P:153-160 _chunk_bounds + P:377-392 _hbmc_sweep: per color, the level-1
 * range is split into `threads` contiguous chunks run concurrently; the end
 * of the parallel region is the per-color fork-join barrier. */
void or_hbmc_sweep(int forward, const i64 *slice_ptr, const i64 *slice_len,
                   const i64 *col_idx, const double *vals, const double *inv_d,
                   const double *src, double *dst, i64 w, i64 b_s, i64 n_c,
                   const i64 *color_lvl1_ranges, int threads) {
    for (i64 idx = 0; idx < n_c; ++idx) {
        i64 c = forward ? idx : n_c - 1 - idx;
        i64 lo = color_lvl1_ranges[c], hi = color_lvl1_ranges[c + 1], cnt = hi - lo;
        if (cnt <= 0) continue;
        i64 parts = threads < 1 ? 1 : threads;
        if (parts > cnt) parts = cnt;
#pragma omp parallel for schedule(static, 1) num_threads((int)parts)
        for (i64 i = 0; i < parts; ++i) {
            i64 k0 = lo + (cnt * i) / parts, k1 = lo + (cnt * (i + 1)) / parts;
            if (forward)
                or_fwd_sell_range(slice_ptr, slice_len, col_idx, vals, inv_d, src, dst, w, b_s, k0, k1);
            else
                or_bwd_sell_range(slice_ptr, slice_len, col_idx, vals, inv_d, src, dst, w, b_s, k0, k1);
        }
    }
}

/* K:174-191 */
void or_greedy_color(i64 n, const i64 *row_ptr, const i64 *col_idx, i64 *color_of) {
    i64 *mark = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    for (i64 i = 0; i <= n; ++i) mark[i] = -1;
    for (i64 i = 0; i < n; ++i) color_of[i] = -1;
    for (i64 i = 0; i < n; ++i) {
        for (i64 p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            i64 j = col_idx[p];
            if (j != i && color_of[j] >= 0) mark[color_of[j]] = i;
        }
        i64 c = 0;
        while (mark[c] == i) ++c;
        color_of[i] = c;
    }
    free(mark);
}

/* K:194-206 */
static i64 heap_push(i64 *heap, i64 size, i64 val) {
    heap[size] = val;
    i64 i = size;
    while (i > 0) {
        i64 parent = (i - 1) >> 1;
        if (heap[parent] <= heap[i]) break;
        i64 tmp = heap[parent]; heap[parent] = heap[i]; heap[i] = tmp;
        i = parent;
    }
    return size + 1;
}

/* K:209-229 */
static i64 heap_pop(i64 *heap, i64 size, i64 *top) {
    *top = heap[0];
    size -= 1;
    heap[0] = heap[size];
    i64 i = 0;
    for (;;) {
        i64 left = 2 * i + 1, right = left + 1, smallest = i;
        if (left < size && heap[left] < heap[smallest]) smallest = left;
        if (right < size && heap[right] < heap[smallest]) smallest = right;
        if (smallest == i) break;
        i64 tmp = heap[smallest]; heap[smallest] = heap[i]; heap[i] = tmp;
        i = smallest;
    }
    return size;
}

/* K:232-270.  Returns n_blocks. */
i64 or_grow_blocks(i64 n, const i64 *row_ptr, const i64 *col_idx, i64 block_size,
                   i64 *block_of) {
    i64 *heap = (i64 *)malloc(sizeof(i64) * (size_t)(row_ptr[n] + 1));
    for (i64 i = 0; i < n; ++i) block_of[i] = -1;
    i64 next_seed = 0, n_blocks = 0;
    for (;;) {
        while (next_seed < n && block_of[next_seed] >= 0) ++next_seed;
        if (next_seed == n) break;
        i64 b = n_blocks++, hsize = 0, cur = next_seed, count = 0;
        for (;;) {
            block_of[cur] = b;
            if (++count == block_size) break;
            for (i64 p = row_ptr[cur]; p < row_ptr[cur + 1]; ++p) {
                i64 j = col_idx[p];
                if (j != cur && block_of[j] < 0) hsize = heap_push(heap, hsize, j);
            }
            i64 nxt = -1;
            while (hsize > 0) {
                i64 v;
                hsize = heap_pop(heap, hsize, &v);
                if (block_of[v] < 0) { nxt = v; break; }
            }
            if (nxt < 0) break;
            cur = nxt;
        }
    }
    free(heap);
    return n_blocks;
}

/* K:273-291 */
void or_color_block_graph(const i64 *row_ptr, const i64 *col_idx, const i64 *block_of,
                          i64 n_blocks, const i64 *block_ptr, const i64 *block_nodes,
                          i64 *color_of_block) {
    i64 *mark = (i64 *)malloc(sizeof(i64) * (size_t)(n_blocks + 1));
    for (i64 i = 0; i <= n_blocks; ++i) mark[i] = -1;
    for (i64 b = 0; b < n_blocks; ++b) color_of_block[b] = -1;
    for (i64 b = 0; b < n_blocks; ++b) {
        for (i64 q = block_ptr[b]; q < block_ptr[b + 1]; ++q) {
            i64 i = block_nodes[q];
            for (i64 p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
                i64 bj = block_of[col_idx[p]];
                if (bj != b && color_of_block[bj] >= 0) mark[color_of_block[bj]] = b;
            }
        }
        i64 c = 0;
        while (mark[c] == b) ++c;
        color_of_block[b] = c;
    }
    free(mark);
}

/* ------------------------------------------------------------------ host
 * Sparse-matrix plumbing of the reference's Python layer restated in C so
 * the oracle can build the 512^3 config (N = 134M, nnz = 938M) inside the
 * GPU box's host RAM; each is equivalent to the numpy code it cites. */

/* Row-parallel K:16-23 (same per-row arithmetic, rows independent). */
void or_spmv_csr_par(i64 n, const i64 *row_ptr, const i64 *col_idx, const double *vals,
                     const double *x, double *out, int threads) {
#pragma omp parallel for schedule(static, 4096) num_threads(threads)
    for (i64 i = 0; i < n; ++i) {
        double s = 0.0;
        for (i64 p = row_ptr[i]; p < row_ptr[i + 1]; ++p) s += vals[p] * x[col_idx[p]];
        out[i] = s;
    }
}

typedef struct { i64 c; double v; } cv_t;

static int cv_cmp(const void *a, const void *b) {
    i64 x = ((const cv_t *)a)->c, y = ((const cv_t *)b)->c;
    return (x > y) - (x < y);
}

/* Sort one row's (col, val) pairs by column: insertion sort (stable) for the
 * short rows of the BASELINE matrices, qsort for long rows.  Returns the
 * first position whose column equals its predecessor's, or -1. */
static i64 sort_row(i64 *ci, double *v, i64 len) {
    if (len <= 64) {
        for (i64 a = 1; a < len; ++a) {
            i64 c = ci[a];
            double x = v[a];
            i64 b = a - 1;
            while (b >= 0 && ci[b] > c) { ci[b + 1] = ci[b]; v[b + 1] = v[b]; --b; }
            ci[b + 1] = c;
            v[b + 1] = x;
        }
    } else {
        cv_t *t = (cv_t *)malloc(sizeof(cv_t) * (size_t)len);
        for (i64 a = 0; a < len; ++a) { t[a].c = ci[a]; t[a].v = v[a]; }
        qsort(t, (size_t)len, sizeof(cv_t), cv_cmp);
        for (i64 a = 0; a < len; ++a) { ci[a] = t[a].c; v[a] = t[a].v; }
        free(t);
    }
    for (i64 a = 1; a < len; ++a)
        if (ci[a] == ci[a - 1]) return a;
    return -1;
}

/* src/matrix.py:168-197 coo_to_csr (ensure_diagonal=False): entries bucketed
 * by row, then each row sorted by column == np.lexsort((col, row)); a
 * duplicate (row, col) is an error.  Returns -1, or the CSR position of the
 * first duplicate (its row / column are then rp / ci at that position). */
i64 or_coo_to_csr(i64 n, i64 nnz, const i64 *row, const i64 *col, const double *val,
                  i64 *rp, i64 *ci, double *v, int threads) {
    for (i64 i = 0; i <= n; ++i) rp[i] = 0;
    for (i64 e = 0; e < nnz; ++e) rp[row[e] + 1]++;
    for (i64 i = 0; i < n; ++i) rp[i + 1] += rp[i];
    i64 *pos = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    memcpy(pos, rp, sizeof(i64) * (size_t)(n + 1));
    for (i64 e = 0; e < nnz; ++e) {
        i64 p = pos[row[e]]++;
        ci[p] = col[e];
        v[p] = val[e];
    }
    free(pos);
    i64 dup = -1;
#pragma omp parallel for schedule(dynamic, 8192) num_threads(threads)
    for (i64 i = 0; i < n; ++i) {
        i64 d = sort_row(ci + rp[i], v + rp[i], rp[i + 1] - rp[i]);
        if (d >= 0) {
#pragma omp critical
            if (dup < 0 || rp[i] + d < dup) dup = rp[i] + d;
        }
    }
    return dup;
}

/* src/matrix.py:293-304 permute_system's matrix part: entry (i, j) of A
 * moves to (q[i], q[j]); rows re-sorted by column (the reference's COO ->
 * lexsort).  Rows are independent. */
void or_permute_csr(i64 n, const i64 *rp, const i64 *ci, const double *v, const i64 *q,
                    i64 *rp_out, i64 *ci_out, double *v_out, int threads) {
    rp_out[0] = 0;
    for (i64 i = 0; i < n; ++i) rp_out[q[i] + 1] = rp[i + 1] - rp[i];
    for (i64 i = 0; i < n; ++i) rp_out[i + 1] += rp_out[i];
#pragma omp parallel for schedule(dynamic, 8192) num_threads(threads)
    for (i64 i = 0; i < n; ++i) {
        i64 d = rp_out[q[i]], len = rp[i + 1] - rp[i];
        for (i64 t = 0; t < len; ++t) {
            ci_out[d + t] = q[ci[rp[i] + t]];
            v_out[d + t] = v[rp[i] + t];
        }
        sort_row(ci_out + d, v_out + d, len);
    }
}

/* src/matrix.py:205-208 csr_transpose: bucket by column, rows visited in
 * ascending order, so every output row is already column-sorted (== the
 * lexsort of (row, col) after the swap). */
void or_csr_transpose(i64 n, const i64 *rp, const i64 *ci, const double *v, i64 *rp_out,
                      i64 *ci_out, double *v_out) {
    for (i64 i = 0; i <= n; ++i) rp_out[i] = 0;
    for (i64 p = 0; p < rp[n]; ++p) rp_out[ci[p] + 1]++;
    for (i64 i = 0; i < n; ++i) rp_out[i + 1] += rp_out[i];
    i64 *pos = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
    memcpy(pos, rp_out, sizeof(i64) * (size_t)(n + 1));
    for (i64 i = 0; i < n; ++i)
        for (i64 p = rp[i]; p < rp[i + 1]; ++p) {
            i64 d = pos[ci[p]]++;
            ci_out[d] = i;
            v_out[d] = v[p];
        }
    free(pos);
}

/* src/precond.py:163-169 _strict_tri(upper=False) plus A.diagonal()
 * (src/matrix.py:78-81: 0.0 where a row stores no diagonal).  Pass 1
 * (lrp == NULL is not allowed): counts into lrp; pass 2 (fill != 0): fill. */
void or_split_lower(i64 n, const i64 *rp, const i64 *ci, const double *v, i64 *lrp,
                    i64 *lci, double *lv, double *diag, int fill, int threads) {
    if (!fill) {
        lrp[0] = 0;
#pragma omp parallel for schedule(static, 8192) num_threads(threads)
        for (i64 i = 0; i < n; ++i) {
            i64 c = 0;
            double dg = 0.0;
            for (i64 p = rp[i]; p < rp[i + 1]; ++p) {
                if (ci[p] < i) ++c;
                else if (ci[p] == i) dg = v[p];
            }
            lrp[i + 1] = c;
            diag[i] = dg;
        }
        for (i64 i = 0; i < n; ++i) lrp[i + 1] += lrp[i];
        return;
    }
#pragma omp parallel for schedule(static, 8192) num_threads(threads)
    for (i64 i = 0; i < n; ++i) {
        i64 d = lrp[i];
        for (i64 p = rp[i]; p < rp[i + 1]; ++p)
            if (ci[p] < i) { lci[d] = ci[p]; lv[d] = v[p]; ++d; }
    }
}

/* src/matrix.py:211-261 csr_to_sell fill (slice_ptr / slice_len computed by
 * the caller): padding slots hold column = own row and value 0.0; entry t
 * of row i at slice_ptr[i / w] + i % w + w * t. */
void or_csr_to_sell_fill(i64 n, i64 n_slices, i64 w, const i64 *rp, const i64 *ci,
                         const double *v, const i64 *slice_ptr, const i64 *slice_len,
                         i64 *col_out, double *val_out, int threads) {
#pragma omp parallel for schedule(static, 1024) num_threads(threads)
    for (i64 s = 0; s < n_slices; ++s) {
        for (i64 t = 0; t < slice_len[s]; ++t)
            for (i64 j = 0; j < w; ++j) {
                col_out[slice_ptr[s] + t * w + j] = s * w + j;
                val_out[slice_ptr[s] + t * w + j] = 0.0;
            }
        for (i64 j = 0; j < w; ++j) {
            i64 i = s * w + j;
            if (i >= n) break;
            for (i64 p = rp[i]; p < rp[i + 1]; ++p) {
                col_out[slice_ptr[s] + j + w * (p - rp[i])] = ci[p];
                val_out[slice_ptr[s] + j + w * (p - rp[i])] = v[p];
            }
        }
    }
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
