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

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
