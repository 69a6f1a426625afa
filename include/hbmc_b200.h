/*
 * hbmc_b200.h -- C ABI of the B200-native HBMC-ordered ICCG hot path.
 *
 * One shared library (paper_1908_00741_b200/libhbmc_b200.so) exports every
 * entry point below.  Plain pointers and sizes only: index arrays are
 * int64_t on the host (the reference's dtype, numpy int64) and int32_t on the
 * device; values are IEEE double everywhere.  Every function returns an int
 * status (TB_OK == 0); tb_last_error() returns a thread-local message for the
 * last failing call on the calling thread.
 *
 * The reference interface each entry point replaces is cited as
 *   K/ = /root/reference/pkg/src/trilab/_kernels/   (numba kernel seam)
 *   src/ = /root/reference/pkg/src/trilab/          (Python wrappers)
 * Host builders are bit-exact restatements; device operators are bit-exact
 * for the substitutions and the SpMV (non-contracted mul/sub in the same
 * per-row order), see DESIGN.md.
 */
#ifndef HBMC_B200_H
#define HBMC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define TB_OK 0
#define TB_EINVAL 1          /* argument / shape error -> ValueError          */
#define TB_EIC_BREAKDOWN 2   /* non-positive pivot -> IcBreakdownError         */
#define TB_ECG_BREAKDOWN 3   /* p.Ap <= 0 -> CgBreakdownError                  */
#define TB_ECUDA 4           /* CUDA runtime failure (message has the detail)  */
#define TB_ENOMEM 5          /* host or device allocation failure              */
#define TB_EDUP 6            /* duplicate (row, col) in COO input -> ValueError*/
#define TB_ENODEV 7          /* no CUDA device visible                         */

const char *tb_last_error(void);
int tb_abi_version(void);            /* bumps on any signature change */

/* =========================================================================
 * Host construction kernels.  Same arguments, same outputs, same
 * determinism as the numba kernels they replace.
 * ========================================================================= */

/* K/numba_backend.py:232-270 grow_blocks(row_ptr, col_idx, block_size)
 * -> block_of[n] (caller-allocated), *n_blocks. */
int tb_grow_blocks(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                   int64_t block_size, int64_t *block_of, int64_t *n_blocks);

/* K/numba_backend.py:273-291 color_block_graph(row_ptr, col_idx, block_of,
 * n_blocks, block_ptr, block_nodes) -> color_of_block[n_blocks]. */
int tb_color_block_graph(int64_t n, const int64_t *row_ptr,
                         const int64_t *col_idx, const int64_t *block_of,
                         int64_t n_blocks, const int64_t *block_ptr,
                         const int64_t *block_nodes, int64_t *color_of_block);

/* K/numba_backend.py:174-191 greedy_color(row_ptr, col_idx) -> color_of[n]. */
int tb_greedy_color(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                    int64_t *color_of);

/* K/numba_backend.py:40-79 ic0_factor(lrp, lci, lvals, adiag).
 * lvals is overwritten with the factor; d, inv_d are caller-allocated [n].
 * On a non-positive pivot returns TB_EIC_BREAKDOWN with *bad_row / *bad_pivot
 * set (bad_row = -1 on success). */
int tb_ic0_factor(int64_t n, const int64_t *lrp, const int64_t *lci,
                  double *lvals, const double *adiag, double *d, double *inv_d,
                  int64_t *bad_row, double *bad_pivot);

/* K/numba_backend.py:82-111 llt_on_pattern(lrp, lci, lvals, d)
 * -> low[nnz], diag[n] (caller-allocated). */
int tb_llt_on_pattern(int64_t n, const int64_t *lrp, const int64_t *lci,
                      const double *lvals, const double *d, double *low,
                      double *diag);

/* =========================================================================
 * Host bulk builders: the Python per-row / per-block loops of the reference
 * (src/ordering.py, src/matrix.py) as linear-time native passes.
 * ========================================================================= */

/* src/ordering.py:170-173 build_blocks: members of every block in ascending
 * original index.  block_ptr[n_blocks+1], block_nodes[n]. */
int tb_group_by_label(int64_t n, const int64_t *label, int64_t n_labels,
                      int64_t *ptr, int64_t *members);

/* src/ordering.py:206-233 pad_colors, size pass: nbar_of[n_c] and *n_pad. */
int tb_pad_colors_count(int64_t n_c, const int64_t *color_block_ranges,
                        int64_t b_s, int64_t w, int64_t *nbar_of,
                        int64_t *n_pad);

/* src/ordering.py:206-233 pad_colors, fill pass: slots[n_pad] (extended
 * original id at each padded position; dummies numbered from n upward in
 * consumption order).  Returns *n_dummy. */
int tb_pad_colors_fill(int64_t n, int64_t n_c, const int64_t *color_block_ranges,
                       const int64_t *block_order, const int64_t *block_ptr,
                       const int64_t *block_nodes, int64_t b_s, int64_t w,
                       int64_t *slots, int64_t n_pad, int64_t *n_dummy);

/* src/ordering.py:242-257 build_hbmc: composed new_of_old[n_pad] =
 * sec[padded_new_of_old], padded_new_of_old[slots[p]] = p. */
int tb_hbmc_compose(int64_t n_pad, const int64_t *slots, int64_t b_s, int64_t w,
                    int64_t *padded_new_of_old, int64_t *composed_new_of_old);

/* src/matrix.py:168-197 coo_to_csr (ensure_diagonal handled by the caller).
 * Outputs sized [n+1], [nnz], [nnz].  Duplicate (row, col) -> TB_EDUP with
 * *dup_row / *dup_col set to the first duplicate in (row, col) order. */
int tb_coo_to_csr(int64_t n, int64_t nnz, const int64_t *row,
                  const int64_t *col, const double *val, int64_t *row_ptr,
                  int64_t *col_idx, double *vals, int64_t *dup_row,
                  int64_t *dup_col);

/* src/matrix.py:293-304 permute_system (matrix part): entry (i, j) becomes
 * (q[i], q[j]); output rows sorted by column.  Outputs [n+1], [nnz], [nnz]. */
int tb_permute_csr(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                   const double *vals, const int64_t *new_of_old,
                   int64_t *row_ptr_out, int64_t *col_out, double *vals_out);

/* src/matrix.py:205-208 csr_transpose.  Outputs [n+1], [nnz], [nnz]. */
int tb_csr_transpose(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                     const double *vals, int64_t *row_ptr_out, int64_t *col_out,
                     double *vals_out);

/* src/matrix.py:239-261 csr_to_sell, fill pass (slice_ptr/slice_len computed
 * by the caller).  col_out64 and/or col_out32 may be NULL. */
int tb_csr_to_sell_fill(int64_t n, const int64_t *row_ptr,
                        const int64_t *col_idx, const double *vals,
                        int64_t width, int64_t n_slices,
                        const int64_t *slice_ptr, int64_t *col_out64,
                        int32_t *col_out32, double *vals_out);

/* Dependency levels of a strictly triangular CSR factor (forward = lower,
 * rows ascending; backward = upper, rows descending): the schedule that runs
 * the natural-order substitution (src/precond.py:285-298) on the device with
 * per-row arithmetic identical to the sequential sweep. */
int tb_level_schedule(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                      int forward, int64_t *level, int64_t *n_levels);

/* Sequential CSR SpMV in the reference's accumulation order
 * (K/numba_backend.py:16-23); host-side, used to form b = A x* once. */
int tb_spmv_csr_host(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                     const double *vals, const double *x, double *out);

/* MatrixMarket ingestion (src/io.py:70-163), byte scanning only; the
 * caller validates banner / size line / bounds / symmetry / duplicates.
 * tb_mm_locate: the size line (1-based number, byte range) and where the
 * entry lines start.  tb_mm_entries: parse up to `cap` entry lines into
 * rows / cols (1-based as written) / vals with their line numbers; *found
 * counts all entry lines, *kth_line = line of entry number `cap` (the
 * first surplus) or 0; first malformed line: *err_kind 1 = not three fields,
 * 2 = bad index, 3 = non-real value, its line and the offending bytes. */
int tb_mm_locate(const char *buf, int64_t len, int64_t *size_line, int64_t *size_b,
                 int64_t *size_e, int64_t *body_pos, int64_t *lines);
int tb_mm_entries(const char *buf, int64_t len, int64_t body_pos, int64_t first_line,
                  int64_t cap, int64_t *rows, int64_t *cols, double *vals, int64_t *linenos,
                  int64_t *found, int64_t *kth_line, int32_t *err_kind, int64_t *err_line,
                  int64_t *err_b, int64_t *err_e);

/* Setup helpers on a CSR pattern with sorted columns (host, OpenMP):
 * diagonal slot per row (-1 if none); structural symmetry; strictly lower
 * (upper = 0) / upper (upper = 1) part: count pass then fill pass. */
int tb_csr_diag_ptr(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                    int64_t *diag_out);
int tb_csr_is_symmetric(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                        int32_t *symmetric);
int tb_csr_tri_count(int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int32_t upper,
                     int64_t *row_out);
int tb_csr_tri_fill(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                    const double *vals, int32_t upper, const int64_t *row_out,
                    int64_t *col_out, double *val_out);

/* =========================================================================
 * Device operators on caller-owned device buffers (e.g. torch.cuda tensors
 * passed as data_ptr()).  `stream` is a cudaStream_t (NULL = legacy default).
 * Device index arrays are int32 (columns, slice lengths) and int64 (slice and
 * row pointers).
 * ========================================================================= */

/* K/numba_backend.py:26-37 spmv_sell. */
int tb_dev_spmv_sell(int64_t n_slices, const int64_t *slice_ptr,
                     const int32_t *slice_len, const int32_t *col_idx,
                     const double *vals, int64_t width, const double *x,
                     double *out, void *stream);

/* K/numba_backend.py:16-23 spmv_csr. */
int tb_dev_spmv_csr(int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                    const double *vals, const double *x, double *out,
                    void *stream);

/* K/numba_backend.py:132-153 fwd_sell_range over level-1 blocks [k0, k1),
 * which must be mutually independent (one HBMC color or a subrange of it). */
int tb_dev_fwd_sell_range(const int64_t *slice_ptr, const int32_t *slice_len,
                          const int32_t *col_idx, const double *vals,
                          const double *inv_d, const double *r, double *y,
                          int64_t width, int64_t block_rows, int64_t k0,
                          int64_t k1, void *stream);

/* K/numba_backend.py:156-171 bwd_sell_range (mirror image, SELL of U). */
int tb_dev_bwd_sell_range(const int64_t *slice_ptr, const int32_t *slice_len,
                          const int32_t *col_idx, const double *vals,
                          const double *inv_d, const double *y, double *z,
                          int64_t width, int64_t block_rows, int64_t k0,
                          int64_t k1, void *stream);

/* K/numba_backend.py:114-129 fwd_csr_range / bwd_csr_range generalised to a
 * set of independent tasks: task t processes rows rows[task_ptr[t] ..
 * task_ptr[t+1]) sequentially in the listed order (MC: one row per task; BMC:
 * one block per task; natural: one row per task of one dependency level).
 * rows == NULL means the identity list. */
int tb_dev_csr_sweep_tasks(int forward, const int64_t *row_ptr,
                           const int32_t *col_idx, const double *vals,
                           const double *inv_d, const double *src, double *dst,
                           int64_t task0, int64_t task1,
                           const int64_t *task_ptr, const int64_t *rows,
                           void *stream);

/* =========================================================================
 * Device plan: the whole ICCG operator set resident in HBM.
 * ========================================================================= */

#define TB_PRECOND_HBMC 0    /* SELL sweeps, one phase per color            */
#define TB_PRECOND_TASKS 1   /* CSR task sweeps (mc / bmc / natural levels) */
#define TB_SPMV_SELL 0
#define TB_SPMV_CSR 1
#define TB_SPMV_NONE 2      /* preconditioner-only plan (no A uploaded) */

typedef struct {            /* host arrays, SELL with int32 columns */
    int64_t n_slices;
    int64_t width;
    const int64_t *slice_ptr;   /* [n_slices+1] */
    const int32_t *slice_len;   /* [n_slices]   */
    const int32_t *col_idx;     /* [slice_ptr[n_slices]] */
    const double *vals;         /* [slice_ptr[n_slices]] */
} tb_sell_host;

typedef struct {            /* host arrays, CSR with int32 columns */
    int64_t n;
    const int64_t *row_ptr;     /* [n+1] */
    const int32_t *col_idx;     /* [nnz] */
    const double *vals;         /* [nnz] */
} tb_csr_host;

typedef struct {            /* phase -> tasks -> rows schedule */
    int64_t n_phases;
    const int64_t *phase_ptr;   /* [n_phases+1] into tasks */
    const int64_t *task_ptr;    /* [n_tasks+1] into rows   */
    const int64_t *rows;        /* [n_rows] (NULL = identity) */
    int64_t n_rows;
} tb_sched_host;

typedef struct {
    int32_t precond_kind;       /* TB_PRECOND_* */
    int32_t spmv_format;        /* TB_SPMV_* */
    int64_t n;                  /* system size (n_pad for HBMC) */
    int64_t n_real;             /* real unknowns (see real_pos) */
    const double *inv_d;        /* [n] */
    /* HBMC */
    int64_t w, b_s, n_c;
    const int64_t *color_lvl1_ranges;   /* [n_c+1] */
    tb_sell_host L_sell, U_sell;
    /* task sweeps */
    tb_csr_host L_csr, U_csr;
    tb_sched_host fwd_sched, bwd_sched;
    /* SpMV */
    tb_sell_host A_sell;
    tb_csr_host A_csr;
    /* TB_PLAN_* flags (ABI 2) */
    int64_t flags;
    /* ABI 3: the n_real sorted positions of the real unknowns (HbmcLayout
     * real_positions, src/ordering.py:263) when n_real < n, else NULL.  The
     * solver's dot products run over exactly these rows, in this order
     * (src/solver.py:150-153), so dummy rows never change a reduction. */
    const int64_t *real_pos;
} tb_plan_desc;

/* The plan is one rank of a row-partitioned system (partition.py): columns
 * may address halo entries beyond n, and the sweeps run phase by phase
 * (tb_plan_sweep_phase) with halo exchanges in between -- no persistent /
 * dataflow kernel is configured. */
#define TB_PLAN_PARTITIONED 1

typedef struct tb_plan tb_plan;

int tb_plan_create(const tb_plan_desc *desc, int device, tb_plan **out);
int tb_plan_destroy(tb_plan *plan);
/* device bytes held by the plan (matrices + internal vectors) */
int tb_plan_device_bytes(const tb_plan *plan, int64_t *bytes);

/* src/precond.py:395-400 sub_forward_hbmc (y = L^-1 r), device pointers. */
int tb_plan_forward(tb_plan *plan, const double *r, double *y, void *stream);
/* src/precond.py:403-408 sub_backward_hbmc (z = L^-T y). */
int tb_plan_backward(tb_plan *plan, const double *y, double *z, void *stream);
/* src/precond.py:411-425 apply_ic_preconditioner (z = (L L^T)^-1 r). */
int tb_plan_precond(tb_plan *plan, const double *r, double *z, void *stream);
/* src/matrix.py:307-323 spmv with the plan's A. */
int tb_plan_spmv(tb_plan *plan, const double *x, double *y, void *stream);
/* One color phase of the HBMC forward (forward=1, L) or backward (U) sweep:
 * the unit the plan launches between two grid-wide phase boundaries. */
int tb_plan_sweep_phase(tb_plan *plan, int forward, int64_t phase,
                        const double *src, double *dst, void *stream);
/* Which sweep kernel a phase uses: staged (TMA) or simple, and its launch. */
int tb_plan_phase_info(const tb_plan *plan, int forward, int64_t phase,
                       int32_t *staged, int32_t *warps, int32_t *grid,
                       int32_t *max_slots);
/* Whether tb_plan_precond / tb_pcg run as one persistent cooperative launch
 * (all color phases separated by in-kernel grid barriers) and its grid. */
int tb_plan_persistent(const tb_plan *plan, int32_t *precond, int32_t *pcg,
                       int32_t *grid);
/* Whether tb_plan_precond (and the preconditioner node of the tb_pcg graph)
 * runs the item-pipelined dataflow kernel (csrc/flow2.cuh): its grid (0 = not
 * used), ring stages and dynamic shared memory per CTA. */
int tb_plan_flow_info(const tb_plan *plan, int32_t *grid, int32_t *stages,
                      int64_t *smem_bytes);
/* Phase timestamps (%globaltimer, ns) of one steady PCG iteration of the
 * persistent kernel; the plan must be created with TB_TRACE=1 (diagnostics). */
int tb_plan_trace(const tb_plan *plan, uint64_t *out64 /* [64] */);
/* number of grid-wide phase boundaries one sweep crosses (n_c - 1) */
int tb_plan_barriers_per_sweep(const tb_plan *plan, int64_t *count);

typedef struct {
    int64_t iterations;
    int32_t converged;
    int32_t status;             /* TB_OK or TB_ECG_BREAKDOWN */
    int64_t breakdown_iter;
    double breakdown_value;
    int64_t kernel_launches;    /* device kernels launched by this call */
    int64_t host_syncs;         /* device->host convergence polls */
} tb_pcg_report;

/* src/solver.py:157-193 PCG loop entirely on device: x0 = 0, r = b,
 * relative residual history[0..iterations] written to history_host
 * (caller-allocated, max_iters+1 doubles).  b and x are device pointers of
 * length n (system ordering).  check_every = iterations launched between
 * convergence polls (0 = automatic). */
int tb_pcg(tb_plan *plan, const double *b, double *x, double tol,
           int64_t max_iters, int64_t check_every, void *stream,
           tb_pcg_report *report, double *history_host);

/* =========================================================================
 * Row-partitioned ICCG (csrc/dist.cu).  Device pointers; the
 * scalar slots s[] live in device memory and are all-reduced across ranks
 * by the caller (NCCL) between these calls.
 * ========================================================================= */

/* dst[i] = src[idx[i]], i < n: pack one halo exchange step's send buffer. */
int tb_dev_gather(int64_t n, const int32_t *idx, const double *src, double *dst,
                  void *stream);
/* s[slot] = <u, v> over [0, n) (deterministic two-pass; ws >= 1184 doubles).
 * The rank-local part of the dots of src/solver.py:150-153. */
int tb_dev_dot(int64_t n, const double *u, const double *v, double *s, int32_t slot,
               double *ws, void *stream);
/* alpha = s[num] / s[den]; x += alpha p; r -= alpha ap; s[rr] = <r, r>
 * (src/solver.py:178-186, rank-local part). */
int tb_dev_cg_xr(int64_t n, double *s, int32_t num, int32_t den, const double *p,
                 const double *ap, double *x, double *r, int32_t rr_slot, double *ws,
                 void *stream);
/* beta = s[num] / s[den]; p = z + beta p (src/solver.py:190-193). */
int tb_dev_cg_p(int64_t n, const double *s, int32_t num, int32_t den, const double *z,
                double *p, void *stream);

/* NVLink P2P halo exchange (partitioned solve without NCCL on the data path).
 * tb_p2p_alloc: device buffer (zeroed) + its CUDA IPC handle (64 bytes) for
 * peers; tb_p2p_open / close map / unmap a peer's buffer.  tb_p2p_push:
 * dst_remote[i] = src[idx[i]] (remote = peer-mapped), then, after all its
 * stores, *flag_remote = epoch (release, system scope); done_ctr: one zeroed
 * device word of the sender, private to this push.  tb_p2p_wait: block the
 * stream until flags[q] >= epoch for q in [0, count), q != skip (acquire,
 * system scope; traps after ~4 s instead of hanging). */
int tb_p2p_alloc(int64_t bytes, void **ptr, void *handle64);
int tb_p2p_free(void *ptr);
int tb_p2p_open(const void *handle64, void **ptr);
int tb_p2p_close(void *ptr);
int tb_p2p_push(int64_t n, const int32_t *idx, const double *src, double *dst_remote,
                uint32_t *flag_remote, uint32_t epoch, uint32_t *done_ctr, void *stream);
int tb_p2p_wait(const uint32_t *flags, int32_t count, int32_t skip, uint32_t epoch,
                void *stream);

/* One color phase of a partitioned rank's sweep with the halo push FUSED
 * into the sweep kernel: after a thread's lane walk, every row another rank
 * needs is stored straight into that rank's vector (peer-mapped pointer),
 * and the CTA finishing last releases `epoch` into each peer's flag word for
 * this rank (system scope) -- no separate pack / send.  Requires the lean
 * per-phase kernel (w = 32). */
#define TB_MAX_PEERS 16
typedef struct {
    int64_t row0, nrows;        /* local rows of the phase: [row0, row0 + nrows) */
    const int32_t *ptr;         /* device [nrows + 1]: destinations of row0 + r */
    const int32_t *peer;        /* device: index into peer_dst / peer_flag */
    const int32_t *off;         /* device: element index in that peer's vector */
    int32_t npeers;
    double *peer_dst[TB_MAX_PEERS];
    uint32_t *peer_flag[TB_MAX_PEERS];
    uint32_t epoch;
    uint32_t *done_ctr;         /* device word, 0, private to this launch */
} tb_push_desc;
int tb_plan_sweep_phase_push(tb_plan *plan, int forward, int64_t phase, const double *src,
                             double *dst, const tb_push_desc *push, void *stream);
/* tb_dev_cg_p with the SpMV's p-halo push fused in (same desc semantics,
 * rows [row0, row0 + nrows) of the rank's vector). */
int tb_dev_cg_p_push(int64_t n, const double *s, int32_t num, int32_t den, const double *z,
                     double *p, const tb_push_desc *push, void *stream);

/* K/numba_backend.py:40-79 ic0_factor on the device, bitwise, for a system
 * in HBMC order (src/precond.py:179-200 with layout "hbmc"): one launch per
 * color, thread per (level-1 block, lane) walking its b_s rows.  lrp / lci /
 * lvals: strictly-lower CSR of A (device; lvals overwritten with L), adiag =
 * a_ii (1 + shift) (device), d / inv_d outputs (device), pivot_ws: n doubles
 * of device scratch.  A non-positive pivot returns TB_EIC_BREAKDOWN with the
 * first such row (the one the sequential reference stops at) and its pivot. */
int tb_dev_ic0_hbmc(int64_t n, const int64_t *lrp, const int32_t *lci, double *lvals,
                    const double *adiag, double *d, double *inv_d, int64_t w, int64_t b_s,
                    int64_t n_c, const int64_t *color_lvl1_ranges, double *pivot_ws,
                    int64_t *bad_row, double *bad_pivot, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HBMC_B200_H */
