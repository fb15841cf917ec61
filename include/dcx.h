/*
 * dcx.h -- C ABI of the B200-native DOCH/ADOCH Ising solver (libdcx.so).
 *
 * The reference (dcising 0.1.0, /root/reference/pkg/src/dcising, "dc/" below)
 * is pure Python and has no FFI; its hot-path seams are Python calls. Each
 * entry point here names the reference interface it replaces. The Python host
 * package paper_2509_01928_b200 binds these through ctypes (see
 * INTEGRATION.md); plain pointers and sizes only, no torch types.
 *
 * Conventions (mirroring the reference's, dc/coupling.py:23-24, doch.py:101-102):
 *   - every call returns DCX_OK (0) or a negative DCX_E_* code; no exception
 *     crosses the ABI; dcx_last_error(ctx) holds the message;
 *   - input arrays are caller-owned and copied (the reference treats inputs as
 *     immutable, dc/coupling.py:79,137);
 *   - a context is not thread-safe; distinct contexts are independent
 *     ("concurrent runs on shared immutable instances").
 */
#ifndef DCX_H_
#define DCX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DCX_ABI_VERSION 1

#if defined(__GNUC__)
#define DCX_API __attribute__((visibility("default")))
#else
#define DCX_API
#endif

#define DCX_OK 0
#define DCX_E_INVALID (-1) /* maps to ValueError */
#define DCX_E_CUDA (-2)    /* maps to RuntimeError */
#define DCX_E_NCCL (-3)
#define DCX_E_OOM (-4)
#define DCX_E_STATE (-5) /* call order violated */

enum { DCX_SOLVER_DOCH = 0, DCX_SOLVER_ADOCH = 1 };
enum { DCX_WINDOW_ECONOMY = 0, DCX_WINDOW_EXACT = 1 };
enum { DCX_PREC_F64 = 0, DCX_PREC_F32 = 1, DCX_PREC_F16TC = 2 };
enum { DCX_PATH_AUTO = 0, DCX_PATH_MULTIPASS = 1, DCX_PATH_PERSISTENT = 2, DCX_PATH_DENSE_TC = 3 };
/* procedural coupling formulas (dc/coupling.py:293-298 _PROCEDURAL_FORMULAS) */
enum { DCX_FORMULA_SIN_PRODUCT = 0 };
enum {
  DCX_STOP_RUNNING = 0,
  DCX_STOP_CONVERGED = 1,
  DCX_STOP_MAX_ITERS = 2,
  DCX_STOP_TIME_BUDGET = 3
};
/* per-replica partial sums exchanged by the row-partitioned solve:
 * q_sum[r] = {sum x^4, sum x.Ax, sum s.Js, sum y^4, sum y.Ay} (all-reduce SUM),
 * q_max[r] = {max |dx| of the pass, max |dx| of the ADOCH update, elapsed s} (all-reduce MAX) */
#define DCX_QSUM 5
#define DCX_QMAX 3
/* history event bits */
enum { DCX_EV_RECORDED = 1, DCX_EV_DESCENT = 2, DCX_EV_ACCEPTED = 4, DCX_EV_REJECTED = 8 };

typedef struct dcx_ctx dcx_ctx;

/* Solver knobs: SolverParams (dc/spectral.py:25-49) + doch_solve/adoch_solve
 * keyword arguments (dc/solvers/doch.py:169-176, :248-256) + the reference
 * constants CONVERGENCE_TOL / DESCENT_WARN_TOL (doch.py:33-34). */
typedef struct {
  int32_t solver;       /* DCX_SOLVER_* */
  int32_t window_mode;  /* DCX_WINDOW_* (adoch only) */
  int32_t precision;    /* DCX_PREC_* */
  int32_t lookback_q;   /* >= 1 */
  int64_t max_iters;    /* >= 0 */
  int64_t trace_stride; /* >= 1 */
  double time_budget_s; /* < 0: no budget */
  double conv_tol;      /* 1e-10 in the reference */
  double descent_tol;   /* 1e-9 in the reference */
  int32_t record_states;
  int32_t path;  /* DCX_PATH_* */
  int32_t chunk; /* iterations per host drain; 0 = auto */
  int32_t reserved;
} dcx_params;

typedef struct {
  int64_t iterations;
  int32_t stop_reason; /* DCX_STOP_* */
  int32_t best_iter;
  double best_energy;
  int64_t n_hist;        /* iterations + 1 history entries available */
  int32_t descent_warn;  /* first descent-violation iteration, -1 if none */
  int32_t path_used;     /* DCX_PATH_* actually executed */
} dcx_summary;

typedef struct {
  int64_t n, nnz;
  int32_t value_kind; /* 0 uniform, 1 int8, 2 int16, 3 f32, 4 f64, 5 procedural */
  int32_t lanes;      /* lanes per row of the R=1 kernels */
  double scale;       /* value = scale * stored integer (integer kinds) */
  int32_t dense;      /* set through dcx_set_dense */
  int32_t lattice_L;  /* > 0: recognised as the periodic L x L torus (the stencil pass runs; R > 1, f32) */
} dcx_coupling_info;

DCX_API int dcx_abi_version(void);
DCX_API const char* dcx_last_error(const dcx_ctx* ctx); /* ctx may be NULL: last global error */

/* Context: owns the CUDA stream and all device buffers of one instance. */
DCX_API int dcx_create(int device, dcx_ctx** out);
DCX_API void dcx_destroy(dcx_ctx* ctx);

/* Coupling upload.
 * dcx_set_csr replaces CsrCoupling(values, col_indices, row_offsets)
 * (dc/coupling.py:115-152): host f64 values, int64 indices, symmetric, sorted
 * columns, zero diagonal. Stored on device as uint32 row offsets, int32
 * columns and the narrowest exact value form (uniform / int8 / int16 x scale,
 * else f32 / f64).
 * dcx_set_dense replaces DenseCoupling(array) (dc/coupling.py:71-112). */
DCX_API int dcx_set_csr(dcx_ctx* ctx, int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* col_indices,
                const double* values);
DCX_API int dcx_set_dense(dcx_ctx* ctx, int64_t n, const double* J_rowmajor);
DCX_API int dcx_coupling(const dcx_ctx* ctx, dcx_coupling_info* out);
/* dcx_set_procedural replaces ProceduralCoupling(n, seed, formula)
 * (dc/coupling.py:209-229; gen_procedural_sin dc/generate.py:115-123):
 * J_ij = sin(i*j + seed) for i != j, 0 on the diagonal, never stored: every
 * product regenerates it on the device (the reference materialises b x b tiles,
 * dc/matvec.py:117-155). Solves run on the multipass path; dcx_power is not
 * available (the reference's auto method is the Wigner estimate for
 * procedural matrices, dc/spectral.py:203-216).
 * dcx_proc_row_stats: out[3i..3i+2] = (sum_j J_ij, sum_j J_ij^2, sum_j |J_ij|)
 * over j != i, f64 -- offdiag_moments and abs_row_sums (dc/coupling.py:248-268). */
DCX_API int dcx_set_procedural(dcx_ctx* ctx, int64_t n, int64_t seed, int32_t formula);
DCX_API int dcx_proc_row_stats(dcx_ctx* ctx, double* out /* [n][3] */);
/* dcx_row_stats: the same [n][3] row statistics for any coupling on the device (CSR rows
 * summed in column order, dense rows by a fixed-order warp tree, procedural as above):
 * offdiag_moments and abs_row_sums (dc/coupling.py:104-109, :197-206) for the Wigner
 * estimate and beta of derive_params (dc/spectral.py:175-189, :246-247). */
DCX_API int dcx_row_stats(dcx_ctx* ctx, double* out /* [n][3] */);

/* Operator seam (dc/matvec.py:99-114 matvec; :181-190 operator_energy;
 * dc/model.py:79-87 energy; dc/solvers/doch.py:76-103 hamiltonian/apply_T).
 * Vectors are [R][n] row-major on the host.
 *   dcx_matvec:  out_r = J v_r
 *   dcx_apply:   tx_r = cbrt((J v_r + alpha_r v_r) / beta_r), h_r = H(v_r)  (either may be NULL)
 *   dcx_energy:  E_r = -1/2 s_r^T J s_r, exact integer accumulation for integer couplings */
DCX_API int dcx_matvec(dcx_ctx* ctx, int32_t R, const double* v, double* out, int32_t precision);
DCX_API int dcx_apply(dcx_ctx* ctx, int32_t R, const double* alpha, const double* beta, const double* v, double* tx,
              double* h, int32_t precision);
DCX_API int dcx_energy(dcx_ctx* ctx, int32_t R, const int8_t* spins, double* energies);

/* Solve R replicas at once: doch_solve / adoch_solve (dc/solvers/doch.py:169,
 * :248) for each replica r with (alpha_r, beta_r, x0_r). x0 is [R][n]
 * (initial_state of doch.py:132-145 is drawn by the caller).
 * dcx_solve_begin uploads and starts the device clock; dcx_solve_step runs up
 * to one chunk and drains the history; *live becomes 0 when every replica
 * has stopped. dcx_solve_run loops dcx_solve_step to the end. */
DCX_API int dcx_solve_begin(dcx_ctx* ctx, const dcx_params* params, int32_t R, const double* alpha, const double* beta,
                    const double* x0);
DCX_API int dcx_solve_step(dcx_ctx* ctx, int32_t* live);
DCX_API int dcx_solve_run(dcx_ctx* ctx);

/* Results (valid after the run, or between steps for the drained part). */
DCX_API int dcx_result_summary(dcx_ctx* ctx, int32_t r, dcx_summary* out);
/* history entries k in [from, from+count): H(x_k), E(sign x_k) (NaN if not
 * recorded), device seconds since dcx_solve_begin, event bits */
DCX_API int dcx_result_history(dcx_ctx* ctx, int32_t r, int64_t from, int64_t count, double* h, double* e, double* t,
                       int32_t* ev);
/* bulk forms for R replicas: per-replica summary columns, and every history
 * entry as [R][K] rows (K >= max n_hist; unused tail entries are not written) */
DCX_API int dcx_result_summaries(dcx_ctx* ctx, int64_t* iterations, int32_t* stop_reason, double* best_energy,
                                 int64_t* n_hist, int32_t* descent_warn);
DCX_API int dcx_result_history_all(dcx_ctx* ctx, int64_t K, double* h, double* e, double* t, int32_t* ev);
DCX_API int dcx_result_best_spins(dcx_ctx* ctx, int8_t* out /* [R][n] */);
DCX_API int dcx_result_state(dcx_ctx* ctx, double* out /* [R][n], final x */);
DCX_API int dcx_result_states(dcx_ctx* ctx, int32_t r, double* out /* [(iterations+1)][n] */);
/* Live profile of the dominant kernel of the current path (the fused pass of
 * the multipass path, the fused GEMM of the dense path): after
 * dcx_solve_begin, launches it `launches` times on the context stream between
 * two CUDA events and returns the mean duration. Consumes the run. */
DCX_API int dcx_profile_kernel(dcx_ctx* ctx, int32_t launches, double* ms_per_launch, int32_t* kernel_id);
/* Power iteration of dc/spectral.py:60-111 (_power_core) on M = shift*I - J
 * (use_shift != 0) or M = -J, entirely on the device (one cooperative kernel;
 * per iteration one product and fixed-order grid reductions). `restart` is the
 * normalised seeded restart vector (n entries) the reference would draw.
 * Outputs (|lambda|, Rayleigh quotient, iterations, converged) as _power_core. */
DCX_API int dcx_power(dcx_ctx* ctx, int32_t use_shift, double shift, double tol, int64_t max_iters,
                      const double* restart, double* mag, double* rayleigh, int64_t* iterations, int32_t* converged);
/* device time of the last dcx_solve_run/step sequence, seconds */
DCX_API int dcx_result_device_seconds(dcx_ctx* ctx, double* out);

/* ---- Detached results (the reference returns host arrays, dc/solvers/common.py:33-43) ----
 * dcx_result_detach moves a finished run's bulk outputs out of the context: the
 * final states and best spins stay in device memory owned by the result, the
 * history stays in the pinned buffer the run drained it into. The host arrays
 * are copied out only when asked for, so a caller reading the energies alone
 * (dcx_result_summaries, on the context) moves no bulk data; the context can
 * begin its next run at once. dcx_res_warn_delta: H(x_k) - H(x_{k-1}) at each
 * replica's descent warning (NaN without one), for the reference's
 * RuntimeWarning (dc/solvers/doch.py:220-226). */
typedef struct dcx_result dcx_result;
DCX_API int dcx_result_detach(dcx_ctx* ctx, dcx_result** out);
DCX_API int dcx_res_state(dcx_result* res, double* out /* [R][n] */);
DCX_API int dcx_res_best_spins(dcx_result* res, int8_t* out /* [R][n] */);
DCX_API int dcx_res_history_all(dcx_result* res, int64_t K, double* h, double* e, double* t, int32_t* ev);
DCX_API int dcx_res_warn_delta(dcx_result* res, double* out /* [R] */);
DCX_API void dcx_result_free(dcx_result* res);

/* ---- Row-partitioned solve (multi-GPU) ----
 * The reference has no distributed solver; this splits the one mat-vec per
 * iteration of doch_solve / adoch_solve (economy window) by rows. A context
 * holds rows [row_base, row_base + n_rows) of the coupling in a spin index
 * space of n_cols entries (columns already mapped into that space, sorted per
 * row). The iterate buffers are caller-owned device arrays of n_cols x R
 * elements (layout [n_cols][R], f64 or f32 by precision), two of them by pass
 * parity; pass p gathers from buffer p&1 and writes this context's rows of
 * buffer (p+1)&1, which the caller completes with an all-gather of every
 * rank's row slice before the next pass. Per-replica partials land in
 * caller-owned device arrays q_sum [R][DCX_QSUM] / q_max [R][DCX_QMAX] that
 * the caller all-reduces (SUM / MAX) between dcx_dist_pass and
 * dcx_dist_control; the control is a deterministic function of the reduced
 * values, so every rank takes the same decisions (stop, ADOCH accept). All
 * work is ordered on the context stream (dcx_stream); collectives must be
 * issued on it. */
DCX_API int dcx_set_csr_block(dcx_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t row_base, int64_t nnz,
                              const int64_t* row_offsets, const int64_t* col_indices, const double* values);
DCX_API int dcx_stream(dcx_ctx* ctx, void** stream /* cudaStream_t */);
DCX_API int dcx_dist_begin(dcx_ctx* ctx, const dcx_params* params, int32_t R, const double* alpha, const double* beta,
                           const double* x0_rows /* [R][n_rows] */, void* x_buf0, void* x_buf1, double* q_sum,
                           double* q_max);
DCX_API int dcx_dist_pass(dcx_ctx* ctx);
/* The pass split in two row ranges so the x exchange can overlap it: the caller orders its
 * rows [interior | boundary] (boundary = rows that reference halo rows or that other ranks
 * read), runs [0, n_interior) while the halo of x_p is in flight, then the boundary rows,
 * then dcx_dist_reduce (both halves of the partial slots into q_sum / q_max), in place of
 * dcx_dist_pass. half: 0 or 1, the slot half the range writes. */
DCX_API int dcx_dist_pass_rows(dcx_ctx* ctx, int64_t row_lo, int64_t row_hi, int32_t half);
DCX_API int dcx_dist_reduce(dcx_ctx* ctx);
DCX_API int dcx_dist_control(dcx_ctx* ctx);
/* synchronises the stream, drains the history; *live = 0 once every replica stopped */
DCX_API int dcx_dist_poll(dcx_ctx* ctx, int32_t* live, int64_t* passes);
/* ends the run (pending best-spin copies, device time); results as for dcx_solve_* with n = n_rows */
DCX_API int dcx_dist_finish(dcx_ctx* ctx);

/* ---- instance generation and ingest on the device ----
 * gen_sparse_9bit of dc/generate.py:80-112 (replaces the per-row numpy loop and the
 * scipy COO -> CSR closure): n spins, n_p = int(102300 // p) (computed by the caller
 * as the reference does), per-row Philox4x64-10 streams keyed (seed, row). The CSR
 * stays in the context until dcx_gen_result copies it out in the reference's layout
 * (int64 row_offsets [n+1], int64 col_indices [nnz], f64 values [nnz]) -- the bytes
 * the reference's CsrCoupling holds. */
DCX_API int dcx_gen_sparse_9bit(dcx_ctx* ctx, int64_t n, int64_t n_p, uint64_t seed, int64_t* nnz);
DCX_API int dcx_gen_result(dcx_ctx* ctx, int64_t* row_offsets, int64_t* col_indices, double* values);
/* CsrCoupling.validate of dc/coupling.py:153-176 on the device (csr_load's ingest check,
 * dc/io.py:272-305): *check = 0 valid, 2 offsets not starting at 0 / decreasing,
 * 3 row_offsets[n] != nnz, 4 column out of range, 5 columns not strictly increasing in
 * row *row, 6 stored diagonal in row *row, 7 non-finite value, 8 asymmetric; the first
 * failing check in the reference's order. *all_int = every value integral (nnz > 0). */
DCX_API int dcx_validate_csr(dcx_ctx* ctx, int64_t n, int64_t nnz, const int64_t* row_offsets,
                             const int64_t* col_indices, const double* values, int32_t* check, int64_t* row,
                             int32_t* all_int);

#ifdef __cplusplus
}
#endif
#endif /* DCX_H_ */
