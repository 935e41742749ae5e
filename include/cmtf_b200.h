/*
 * cmtf_b200.h -- C ABI of the B200-native S^3CMTF training path.
 *
 * This is the drop-in boundary for the reference's in-process C++ library
 * API (CMake package cmtf::core, /root/reference/proj/core).  The reference
 * has no FFI of its own; each entry point below names the reference
 * function it replaces (file:line, relative to /root/reference/proj/core).
 * Plain pointers and sizes only; no torch or CUDA types.  The C++ wrapper
 * in include/cmtf_b200.hpp rebuilds the reference's signatures and
 * exception types on top of it.
 *
 * Conventions (as the reference, include/cmtf/sparse_data.hpp:13-40):
 *  - indices are 0-based u32, tensor entries AoS (order indices per entry),
 *    matrix entries AoS pairs (row, col); values are f64 on the boundary and
 *    f32 on the device;
 *  - the core is row-major with the last mode fastest (src/tucker.cpp:49-54),
 *    factors are row-major I_n x J_n, coupled factors cols x J_mode.
 *
 * Return codes: 0 ok, 1 validation (ValidationError), 2 divergence
 * (DivergenceError), 3 CUDA error, 4 NCCL error, 5 unsupported,
 * 6 parse (ParseError).
 * The message of the last failure is available from cmtf_gpu_last_error()
 * (per calling thread) and cmtf_gpu_ctx_error(ctx).  A context is not
 * thread-safe, as TrainState is not (include/cmtf/trainer.hpp:49-56).
 */
#ifndef CMTF_B200_H_
#define CMTF_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMTF_OK 0
#define CMTF_EVALIDATION 1
#define CMTF_EDIVERGENCE 2
#define CMTF_ECUDA 3
#define CMTF_ENCCL 4
#define CMTF_EUNSUPPORTED 5
#define CMTF_EPARSE 6 /* ParseError (include/cmtf/errors.hpp): text formats */

/* GradientKernel (include/cmtf/trainer.hpp:14) */
#define CMTF_KERNEL_NAIVE 0
#define CMTF_KERNEL_OPT 1

/* Execution mode of an epoch on the device. */
#define CMTF_EXEC_HOGWILD 0 /* lock-free parallel sweep (the product path) */
#define CMTF_EXEC_SERIAL 1  /* exact reference order, P=1 semantics      */

/* TrainConfig (include/cmtf/trainer.hpp:18-36) plus device fields. */
typedef struct cmtf_gpu_config {
  int32_t order;
  const uint32_t *ranks; /* [order] */
  double eta0;           /* default 1e-3 */
  double mu;             /* default 0.1  */
  double lambda_reg;     /* default 0.1  */
  int32_t workers;       /* reference worker count; informs the core-step
                            scale only in CMTF_EXEC_SERIAL (P=1 there)   */
  int32_t max_epochs;    /* default 100  */
  double rel_tol;        /* default 1e-4 */
  uint64_t seed;
  int32_t kernel;         /* CMTF_KERNEL_* */
  int32_t core_structure; /* 0 dense Tucker; 1 CP / hyper-diagonal (equal
                            ranks; model transfers carry its ranks[0]
                            superdiagonal values as the core)           */
  int32_t nonnegative;    /* per-step clamp at 0 (src/trainer.cpp:185) */
  double init_scale;      /* default 1.0 */
  /* ---- device fields ---- */
  int32_t device;        /* CUDA ordinal */
  int32_t exec_mode;     /* CMTF_EXEC_* */
  int32_t hog_threads;   /* concurrent Hogwild workers; 0 = auto        */
  int32_t sort_mode;     /* mode the COO is sorted by; -1 = auto        */
  int32_t force_generic; /* 1: use the generic-N kernels even when a
                            specialised one exists (testing)            */
  int32_t order_policy;  /* entry order of the Hogwild sweep: 0 = sorted
                            by sort_mode (row caching), 1 = a seeded random
                            permutation (the reference's shuffled
                            schedule, src/trainer.cpp:122-128), 2 = the
                            caller's order (DSGD strata)                */
  float hot_tau;         /* rows whose expected concurrent updates
                            (count * workers / nnz) reach hot_tau get a
                            per-block shared-memory replica; 0 = default
                            (0.5), < 0 disables                         */
  float kappa;           /* damping of the merged hot-row replica steps:
                            alpha = kappa / (kappa + q), q = (n_other /
                            cnt) * (1 - exp(-eta * sum|c|^2)), n_other =
                            the row's expected concurrent updates in other
                            blocks; 0 = default (0.5)                   */
  int32_t flush_every;   /* sweep iterations between hot-row replica
                            merges; 0 = default (32 on the tcgen05
                            kernel, 16 on the others)                   */
  int32_t kernel_version;/* 0 = auto (v2 where specialised), 1 = v1     */
  int32_t core_flush_every; /* sweep iterations between block-level core
                            pushes; 0 = default (1)                     */
  float kappa_core;      /* damping of the batched core step; the curvature
                            estimate is the trace E|phi|^2, an upper
                            bound of the top eigenvalue; 0 = default 2.0 */
  int32_t debug_count_visits; /* TrainConfig::debug_count_visits
                            (include/cmtf/trainer.hpp:31-32): count every
                            record visit of the current epoch on the
                            device (cmtf_gpu_visit_counts)              */
} cmtf_gpu_config;

typedef struct cmtf_gpu_ctx cmtf_gpu_ctx;

/* Fills defaults exactly as TrainConfig's member initialisers. */
void cmtf_gpu_config_default(cmtf_gpu_config *cfg);

const char *cmtf_gpu_last_error(void);
const char *cmtf_gpu_ctx_error(const cmtf_gpu_ctx *ctx);
/* ABI version, bumped on any signature change. */
int32_t cmtf_gpu_abi_version(void);

int cmtf_gpu_create(const cmtf_gpu_config *cfg, cmtf_gpu_ctx **out);
int cmtf_gpu_destroy(cmtf_gpu_ctx *ctx);

/* DataBundle (include/cmtf/sparse_data.hpp:80-84) built from the training
 * SparseTensor (:17-40) and CoupledMatrix list (:44-70); counts as
 * count_mode_occurrences (src/sparse_data.cpp:344-362) are derived on the
 * device.  Range and finiteness are validated as check_entries
 * (src/sparse_data.cpp:19-64) on the device: indices in range, finite
 * values, and no duplicate index tuples -- rejected with the reference's
 * message for the lexicographically smallest duplicated tuple.
 * idx/vals may be host (pageable or pinned) or device pointers (UVA). */
int cmtf_gpu_set_tensor(cmtf_gpu_ctx *ctx, const uint32_t *dims,
                        const uint32_t *idx, const double *vals, uint64_t nnz);
int cmtf_gpu_add_matrix(cmtf_gpu_ctx *ctx, int32_t mode0, uint32_t rows,
                        uint32_t cols, const uint32_t *idx, const double *vals,
                        uint64_t nnz, double weight);
/* Drops the matrices (for re-uploading a bundle into the same context). */
int cmtf_gpu_clear_matrices(cmtf_gpu_ctx *ctx);

/* initialize / make_state (src/trainer.cpp:94-103,130-137): the seeded
 * random model (draw law of random_model, src/trainer.cpp:30-58), epoch 0,
 * eta = eta0, schedule = build_schedule. */
int cmtf_gpu_make_state(cmtf_gpu_ctx *ctx);

/* Model transfer (host f64 <-> device f32).  couplings may be NULL when
 * there are no matrices. */
int cmtf_gpu_set_model(cmtf_gpu_ctx *ctx, const double *core,
                       const double *const *factors,
                       const double *const *couplings);
int cmtf_gpu_get_model(cmtf_gpu_ctx *ctx, double *core, double *const *factors,
                       double *const *couplings);
int cmtf_gpu_get_state(cmtf_gpu_ctx *ctx, int32_t *epoch, double *eta);
int cmtf_gpu_set_state(cmtf_gpu_ctx *ctx, int32_t epoch, double eta);

/* run_epoch (src/trainer.cpp:267-316): one sweep over every training entry
 * and matrix entry, then epoch += 1, eta = eta0 / (1 + mu * epoch), and the
 * non-finite scan (returns CMTF_EDIVERGENCE with the reference's message).
 * Serial mode replays the reference schedule (build_schedule +
 * shuffle_schedule, src/trainer.cpp:114-128) on the device. */
int cmtf_gpu_run_epoch(cmtf_gpu_ctx *ctx);

/* epoch_stats (src/eval.cpp:120-144). */
int cmtf_gpu_epoch_stats(cmtf_gpu_ctx *ctx, double lambda_reg,
                         double *train_rmse, double *objective);

/* test_rmse (src/eval.cpp:101-107) for a held-out tensor. */
int cmtf_gpu_test_rmse(cmtf_gpu_ctx *ctx, const uint32_t *idx,
                       const double *vals, uint64_t nnz, double *rmse);

/* matrix_rmse (src/eval.cpp:109-118) for coupled matrix m of the bundle. */
int cmtf_gpu_matrix_rmse(cmtf_gpu_ctx *ctx, int32_t m, double *rmse);

/* The tail of train() (src/trainer.cpp:342-345) applied to the current
 * model, into host buffers laid out like cmtf_gpu_get_model.  Nonnegative
 * configurations: apply_nonnegative_projection (src/trainer.cpp:348-387).
 * Otherwise finalize_orthogonalize (src/tucker.cpp:226-283): U_n = Q R with Q
 * orthonormal and R upper triangular with a nonnegative diagonal (the
 * reference's sign-fixed Householder QR; unique for full-rank factors,
 * computed as CholeskyQR2 in f64 on the device), core <- core x_n R, coupled
 * factors V <- V R^T.  The device training state is not modified.
 * CMTF_EVALIDATION if a mode has fewer rows than its rank or a factor is
 * rank deficient. */
int cmtf_gpu_finalize_model(cmtf_gpu_ctx *ctx, double *core, double *const *factors,
                            double *const *couplings);

/* train (src/trainer.cpp:318-346) up to the finalisation (see
 * cmtf_gpu_finalize_model for the tail of the reference's train()): epochs until
 * |delta rmse| / rmse < rel_tol or max_epochs.  log receives 4 doubles per
 * epoch (epoch, train_rmse, objective, seconds); capacity in entries. */
int cmtf_gpu_train(cmtf_gpu_ctx *ctx, double *log, int32_t log_capacity,
                   int32_t *n_log);

/* Per-entry probe at the frozen model: compute_gradient(_opt)
 * (src/gradients.cpp:83-223) for training entries ids[0..n).  grow holds
 * n * (J_1 + ... + J_N) row gradients, gcore n * prod(J) core gradients
 * (may be NULL), xhat / residual n values each (may be NULL). */
int cmtf_gpu_entry_grads(cmtf_gpu_ctx *ctx, const uint64_t *ids, uint64_t n,
                         double *xhat, double *residual, double *grow,
                         double *gcore);

/* The product epoch kernel's own arithmetic at the frozen device model
 * (order 3, opt kernel, tcgen05 path): one sweep with eta = 0 -- the model is
 * unchanged -- recording for every training entry (caller order) x_hat, the
 * residual and the row gradients [nnz][3 J] (compute_gradient_opt,
 * src/gradients.cpp:130-223, as computed inside the epoch kernel's tensor-core
 * tiles), plus the summed data term of the core gradient,
 * sum_e -r_e u1 (x) u2 (x) u3 [J^3].  Any output may be NULL.
 * CMTF_EUNSUPPORTED when the epoch does not run that kernel. */
int cmtf_gpu_kernel_probe(cmtf_gpu_ctx *ctx, double *xhat, double *residual,
                          double *grow, double *gcore_data);

/* Stateless batched form of compute_gradient / compute_gradient_opt
 * (include/cmtf/gradients.hpp:59-74): n independent entries, each with its
 * own x, N rows (rows[e*sumJ ...]) and N counts, sharing one core, computed
 * in f64 on the device (the reference's algorithms term for term, incl.
 * the opt kernel's 1e-12 divisor fallbacks).  core_structure 0: dense core
 * (prod J values); 1: CP / hyper-diagonal (src/gradients.cpp:108-115,
 * 145-152,192-205): core, each entry's core gradient and intermediate tensor
 * hold the ranks[0] superdiagonal values, all ranks equal.  intermediate
 * (opt only, may be NULL): KernelWorkspace::s, the intermediate tensor
 * S[d] = g_d prod_n u_n[j_n] of each entry. */
int cmtf_gpu_compute_gradient(int32_t kernel, int32_t order,
                              const uint32_t *ranks, int32_t core_structure,
                              const double *core, uint64_t n, const double *x,
                              const double *rows, const uint32_t *counts,
                              double lambda_reg, uint64_t nnz_total,
                              int32_t with_core, double *grow, double *gcore,
                              double *residual, double *intermediate,
                              int32_t device);

/* Batched matrix_entry_gradients (include/cmtf/gradients.hpp:83-86), f64
 * on the device like cmtf_gpu_compute_gradient. */
int cmtf_gpu_matrix_entry_gradients(uint64_t n, uint32_t j, const double *y,
                                    const double *u, const double *v,
                                    double lambda_m, double lambda_reg,
                                    const uint32_t *col_count, double *du,
                                    double *dv, double *residual,
                                    int32_t device);

/* collapse (include/cmtf/gradients.hpp:32-34, src/gradients.cpp:35-60) of
 * an intermediate tensor (prod J values; CP: ranks[0]) along `mode`, f64 on
 * the device; out has ranks[mode] values. */
int cmtf_gpu_collapse(int32_t order, const uint32_t *ranks, int32_t core_structure,
                      const double *values, int32_t mode, double *out,
                      int32_t device);

/* The next serial-mode epoch replays exactly this schedule (tensor ids
 * [0, nnz) then matrix entries in bundle order, as build_schedule,
 * src/trainer.cpp:114-120) instead of shuffling its own persisted copy: a
 * caller holding TrainState::schedule (shuffle_schedule on the host, as the
 * reference's run_epoch does) passes it here before cmtf_gpu_run_epoch. */
int cmtf_gpu_set_schedule(cmtf_gpu_ctx *ctx, const uint64_t *schedule, uint64_t n);

/* ---- DSGD (multi-GPU) support: SURVEY.md 8(e) ----------------------
 * A rank uploads its local bundle grouped by stratum (order_policy 2 keeps
 * the caller's order) and runs each sub-epoch over record ranges.        */

/* One Hogwild sweep over tensor records [t_lo, t_hi) and, for each coupled
 * matrix m, records [m_lo[m], m_hi[m]) (caller order).  No epoch
 * bookkeeping; m_lo/m_hi may be NULL (no matrix entries). */
int cmtf_gpu_sweep_range(cmtf_gpu_ctx *ctx, uint64_t t_lo, uint64_t t_hi,
                         const uint64_t *m_lo, const uint64_t *m_hi);
/* epoch += 1, eta decay, non-finite scan (the tail of run_epoch). */
int cmtf_gpu_end_epoch(cmtf_gpu_ctx *ctx);
/* Declare the replicated parameters and the number of ranks updating them
 * concurrently (their batched steps are damped for world * local
 * concurrency).  mode_mask / mat_mask: bit n = factor n / coupled factor n. */
int cmtf_gpu_set_shared(cmtf_gpu_ctx *ctx, int32_t world, uint32_t mode_mask,
                        uint32_t mat_mask, uint64_t nnz_global);
/* Override observation counts with the GLOBAL counts (a rank's local bundle
 * sees only its own entries): which = mode n (0..N-1) or 100 + m for the
 * column counts of coupled matrix m.  Recomputes lambda/count. */
int cmtf_gpu_set_counts(cmtf_gpu_ctx *ctx, int32_t which, const uint32_t *counts,
                        uint32_t n);
/* NCCL communicator over the ranks (unique id from rank 0, 128 bytes). */
int cmtf_gpu_comm_unique_id(void *id_out);
int cmtf_gpu_comm_init(cmtf_gpu_ctx *ctx, int32_t nranks, int32_t rank,
                       const void *unique_id);
/* Sum the deltas (current - base) of the selected parameters over the
 * ranks with ncclAllReduce and re-base: afterwards every rank holds
 * base + sum of all ranks' deltas.  core != 0 includes the core. */
int cmtf_gpu_sync(cmtf_gpu_ctx *ctx, uint32_t mode_mask, uint32_t mat_mask,
                  int32_t core);
/* Row-block rotation of a stratified factor (U2 / U3
 * blocks move along the ring instead of being all-reduced): send rows
 * [send_lo, send_hi) of factor `which` (mode n, or 100 + m for coupled
 * factor m) to rank send_peer and receive rows [recv_lo, recv_hi) from rank
 * recv_peer, as one NCCL group on the context's stream (no host wait). */
int cmtf_gpu_exchange_rows(cmtf_gpu_ctx *ctx, int32_t which, uint32_t send_lo,
                           uint32_t send_hi, int32_t send_peer, uint32_t recv_lo,
                           uint32_t recv_hi, int32_t recv_peer);
/* Consolidation of a block-distributed factor: rank b broadcasts rows
 * [lo[b], hi[b]) to every rank (n_blocks = number of ranks). */
int cmtf_gpu_broadcast_rows(cmtf_gpu_ctx *ctx, int32_t which, int32_t n_blocks,
                            const uint32_t *lo, const uint32_t *hi);
/* Single-device emulation of one rotation step: copy rows [lo, hi) of
 * factor `which` from context src to context dst. */
int cmtf_gpu_exchange_rows_local(cmtf_gpu_ctx *src, cmtf_gpu_ctx *dst,
                                 int32_t which, uint32_t lo, uint32_t hi);
/* The same reduction for n contexts living on ONE device (single-GPU
 * emulation of the ranks, used by tests). */
int cmtf_gpu_sync_local(cmtf_gpu_ctx *const *ctxs, int32_t n, uint32_t mode_mask,
                        uint32_t mat_mask, int32_t core);

/* The exactly-once visit check (TrainState::visit_counts,
 * include/cmtf/trainer.hpp:55; the reference's test_trainer.cpp:207-219):
 * visits of the last epoch per training entry (caller order, nnz values) and
 * per coupled-matrix record of the merged shuffled stream (sum of matrix nnz
 * values).  Needs debug_count_visits; CMTF_EUNSUPPORTED after a serial-mode
 * epoch (one thread block replays the schedule; nothing to count). */
int cmtf_gpu_visit_counts(cmtf_gpu_ctx *ctx, uint32_t *tensor_counts,
                          uint32_t *matrix_counts);

/* Device-side timing marks on the context's launching stream: record event
 * `slot` (0..7); elapsed milliseconds between two recorded marks. */
int cmtf_gpu_mark(cmtf_gpu_ctx *ctx, int32_t slot);
int cmtf_gpu_elapsed_ms(cmtf_gpu_ctx *ctx, int32_t from, int32_t to, double *ms);

/* Timing and introspection for the harness.  Events bracket the last
 * run_epoch on the launching stream.  kernel_ms[0..3] = tensor sweep,
 * matrix sweep(s), non-finite scan, total; launches = kernels launched. */
int cmtf_gpu_last_epoch_timing(cmtf_gpu_ctx *ctx, double *kernel_ms,
                               int32_t *launches);
/* Which tensor kernel the context selected: 0 generic, 1 specialised N=3,
 * 2 specialised N=4; hog_threads actually used. */
int cmtf_gpu_kernel_info(cmtf_gpu_ctx *ctx, int32_t *which,
                         int32_t *hog_threads, int32_t *sort_mode);
/* The tensor records' visiting layout: *blocks = B when the order-3
 * tcgen05 epoch runs the L2-blocked order (B x B strata of mode-1 x mode-2
 * row blocks, stratum-major records, random stratum sequence per epoch; set
 * up on the first whole random-order epoch), else 0.  positions (NULL or
 * nnz entries): the current record position of every training entry. */
int cmtf_gpu_order_blocks(cmtf_gpu_ctx *ctx, int32_t *blocks, uint32_t *positions);

/* ---- text formats and host-side data preparation ----
 * Host C++ (io.cpp), all host threads; no device is needed except for
 * cmtf_gpu_check_entries. */

/* parse_coo_file + infer_dims (src/sparse_data.cpp:124-227): the reference's
 * text format -- an optional dims header (detected from the first two data
 * lines), then one entry per line, 1-based indices and the value; '#'
 * comments and blank lines ignored.  expected_order 0 = any (load_tensor),
 * 2 = a matrix file (load_matrix).  Errors: CMTF_EPARSE with the reference's
 * ParseError message (line numbers included).  The parsed object owns
 * 0-based AoS indices and f64 values; dims = the header or the per-mode
 * maximum index.  threads <= 0: all hardware threads. */
typedef struct cmtf_coo cmtf_coo;
int cmtf_coo_parse(const char *path, int32_t expected_order, int32_t threads,
                   cmtf_coo **out);
int32_t cmtf_coo_order(const cmtf_coo *c);
uint64_t cmtf_coo_nnz(const cmtf_coo *c);
int32_t cmtf_coo_has_header(const cmtf_coo *c);
const uint32_t *cmtf_coo_dims(const cmtf_coo *c);
const uint32_t *cmtf_coo_indices(const cmtf_coo *c);
const double *cmtf_coo_values(const cmtf_coo *c);
void cmtf_coo_free(cmtf_coo *c);

/* write_coo (src/sparse_data.cpp:279-302) behind save_tensor / save_matrix:
 * the dims line, then "i1 .. iN %.17g" per entry (1-based). */
int cmtf_coo_write(const char *path, int32_t order, const uint32_t *dims,
                   const uint32_t *idx, const double *vals, uint64_t nnz,
                   int32_t threads);

/* check_entries (src/sparse_data.cpp:19-64), the validation of the
 * SparseTensor (is_matrix 0) and CoupledMatrix (is_matrix 1) constructors,
 * on the device: order >= 2 for tensors, positive dims, indices in range,
 * finite values, no duplicate tuples -- the reference's ValidationError
 * messages.  idx/vals: host or device pointers. */
int cmtf_gpu_check_entries(int32_t device, int32_t order, const uint32_t *dims,
                           const uint32_t *idx, const double *vals,
                           uint64_t nnz, int32_t is_matrix);

/* split_train_test (src/sparse_data.cpp:311-342): Fisher-Yates over the
 * entry ids with make_rng(seed, Split); test = the first
 * round(test_fraction * nnz) shuffled ids, train = the rest, both in
 * shuffled order.  Output buffers hold (nnz - n_test) / n_test entries; all
 * four NULL = size query (*n_test_out only). */
int cmtf_split_train_test(int32_t order, const uint32_t *idx, const double *vals,
                          uint64_t nnz, double test_fraction, uint64_t seed,
                          uint32_t *train_idx, double *train_vals,
                          uint32_t *test_idx, double *test_vals,
                          uint64_t *n_test_out, int32_t threads);

/* save_model (src/model_io.cpp:94-126): CORE (ranks line, row-major
 * values, J_N per line; a CP core -- its ranks[0] superdiagonal values --
 * is written densely), FACTOR n (rows cols, values), COUPLED m (rows cols,
 * values), 17 significant digits.  validate_model's checks
 * (src/tucker.cpp:208-224). */
int cmtf_model_save(const char *path, int32_t order, const uint32_t *ranks,
                    int32_t cp, const double *core, const uint32_t *factor_rows,
                    const double *const *factors, int32_t n_coupled,
                    const int32_t *coupled_modes, const uint32_t *coupled_rows,
                    const double *const *couplings);

/* load_model (src/model_io.cpp:128-179); the core is dense. */
typedef struct cmtf_model_file cmtf_model_file;
int cmtf_model_load(const char *path, cmtf_model_file **out);
int32_t cmtf_model_order(const cmtf_model_file *m);
const uint32_t *cmtf_model_ranks(const cmtf_model_file *m);
const double *cmtf_model_core(const cmtf_model_file *m);
uint32_t cmtf_model_factor_rows(const cmtf_model_file *m, int32_t n);
const double *cmtf_model_factor(const cmtf_model_file *m, int32_t n);
int32_t cmtf_model_n_coupled(const cmtf_model_file *m);
int32_t cmtf_model_coupled_mode(const cmtf_model_file *m, int32_t c);
uint32_t cmtf_model_coupled_rows(const cmtf_model_file *m, int32_t c);
const double *cmtf_model_coupled(const cmtf_model_file *m, int32_t c);
void cmtf_model_free(cmtf_model_file *m);

#ifdef __cplusplus
}
#endif
#endif /* CMTF_B200_H_ */
