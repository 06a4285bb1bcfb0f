/* potgpu.h — C-ABI of the B200-native entropic partial-OT solver.
 *
 * Drop-in boundary for the reference's header API (namespace pot in
 * /root/reference/proj/include/pot/). Plain pointers, sizes and POD structs
 * only; no C++ or torch types. The C++ mirror in include/pot/ (headers) converts
 * pot::Instance / SolverConfig <-> these structs and rethrows PotError, so a
 * reference user keeps calling pot::solve / aspot_solve / ... unchanged.
 *
 * Return codes: 0 on success, else 1 + the ordinal of the reference's
 * pot::ErrorCode (core.hpp:21-39, order preserved), or one of the
 * POTGPU_ERR_* device codes appended after it. potgpu_last_error() gives the
 * message (thread-local). No pointer passed in is retained after return.
 */
#ifndef POTGPU_H
#define POTGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POTGPU_ABI_VERSION 1

/* pot::ErrorCode ordinals + 1 (core.hpp:21-39). */
enum potgpu_status_code {
  POTGPU_OK = 0,
  POTGPU_DIMENSION_MISMATCH = 1,
  POTGPU_NEGATIVE_ENTRY = 2,
  POTGPU_NON_FINITE_ENTRY = 3,
  POTGPU_BUDGET_EXCEEDS_MASS = 4,
  POTGPU_OVERFLOW = 5,
  POTGPU_NON_POSITIVE_ARGUMENT = 6,
  POTGPU_DEGENERATE_INSTANCE = 7,
  POTGPU_PENALTY_TOO_SMALL = 8,
  POTGPU_UNBALANCED_MARGINALS = 9,
  POTGPU_ZERO_ENTROPY = 10,
  POTGPU_INFEASIBLE = 11,
  POTGPU_SIZE_LIMIT_EXCEEDED = 12,
  POTGPU_ZERO_MASS_PLAN = 13,
  POTGPU_DEGENERATE_SVD = 14,
  POTGPU_EMPTY_INPUT = 15,
  POTGPU_INVALID_ARGUMENT = 16,
  POTGPU_IO_FAILURE = 17,
  /* appended: device-side failures with no reference counterpart */
  POTGPU_ERR_CUDA = 18,
  POTGPU_ERR_NCCL = 19,
  POTGPU_ERR_UNSUPPORTED = 20
};

/* pot::SolverKind (core.hpp:223). */
enum potgpu_solver_kind { POTGPU_ASPOT = 0, POTGPU_FEASIBLE_SINKHORN = 1, POTGPU_TUNED_SINKHORN = 2 };
/* pot::BlockRule (core.hpp:221). */
enum potgpu_block_rule { POTGPU_GREEDY = 0, POTGPU_ROUND_ROBIN = 1 };
/* pot::SolveStatus (core.hpp:284). */
enum potgpu_solve_status { POTGPU_CONVERGED = 0, POTGPU_MAX_ITERATIONS_EXCEEDED = 1, POTGPU_STEP_SIZE_UNDERFLOW = 2 };
/* Arithmetic of the n^2 sweeps. F64: the reference's IEEE-double semantics.
 * F32: fp32 cost stream + MUFU ex2 with exact per-tile shifts, fp64
 * potentials and accumulation across tiles. */
enum potgpu_dtype { POTGPU_F64 = 0, POTGPU_F32 = 1 };
/* Cost representation. DENSE: stored n x n matrix streamed from HBM.
 * SQEUCLIDEAN: C_ij = cost_scale * |x_i - y_j|^2 regenerated per tile from
 * n x d point coordinates (d <= 4); never materialised. */
enum potgpu_cost_kind {
  POTGPU_COST_DENSE = 0,
  POTGPU_COST_SQEUCLIDEAN = 1,
  /* points given as for SQEUCLIDEAN, but the cost is built once on the device
   * and STORED (n x n in the problem dtype), then streamed like DENSE. */
  POTGPU_COST_SQEUCLIDEAN_STORED = 2
};

/* pot::Instance (core.hpp:108-118) plus the cost representation. Host
 * pointers, or device pointers on the context's device when device_ptrs = 1
 * (a dense C is then read in place; r, c and point coordinates, O(n), are
 * staged through the host for the setup logic). */
typedef struct potgpu_problem {
  int64_t n;
  int dtype;            /* potgpu_dtype */
  int cost_kind;        /* potgpu_cost_kind */
  /* DENSE: element (i, j) at C[i*ldc + j] if row_major, else C[i + j*ldc]
   * (Eigen's column-major MatrixXd layout, core.hpp:19). */
  const double* C;
  int64_t ldc;
  int row_major;
  /* SQEUCLIDEAN: X, Y are n x d row-major; cost_scale <= 0 means 1/max C. */
  const double* X;
  const double* Y;
  int d;
  double cost_scale;
  const double* r;
  const double* c;
  double s;
  int device_ptrs;
  /* device_ptrs = 1 only: where the arrays were produced, so the solver's
   * reads are ordered after the producer's writes (its context stream is a
   * non-blocking stream and does not synchronise with the default stream).
   * The __cuda_array_interface__ v3 "stream" convention:
   *   0  = unknown: the device is synchronised before the arrays are read
   *        (the zero-initialised default; always correct),
   *   1  = the legacy default stream, 2 = the per-thread default stream,
   *   -1 = the producer guarantees the arrays are complete (CAI "stream": None),
   *   else a cudaStream_t handle: the solver's stream waits on an event
   *        recorded on it (work queued there later is not waited for). */
  int64_t producer_stream;
} potgpu_problem;

/* pot::SolverConfig (core.hpp:241-267) + device options. */
typedef struct potgpu_config {
  double epsilon;            /* 0.1 */
  double gamma_override;     /* <= 0: derived (the reference's std::nullopt) */
  int64_t max_iterations;    /* 50000 */
  int block_rule;            /* POTGPU_GREEDY */
  double tuning_exponent_p;  /* 1.0 */
  int deterministic;         /* 1 (unused by the reference too, core.hpp:247) */
  int64_t log_every;         /* 1 */
  int record_rounded_cost;   /* 1: every trace record carries rounded_cost like the reference */
  int materialize_plan;      /* 1: write the dense n x n plan to outputs->X */
  int collect_iter_log;      /* 1: per-iteration decision log (outputs->iter_log) */
  int use_graphs;            /* 1: replay the per-attempt kernel sequence as a CUDA graph */
  int sync_every;            /* host polls the device state every k attempts (default 8) */
} potgpu_config;

typedef struct potgpu_trace_record {  /* pot::TraceRecord (core.hpp:269-275) */
  int64_t t;
  double error;
  double phi;
  double rounded_cost;  /* NaN when absent (std::nullopt) */
  double elapsed_s;
} potgpu_trace_record;

typedef struct potgpu_iter_log {  /* decision log of one accepted ASPOT iteration */
  int64_t t;
  int32_t halvings;
  int32_t block_hat;        /* Greenkhorn block picked at z_grave (solvers.hpp:340) */
  int32_t zbest_is_check;   /* phi(z_check) <= phi_hat (solvers.hpp:342) */
  int32_t block_check;      /* Greenkhorn block picked at z_best (solvers.hpp:344) */
  double error;
  double phi_check;
  double phi_hat;
  double theta;
} potgpu_iter_log;

/* pot::SolveResult scalars (solvers.hpp:176-186) + plan metrics. */
typedef struct potgpu_summary {
  int status;
  int64_t iterations;
  double gamma;
  double tolerance;
  double final_error;
  double wall_seconds;       /* the reference's definition (solver entry -> rounded plan) */
  double loop_seconds;       /* accepted-iteration loop only (iterations/s) */
  int has_bounds;
  double bound_R, bound_L, bound_mu_f, iteration_bound;
  double cost;               /* transport_cost(C, X) of the returned plan (core.hpp:199) */
  double feasibility_gap;    /* plan_feasibility_gap (core.hpp:207) */
  double mass;               /* 1^T X 1 */
  double phi;                /* dual value at the stopping iterate */
  int64_t trace_len;
  int64_t iter_log_len;
  int64_t sweeps;            /* n^2 passes executed on the device */
  int64_t attempts;          /* step attempts incl. halvings */
  char stopping_iterate[24]; /* "z_check" | "extended-marginals" | "trivial" */
} potgpu_summary;

/* Caller-owned optional outputs (NULL / 0 capacity = not wanted). */
typedef struct potgpu_outputs {
  double* X;            /* n x n row-major plan, needs config.materialize_plan */
  double* row_slack;    /* r - X 1 */
  double* col_slack;    /* c - X^T 1 */
  potgpu_trace_record* trace;
  int64_t trace_cap;
  potgpu_iter_log* iter_log;
  int64_t iter_log_cap;
  double* u;            /* final potentials (ASPOT: z_check; Sinkhorn: extended u[0..n], v[0..n]) */
  double* v;
  double* w;
} potgpu_outputs;

typedef struct potgpu_ctx potgpu_ctx;

int potgpu_abi_version(void);
const char* potgpu_last_error(void);
void potgpu_config_default(potgpu_config* cfg);

/* Context: owns the device, stream, workspaces and (optionally) the NCCL
 * communicator of a row-block-sharded multi-GPU solve. */
int potgpu_create(int device, potgpu_ctx** out);
int potgpu_destroy(potgpu_ctx* ctx);

/* pot::solve (solvers.hpp:591) / aspot_solve (:265) /
 * feasible_sinkhorn_solve (:516) / tuned_sinkhorn_solve (:547, :586). */
int potgpu_solve(potgpu_ctx* ctx, int solver_kind, const potgpu_problem* problem, const potgpu_config* config,
                 potgpu_summary* summary, potgpu_outputs* outputs);

/* Batched independent problems (BASELINE configs[4]; no reference
 * counterpart): `concurrency` workers (0 = 8), each with its own stream, run
 * complete solves concurrently. summaries[count]; outputs may be NULL or an
 * array of count entries. Returns the first failure (message names the
 * problem index). */
int potgpu_solve_batched(potgpu_ctx* ctx, int solver_kind, const potgpu_problem* problems, int64_t count,
                         const potgpu_config* config, potgpu_summary* summaries, potgpu_outputs* outputs,
                         int concurrency);

/* Step-wise form of potgpu_solve (no reference counterpart; used to time a
 * fixed number of iterations and to drive the loop from a host runtime):
 * begin = validation + setup + the first evaluation (+ record(0));
 * iterate = run until k more iterations are accepted or the solve stops
 * (k < 0: until it stops), device time of that loop in *device_ms;
 * finish = final rounding + outputs; a session still paused after iterate(k)
 * finishes exactly like a solve with max_iterations = t (status
 * MAX_ITERATIONS_EXCEEDED, the plan rounded at the current iterate).
 * potgpu_solve == begin; iterate(-1); finish. */
typedef struct potgpu_session potgpu_session;
int potgpu_session_begin(potgpu_ctx* ctx, int solver_kind, const potgpu_problem* problem, const potgpu_config* config,
                         int64_t trace_cap, int64_t iter_log_cap, potgpu_session** out);
int potgpu_session_iterate(potgpu_session* s, int64_t k, double* device_ms, int64_t* iterations, int* finished);
int potgpu_session_finish(potgpu_session* s, potgpu_summary* summary, potgpu_outputs* outputs);
int potgpu_session_destroy(potgpu_session* s);
/* Roofline probe: average device time of one hot-path sweep launch at the
 * session's current iterate (reps back-to-back launches between CUDA events
 * on the session stream), with the algorithmic elements (n^2 exponentials)
 * and HBM bytes (stored cost only) of one launch. */
int potgpu_session_time_sweep(potgpu_session* s, int reps, double* ms_per_sweep, double* elements, double* bytes);
/* Roofline probe of the accelerated solver's one-sided pass (fp32 on-the-fly
 * cost: z_check' when its Greenkhorn block is u (block = 0) or v (block = 1),
 * fused with the next z_bar when the session runs K1''; reference points:
 * solvers.hpp:345 and :337). Average device time of one launch at the
 * current z_check (n^2 exponentials). The session cannot iterate afterwards.
 * POTGPU_ERR_UNSUPPORTED for any other solver or cost representation. */
int potgpu_session_time_one_sided(potgpu_session* s, int reps, int block, double* ms_per_pass);
/* The accelerated solver's state after the last accepted iteration, for
 * the reference's AspotObserver (solvers.hpp:188-204, 364-367): point
 * which = 0 z_best, 1 z_check, 2 z_hat, 3 z_grave (u, v: n doubles; w: 1;
 * any may be NULL); scalars[6] = {t, theta, error, phi_hat, phi_best,
 * phi_check}. POTGPU_ERR_UNSUPPORTED for the Sinkhorn solvers. */
int potgpu_session_read_state(potgpu_session* s, int which, double* u, double* v, double* w, double scalars[6]);
/* Counters of the session so far: kernels launched by iterate(), step
 * attempts (incl. halvings) and n^2 sweeps executed. */
int potgpu_session_stats(potgpu_session* s, int64_t* kernel_launches, int64_t* attempts, int64_t* sweeps);
/* CTAs of the fp32 points sweep (sweep_pts2_f32) so far that exponentiated
 * at a carried shift / at the exact row maxima (both 0 for
 * other problem kinds or with POTGPU_CARRY=0). */
int potgpu_session_carry_stats(potgpu_session* s, int64_t* carried, int64_t* exact);
/* Device and pinned host blocks freed by finished solves are cached per
 * device and size class and reused by the next solve (no cudaMalloc /
 * cudaFree on the solve path after the first); this returns them all. */
void potgpu_release_cached_memory(void);
/* The context's CUDA stream (cudaStream_t), for callers that time with events. */
void* potgpu_ctx_stream(potgpu_ctx* ctx);

/* B(z) reductions at a dual point for logK = -C/gamma with marginals
 * (r, c, s) taken from `problem` as given (no mixing): the helpers
 * b_matrix / dual_objective / dual_gradient / feasibility_error
 * (dual.hpp:104-141) and greenkhorn_step's sums (solvers.hpp:46-52).
 * row/col: n doubles (B 1, B^T 1). scalars[6] = {total, max_exponent, phi,
 * feasibility_error, grad_w, overflow(0/1)}. Returns POTGPU_OVERFLOW exactly
 * when the reference's range checks would throw (scalars still filled). */
int potgpu_dual_eval(potgpu_ctx* ctx, const potgpu_problem* problem, double gamma, const double* u, const double* v,
                     double w, double* row, double* col, double* scalars);

/* exponent_matrix (which = 0) / b_matrix (which = 1) (dual.hpp:93-109) at
 * z = (u, v, w) for logK = -C/gamma of `problem` (fp64 semantics): out is
 * the dense n x n row-major matrix. POTGPU_OVERFLOW for B when the largest
 * exponent is not <= 700 (check_exp_range; out is still written). */
int potgpu_dual_matrix(potgpu_ctx* ctx, const potgpu_problem* problem, double gamma, const double* u, const double* v,
                       double w, int which, double* out);

/* round_pot (rounding.hpp:46-77) on the device for a dense row-major n x n
 * plan X (r, c, s validated as by validate(), core.hpp:131-169). */
int potgpu_round_pot(potgpu_ctx* ctx, int64_t n, const double* X, const double* r, const double* c, double s,
                     double* X_out);
/* round_balanced (rounding.hpp:14-39) on a dense row-major rows x cols plan;
 * POTGPU_UNBALANCED_MARGINALS when |r|_1 != |c|_1. */
int potgpu_round_balanced(potgpu_ctx* ctx, int64_t rows, int64_t cols, const double* X, const double* r,
                          const double* c, double* X_out);

/* Multi-GPU row-block sharding (no reference counterpart —
 * the reference is single-threaded). One process per GPU: rank 0 creates the
 * id, the caller broadcasts its 128 bytes (e.g. torch.distributed), then
 * every rank calls potgpu_comm_init on its context and runs the SAME solve
 * calls with the SAME full problem; each rank sweeps its contiguous block of
 * rows and one NCCL all-reduce per sweep combines the sums, so every rank
 * returns the same summary (a materialised plan holds the rank's own rows).
 * NCCL is loaded at run time (libnccl.so.2 or $POTGPU_NCCL_LIB);
 * POTGPU_ERR_NCCL when it is missing or fails. */
int potgpu_comm_unique_id(unsigned char id_out[128]);
int potgpu_comm_init(potgpu_ctx* ctx, int rank, int world_size, const unsigned char id[128]);
/* The context computes `shards` row shards itself (per rank when combined
 * with potgpu_comm_init) and reduces them with a fixed-order device sum: the
 * sharded arithmetic on one GPU, for testing; shards = 1 is the default. */
int potgpu_comm_init_local(potgpu_ctx* ctx, int shards);
int potgpu_comm_info(potgpu_ctx* ctx, int* rank, int* world_size, int* shards_per_rank);
/* Host collective backend: the same row-sharded job with the cross-process
 * reduction done by a caller-supplied function on host memory instead of
 * NCCL (MPI, gloo, a test harness; several processes may share one GPU).
 * `allreduce(buf, count, op, user)` must replace buf[0..count) in place with
 * the element-wise SUM (op = POTGPU_REDUCE_SUM) or MAX (POTGPU_REDUCE_MAX)
 * over the ranks, every rank calling it the same number of times in the
 * same order; it runs on a CUDA host-callback thread (it may block, it must
 * not call CUDA). Each sweep's all-reduce vector makes a device -> host ->
 * device round trip, so this is for correctness and portability, not speed. */
enum potgpu_reduce_op { POTGPU_REDUCE_SUM = 0, POTGPU_REDUCE_MAX = 2 };
typedef void (*potgpu_host_allreduce_fn)(double* buf, int64_t count, int op, void* user);
int potgpu_comm_init_host(potgpu_ctx* ctx, int rank, int world_size, potgpu_host_allreduce_fn allreduce, void* user);

/* Rigid point-cloud registration (registration.hpp).
 * pot::RegistrationConfig (registration.hpp:75-100) without `solve`, which
 * is passed as a potgpu_config. */
typedef struct potgpu_reg_config {
  double alpha;               /* 0.4: transported fraction of the smaller mass */
  double gamma0;              /* 4.4e-3: initial regularization */
  double anneal_rate;         /* 0.83: gamma multiplier per registration */
  double transform_threshold; /* 1e-5: stop when the increment falls below */
  int max_registrations;      /* 60 */
} potgpu_reg_config;

typedef struct potgpu_reg_record {  /* pot::RegistrationRecord (registration.hpp:102-109) */
  int32_t round;
  int64_t inner_iterations;
  int64_t accumulated_iterations;
  double cost;
  double increment;
  double gamma;
} potgpu_reg_record;

typedef struct potgpu_reg_result {  /* pot::RegistrationResult (registration.hpp:111-115) */
  double R[9];     /* row-major rotation of the transform mapping moving onto reference */
  double t[3];
  int converged;
  int64_t rounds;  /* registration rounds run (records written: min(rounds, cap)) */
} potgpu_reg_result;

void potgpu_reg_config_default(potgpu_reg_config* cfg);
/* register_point_clouds (registration.hpp:127-199): reference m x 3 and
 * moving n x 3 row-major host arrays; every round builds the padded
 * max(m,n)^2 cost on the device (fp64 coordinates; dtype = arithmetic of
 * the solves), solves it and fits the rigid increment from the implicit
 * plan (device moments, 3x3 SVD on the host). */
int potgpu_register_point_clouds(potgpu_ctx* ctx, int solver_kind, const double* reference, int64_t m,
                                 const double* moving, int64_t n, const potgpu_reg_config* reg,
                                 const potgpu_config* solve, int dtype, potgpu_reg_result* result,
                                 potgpu_reg_record* records, int64_t records_cap);
/* fit_rigid (registration.hpp:40-71) on a dense row-major m x n coupling pi
 * between x (m x 3) and y (n x 3): R (row-major 3x3) and t with x ~ R y + t. */
int potgpu_fit_rigid(potgpu_ctx* ctx, const double* pi, int64_t m, int64_t n, const double* x, const double* y,
                     double R[9], double t[3]);

/* Colour quantisation for colour transfer (color_transfer.hpp:34-118;
 * SURVEY.md §8(f) row 4): k-means++ seeding with the reference's
 * std::mt19937_64 draws (host, sequential by definition), Lloyd rounds on
 * the device until the largest centroid move < 1e-6 or 100 rounds.
 * points: n x 3 row-major; centroids k x 3 row-major; weights = cluster
 * sizes / n; assignments (may be NULL): n cluster indices. */
int potgpu_kmeans_quantize(potgpu_ctx* ctx, const double* points, int64_t n, int k, uint64_t seed, double* centroids,
                           double* weights, int32_t* assignments);

/* Synthetic fixtures: make_synthetic_instance (synthetic.hpp:15-54) and the
 * BASELINE.json config recipes. Host buffers:
 * r, c: n; C: n*n row-major (may be NULL for point configs); X, Y: n*3. */
int potgpu_make_synthetic(int64_t n, uint64_t seed, double mass_r, double mass_c, double s_frac, double* r, double* c,
                          double* C, double* s);
int potgpu_make_config(int config_id, int64_t n, uint64_t seed, double* r, double* c, double* X, double* Y, int* d,
                       double* s, double* cost_scale);

#ifdef __cplusplus
}
#endif

#endif /* POTGPU_H */
