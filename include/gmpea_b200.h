/* gmpea_b200.h — C ABI of the B200-native GMPEA engine (libgmpea_b200.so).
 *
 * Plain pointers and sizes only; every host array is row-major f64 exactly as
 * the reference's gmpea::Matrix (proj/include/gmpea/matrix.hpp:13-31).  Each
 * entry point replaces one reference interface, cited per function.  The
 * device holds fp32 structure-of-arrays copies; results come back as f64.
 *
 * Errors: every int-returning call returns GMPEA_OK or an error code and
 * leaves a message retrievable with gmpea_last_error() (thread-local).  The
 * messages reproduce the reference's exception texts; GMPEA_EINVAL maps to
 * std::invalid_argument, GMPEA_ERUNTIME to std::runtime_error.  There is no
 * CPU fallback: without a usable sm_100 device every compute call returns
 * GMPEA_ECUDA.
 *
 * Threading: a gmpea_engine is one run (single writer, gmpea.hpp:140-144);
 * distinct engines and the stateless operator calls may be used from
 * different threads.
 */
#ifndef GMPEA_B200_H
#define GMPEA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GMPEA_OK 0
#define GMPEA_EINVAL 1   /* std::invalid_argument in the reference */
#define GMPEA_ERUNTIME 2 /* std::runtime_error in the reference */
#define GMPEA_ECUDA 3    /* CUDA runtime failure / no device */
#define GMPEA_ENCCL 4    /* NCCL failure (sharded multi-process runs) */

#define GMPEA_OP_SBX_PM 0 /* VariationOp::sbx_pm (gmpea.hpp:56) */
#define GMPEA_OP_DE 1     /* VariationOp::de */

/* subproblem aggregation of the selection keys: PBI (scalarize.cpp:72-89, the
 * reference's only one) or the weighted Tchebycheff function
 * g = max_k max(w_k, 1e-6) |f_k - z_k| the north-star names (an engine
 * extension without a reference counterpart: parity against the oracle's
 * f64 restatement only) */
#define GMPEA_AGG_PBI 0
#define GMPEA_AGG_TCH 1

typedef struct gmpea_problem gmpea_problem;
typedef struct gmpea_engine gmpea_engine;

const char* gmpea_last_error(void);
int gmpea_abi_version(void);

/* ---- problems: replaces make_problem / ProblemDef (problems.hpp:19-45,
 * problems.cpp:531-550) and make_wta_problem / load_wta (wta.hpp:30-48).
 * Names: LIRCMOP1..14, C1-DTLZ1, C1-DTLZ3, C2-DTLZ2, C3-DTLZ4,
 * DC{1,2,3}-DTLZ{1,3}, WTA-P1..P10, MW1..MW14, DASCMOP1..9 (alias DAS-CMOP1..9;
 * MW and DAS-CMOP are not in the reference: restated, parity unpinned). */
int gmpea_problem_create(const char* name, gmpea_problem** out);
/* custom WTA scenario (load_wta, wta.cpp:148-192): p holds sum(strikes)
 * interception probabilities, target-major */
int gmpea_problem_create_wta(const char* scenario, int32_t targets, int32_t vehicles,
                             const int32_t* strikes, const int32_t* capacity, const double* p,
                             gmpea_problem** out);
/* built-in scenario tables P1..P10 (wta_scenario, wta.cpp:23-49); host-only.
 * strikes: targets entries, capacity: vehicles entries, p: sum(strikes) */
int gmpea_wta_scenario(int32_t num, int32_t* targets, int32_t* vehicles, int32_t* strikes,
                       int32_t* capacity, double* p);
int gmpea_problem_info(const gmpea_problem* p, int32_t* d, int32_t* m, int32_t* n_ineq,
                       int32_t* n_eq);
int gmpea_problem_bounds(const gmpea_problem* p, double* lo, double* hi);
void gmpea_problem_destroy(gmpea_problem* p);
/* names of all registered problems, '\n'-separated (problem_names, problems.cpp:531-540) */
const char* gmpea_problem_names(void);

/* ---- evaluation: replaces evaluate (problems.hpp:47-51, problems.cpp:552-573)
 * plus cv_batch (evaluate_population, gmpea.cpp:15-23).  X: n x d; F: n x m;
 * G: n x (n_ineq + n_eq) raw constraints (<= 0 feasible); cv: n (may be NULL).
 * Rows outside the bounds (or NaN) fail with GMPEA_EINVAL
 * "evaluate: out-of-bounds rows: r1 r2 ...". */
int gmpea_evaluate(const gmpea_problem* p, const double* X, int64_t n, double* F, double* G,
                   double* cv);

/* ---- reference vectors and neighbourhoods (gmpea.hpp:37-51, gmpea.cpp:27-100) */
int gmpea_reference_vectors(int32_t m, int64_t n, double* W);
/* t-NN of arbitrary W (n x m, m <= 3) by fp64 distance, ties to the lower index */
int gmpea_build_neighborhoods(const double* W, int64_t n, int32_t m, int32_t t1, int32_t t2,
                              uint32_t* B1, uint32_t* B2);
/* same, for W = reference_vectors(m, n), by a provably sufficient window */
int gmpea_lattice_neighborhoods(int32_t m, int64_t n, int32_t t1, int32_t t2, uint32_t* B1,
                                uint32_t* B2);

/* ---- variation: replaces reproduce (gmpea.hpp:56-73, gmpea.cpp:113-206).
 * The reference draws from one mt19937_64 stream (rng.hpp); the engine draws
 * from Philox4x32-10 keyed by (seed; slot, gen, pop, stream, index) — see
 * DESIGN.md "Random streams".  pm_prob < 0 means 1/d. */
typedef struct {
    double sbx_prob, sbx_eta, pm_eta, de_cr, de_f, pm_prob;
} gmpea_operator_params;
int gmpea_operator_params_default(gmpea_operator_params* out);
int gmpea_reproduce(const gmpea_problem* p, const double* X, int64_t n, const uint32_t* nbrs,
                    int32_t t, int32_t op, const gmpea_operator_params* params, uint64_t seed,
                    uint32_t gen, uint32_t pop, double* off);

/* ---- environmental selection: replaces op1/op2/op3 and
 * environmental_selection (gmpea.hpp:75-111, gmpea.cpp:248-399).
 * Populations are (X n x d, F n x m, C n x nc, cv n).  Outputs are assembled
 * from the f64 inputs, so surviving rows are bit-identical copies.
 * winner[j] (optional): -1 parent kept, c in [0,n): off1 row c,
 * n + c: off2 row c (the row the offspring stream held after OP1). */
typedef struct {
    const double *X, *F, *C, *cv;
} gmpea_population_view;
typedef struct {
    double *X, *F, *C, *cv;
} gmpea_population_out;
int gmpea_environmental_selection(int64_t n, int32_t d, int32_t m, int32_t nc,
                                  const gmpea_population_view* pop1,
                                  const gmpea_population_view* pop2,
                                  const gmpea_population_view* off1,
                                  const gmpea_population_view* off2, const double* W,
                                  const double* z, double theta, const uint32_t* B1, int32_t t1,
                                  const uint32_t* B2, int32_t t2, gmpea_population_out* out1,
                                  gmpea_population_out* out2, int32_t* winner1, int32_t* winner2);
/* the same with the aggregation chosen (GMPEA_AGG_*; theta is used by PBI only) */
int gmpea_environmental_selection_ex(int64_t n, int32_t d, int32_t m, int32_t nc,
                                     const gmpea_population_view* pop1,
                                     const gmpea_population_view* pop2,
                                     const gmpea_population_view* off1,
                                     const gmpea_population_view* off2, const double* W,
                                     const double* z, double theta, int32_t aggregation,
                                     const uint32_t* B1, int32_t t1, const uint32_t* B2, int32_t t2,
                                     gmpea_population_out* out1, gmpea_population_out* out2,
                                     int32_t* winner1, int32_t* winner2);

/* ---- metrics: replaces igd / hypervolume / metric_front (metrics.hpp:15-29) */
int gmpea_igd(const double* A, int64_t na, const double* R, int64_t nr, int32_t m, double* out);
int gmpea_metric_front(const double* F, const double* cv, int64_t n, int32_t m, int64_t* idx,
                       int64_t* count);
int gmpea_hypervolume(const double* P, int64_t n, int32_t m, const double* ref, double* out);
/* replaces pf_reference (fronts.cpp:54-84, fronts.hpp): the problem's analytic
 * front candidates built and evaluated in fp64 on the device, feasible rows
 * only, nondominated-filtered, subsampled to n_points (subsample_front).
 * Writes *rows (<= n_points unless the front is smaller) rows of m values;
 * MW / DAS-CMOP (restated suites) use restated candidates: per position the
 * smallest feasible distance value (level scan + bisection), realised in
 * decision space.  Fails (status 2, the reference's runtime_error text) for
 * WTA (no analytic front).  cap: capacity of out in rows. */
int gmpea_pf_reference(const gmpea_problem* p, int64_t n_points, double* out, int64_t cap, int64_t* rows);

/* ---- comparison-algorithm operators: replace baselines.hpp (baselines.cpp:22-190).
 * fp64 inputs, row-major F (n x m); results equal the reference's exactly.
 * use_cdp: constrained domination (cdp_better) instead of pareto_dominates;
 * a negative cv is rejected as cdp_better does. */
int gmpea_nondominated_sort(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp,
                            int64_t* rank);
int gmpea_crowding_distance(const double* F, int64_t n, int32_t m, const int64_t* front, int64_t k,
                            double* dist);
int gmpea_spea2_fitness(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp, double* fit);
/* keep: capacity >= min(n, capacity) entries; *count rows kept, ascending */
int gmpea_spea2_select(const double* F, const double* cv, int64_t n, int32_t m, int32_t use_cdp,
                       int64_t capacity, int64_t* keep, int64_t* count);

/* ---- the run: replaces run_gmpea (gmpea.hpp:113-144, gmpea.cpp:421-493) */
typedef struct {
    int64_t n;             /* requested population size */
    int64_t k_max;         /* generation cap (0 = unbounded when a budget is set) */
    double time_budget_s;  /* <= 0: none */
    int64_t eval_budget;   /* <= 0: none */
    uint64_t seed;
    int32_t op;            /* GMPEA_OP_* */
    gmpea_operator_params params;
    double theta;
    int32_t t1, t2;
    int32_t record_walltime;
    /* engine extensions */
    int32_t device;        /* CUDA device ordinal */
    uint64_t stream;       /* cudaStream_t to run on; 0 = the engine's own stream */
    /* optional per-generation IGD hook (RunConfig::igd_metric, gmpea.hpp:123,
     * as the harness installs it, experiment.cpp:200-205): igd(metric_front(
     * pop1), igd_reference) on the device after generation 0 and every kept
     * generation, outside the loop clock; GenRecord.igd / has_igd carry it.
     * igd_reference: igd_reference_rows x m, copied at create.  Unsharded runs. */
    const double* igd_reference;
    int64_t igd_reference_rows;
    /* weight-region sharding: this engine owns the slots
     * [shard_begin, shard_end) of n; 0, 0 = all of them */
    int64_t shard_begin, shard_end;
    int32_t aggregation;   /* GMPEA_AGG_PBI (default, the reference's) or GMPEA_AGG_TCH */
    /* weight-region sharding over NCCL, one process per GPU:
     * world > 1 ranks, this process is `rank` and owns the balanced slot range
     * [rank n / world, (rank + 1) n / world); nccl_id points to the 128-byte
     * id gmpea_nccl_unique_id made on rank 0 and the caller shared.  The
     * ideal-point all-reduce and the boundary-row exchange run inside every
     * generation's CUDA graph; rank 0 keeps the loop clock of a time budget. */
    int32_t world, rank;
    const void* nccl_id;
} gmpea_run_config;

typedef struct {
    int64_t gen, evals;
    double wall_ms, feasible_ratio;
    double igd, hv;
    int32_t has_igd, has_hv;
} gmpea_gen_record;

int gmpea_run_config_default(gmpea_run_config* out);
/* setup: reference vectors, neighbourhoods, initial populations (Philox INIT
 * stream), their evaluation, the ideal point and record 0 */
/* comparison algorithms as whole runs: replace run_cnsga2 / run_ccmo
 * (baselines.cpp:320-459, baselines.hpp:33-34) on the device.  cfg: n, k_max,
 * time_budget_s, eval_budget, seed, params (SBX + PM, the operator field is
 * ignored as in the reference), record_walltime, device.  igd_ref (n_ref x m,
 * optional): the IGD metric hook of experiment.cpp:200-205, evaluated on the
 * device after every generation outside the loop clock.  Writes the history
 * (up to hist_cap rows; *n_hist = all) and pop1 (n x d, n x m,
 * n x (n_ineq + n_eq), n). */
#define GMPEA_ALGO_CNSGA2 0
#define GMPEA_ALGO_CCMO 1
/* host metric hook (RunConfig::igd_metric / hv_metric, gmpea.hpp:123-124):
 * called with pop1 (n rows, host memory) after every generation, outside the
 * loop clock; sets *igd / *hv and the has_ flags for the values it computed */
typedef void (*gmpea_pop_hook)(void* user, int64_t n, const double* X, const double* F, const double* C,
                               const double* cv, double* igd, double* hv, int32_t* has_igd, int32_t* has_hv);
int gmpea_run_baseline(const gmpea_problem* p, int32_t algo, const gmpea_run_config* cfg,
                       const double* igd_ref, int64_t n_ref, gmpea_pop_hook hook, void* hook_user,
                       gmpea_gen_record* hist, int64_t hist_cap, int64_t* n_hist, double* X, double* F,
                       double* C, double* cv);

int gmpea_engine_create(const gmpea_problem* p, const gmpea_run_config* cfg, gmpea_engine** out);
/* one handle driving a sharded run over several devices of this process
 * (SURVEY.md §8(b) devices[] / ndev): shard k on devices[k] owns the balanced
 * slot range k of ndev; each generation is one multi-device CUDA graph (ideal
 * point MIN over peer memory, boundary rows by peer copies).  Every other
 * gmpea_engine_* call works on the handle as on an unsharded engine (pop1 /
 * history of all N slots).  A device may repeat (shards sharing a GPU). */
int gmpea_engine_create_multi(const gmpea_problem* p, const gmpea_run_config* cfg, const int32_t* devices,
                              int32_t ndev, gmpea_engine** out);
/* a new NCCL unique id (128 bytes) for gmpea_run_config.nccl_id */
int gmpea_nccl_unique_id(void* id128);
/* replace population `which` (1 or 2) by host rows X (n x d) and re-evaluate.
 * Asynchronous (stream-ordered, no host round trip): rows outside the bounds
 * are reported as evaluate's GMPEA_EINVAL "evaluate: out-of-bounds rows: ..."
 * by the next call that synchronises (step's successors, sync, population,
 * history); pass pinned host memory for a truly asynchronous copy. */
int gmpea_engine_set_population(gmpea_engine* e, int32_t which, const double* X);
/* run to completion under k_max / eval_budget / time_budget semantics */
int gmpea_engine_run(gmpea_engine* e);
/* enqueue up to `gens` more generations (no host sync) */
int gmpea_engine_step(gmpea_engine* e, int64_t gens);
int gmpea_engine_sync(gmpea_engine* e);
int64_t gmpea_engine_effective_n(const gmpea_engine* e);
int gmpea_engine_history(gmpea_engine* e, gmpea_gen_record* out, int64_t cap, int64_t* n);
/* the newest record only (blocks until the enqueued generations finished) */
int gmpea_engine_last_record(gmpea_engine* e, gmpea_gen_record* out);
/* diagnostic (no reference counterpart; SURVEY.md §8d "report the replacement
 * rate"): per generation, the number of owned slots of both populations that
 * took an offspring in OP3; out[0] (initialisation) is 0.  Same indexing and
 * count semantics as gmpea_engine_history. */
int gmpea_engine_replacements(gmpea_engine* e, int64_t* out, int64_t cap, int64_t* n);
/* the newest enqueued generation's raw record, copied to host memory dst
 * (pinned for a true async copy) in stream order WITHOUT waiting: the
 * per-step result of a pipelined loop, read by the caller after its next
 * gmpea_engine_sync.  Layout of the 16 bytes: */
typedef struct {
    uint32_t feasible; /* rows of pop1 (owned slots) with cv == 0 */
    uint32_t replaced; /* owned slots of both populations that took an offspring */
    uint64_t loop_ns;  /* accumulated loop time (device clock) */
} gmpea_raw_record;
int gmpea_engine_record_async(gmpea_engine* e, gmpea_raw_record* dst);
int gmpea_engine_get_population(gmpea_engine* e, int32_t which, double* X, double* F, double* C,
                                double* cv);
/* diagnostic (parity harness): offspring stream `which` (1: off1, 2: off2) of
 * the last generation exactly as variation + evaluation produced it, before
 * OP1 (gmpea.cpp:463-468); same layout as gmpea_engine_get_population */
int gmpea_engine_get_offspring(gmpea_engine* e, int32_t which, double* X, double* F, double* C,
                               double* cv);
int gmpea_engine_ideal(gmpea_engine* e, double* z);
/* neighbourhood tables the run uses (n x t1, n x t2) */
int gmpea_engine_neighborhoods(gmpea_engine* e, uint32_t* B1, uint32_t* B2);
/* run `gens` generations kernel by kernel with CUDA events around each launch
 * and return the average device milliseconds of [vary_eval, op1, select,
 * end_gen] plus the total per generation in ms[4] */
int gmpea_engine_profile(gmpea_engine* e, int64_t gens, double* ms);
void gmpea_engine_destroy(gmpea_engine* e);

/* ---- sharded runs (one engine per GPU).  Slot ranges are
 * global; the engine keeps parent rows for [window_begin, window_end) =
 * own +- 2*reach, regenerates offspring for [vary_begin, vary_end) = own +-
 * reach (Philox keys are global, so they equal their owners' offspring) and
 * selects its own slots. */
typedef struct {
    int64_t n_global, window_begin, window_end, vary_begin, vary_end, own_begin, own_end, reach;
} gmpea_shard_info;
int gmpea_engine_shard_info(gmpea_engine* e, gmpea_shard_info* out);
/* one generation in two phases: 1 = variation + evaluation (+ local ideal
 * point), 2 = OP1 + selection + bookkeeping.  Between them the caller
 * all-reduces (MIN) the ideal-point words; after phase 2 it exchanges the
 * boundary rows (own +- 2*reach) with the neighbouring shards. */
int gmpea_engine_phase(gmpea_engine* e, int32_t phase);
typedef struct {
    void* ideal_bits;  /* uint32[4], order-preserving encoding of the ideal point (all-reduce MIN) */
    void* rows[2];     /* pop1 / pop2 rows; window-local row r at rows + r * row_bytes */
    void* keys[2];     /* pop1 / pop2 packed keys {f0, f1, f2, cv}, 16 bytes per row */
    int64_t row_bytes;
} gmpea_device_buffers;
int gmpea_engine_device_buffers(gmpea_engine* e, gmpea_device_buffers* out);

#ifdef __cplusplus
}
#endif
#endif
