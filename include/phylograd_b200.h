/*
 * phylograd-b200 C-ABI — the drop-in boundary for the logL + branch-gradient
 * hot path of phylograd (reference: /root/reference/proj/include/phylograd).
 *
 * The reference exposes the path as the header-only C++ class
 * phylograd::LikelihoodEngine (engine.hpp:47-438) with no FFI.  Each entry
 * point below replaces one piece of that class (cited per function); the C++
 * facade in include/phylograd_b200/engine.hpp rebuilds the reference's class
 * surface on top of these calls, and paper_1905_12146_b200/ mirrors it in
 * Python.  Plain pointers and sizes only; all arrays are HOST memory unless a
 * name says _device.  No CPU fallback: every compute call runs CUDA kernels on
 * the engine's device and fails with PG_ERR_CUDA if that is impossible.
 *
 * Node numbering follows the reference (tree.hpp:6-8): tips 1..N, internal
 * nodes N+1..2N-1, root 2N-1; branch i is named by its child node, output
 * index i-1.
 */
#ifndef PHYLOGRAD_B200_H
#define PHYLOGRAD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The facade rethrows them as the reference's exception types
 * (engine.hpp:58-70, :117-120, :211-215, :226-227; tree.hpp:141-146). */
enum pg_status {
  PG_OK = 0,
  PG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  PG_ERR_RUNTIME = 2,          /* std::runtime_error ("underflowed", "non-finite") */
  PG_ERR_LOGIC = 3,            /* std::logic_error (pass ordering) */
  PG_ERR_NEWICK = 4,           /* phylograd::NewickError (position in pg_last_error) */
  PG_ERR_CUDA = 5,             /* device / driver failure */
  PG_ERR_NOT_SUPPORTED = 6,
  PG_ERR_NCCL = 7              /* NCCL load / communicator / collective failure */
};

/* Evaluation flags for pg_evaluate (engine.hpp:146-164; clock.hpp:146-152). */
enum pg_eval_flags {
  PG_EVAL_LOGL = 1,      /* log_likelihood() */
  PG_EVAL_GRAD = 2,      /* branch_gradient(): d logL / d b_i */
  PG_EVAL_HESS = 4,      /* branch_gradient(true): Hessian diagonal */
  PG_EVAL_RATE_GRAD = 8, /* chain rule to branch rates: d logL / d r_i = dt_i * g_i (needs durations) */
  PG_EVAL_FORCE = 16,    /* recompute even when caches are valid (invalidate_caches()) */
  PG_EVAL_POST_PASS = 32, /* logL through the cached post-order route: post_order_pass() (engine.hpp:182) */
  PG_EVAL_REQUIRE_POST = 64 /* pre_order_pass(): PG_ERR_LOGIC unless the post pass is current (engine.hpp:226-227) */
};

/* engine.hpp:33-37 EngineOptions + device placement. */
typedef struct pg_options {
  double rescaling_threshold; /* default 1e-150 */
  int force_rescaling;        /* rescale at every internal visit */
  int disable_rescaling;      /* never rescale (testing only) */
  int device;                 /* CUDA ordinal */
  int capture_partials;       /* keep per-node post/pre partials for pg_get_partials (debug, small P) */
  int reserved[8];
} pg_options;

typedef struct pg_engine pg_engine;

void pg_default_options(pg_options* opt);
/* Thread-local text of the last failure (also after a failed pg_create). */
const char* pg_last_error(void);

/* ---- engine lifecycle (replaces the LikelihoodEngine ctor, engine.hpp:49-110).
 * The reference holds const references to tree/alignment/model (:416-418);
 * the C-ABI copies everything to the device instead, so callers may free
 * their host arrays after each setter returns. */
int pg_create(const pg_options* opt, pg_engine** out);
void pg_destroy(pg_engine* e);

/* ---- multi-GPU from one process (SURVEY.md §8b pg_create(desc{G, devices}),
 * §8e).  Patterns shard contiguously: entry r of `devices` owns patterns
 * [floor(r P / G), floor((r+1) P / G)) and runs both traversals locally; one
 * reduction of [logL, g (2N-2), h (2N-2)] per evaluation combines them:
 *  - PG_REDUCE_NCCL: ncclCommInitAll over the device list (distinct devices)
 *    and one in-place ncclAllReduce(sum, float64) per shard stream inside
 *    ncclGroupStart/End (libnccl.so.2 is loaded at this call, not at link time);
 *  - PG_REDUCE_FIXED_ORDER: every shard's result is copied to the first
 *    device (peer copy) and summed in rank order 0..G-1 by one kernel, so the
 *    result is bit-reproducible for a fixed device list; repeated devices
 *    are allowed (several shards on one GPU).
 * The returned handle takes every setter and pg_evaluate / pg_clock_gradient
 * like a single-device engine (callers such as clock.hpp:146-147 and
 * cli.hpp:313-317 need no change); device-pointer entry points, pg_set_stream
 * and the debug partial accessors return PG_ERR_NOT_SUPPORTED on a group. */
enum pg_reduce { PG_REDUCE_NCCL = 0, PG_REDUCE_FIXED_ORDER = 1 };
int pg_create_multi(const pg_options* opt, int device_count, const int* devices, int reduce_mode, pg_engine** out);
/* shard_count (1 for a single-device engine), NCCL version (0 unless the
 * NCCL reduction is in use), reduce mode. */
int pg_group_info(const pg_engine* e, int* shard_count, int* nccl_version, int* reduce_mode);

/* tree.hpp:27-77: parent[2N] (parent[root]=0), children[2N][2] ({0,0} for
 * tips), post_order[2N-1] (validated as an admissible order: children before
 * parents, tree.hpp:81-126).  Branch lengths come from pg_set_branch_lengths. */
int pg_set_topology(pg_engine* e, int tip_count, const int32_t* parent, const int32_t* children,
                    const int32_t* post_order);

/* alignment.hpp:129-238 + engine.hpp:64-79 (tip codes).  codes is tip-major
 * [tip_count][pattern_count] int8 (compact tip codes; the reference keeps
 * dense m x P tip partials, alignment.hpp:219-227): 0..m-1 = observed state,
 * -1 = missing (all-ones partial), m+a = ambiguity class a whose partial is
 * ambiguity[a*m .. a*m+m) (m + ambiguity_count <= 127).  weights are the
 * integer pattern multiplicities (alignment.hpp:135). */
int pg_set_patterns(pg_engine* e, int state_count, int pattern_count, const int8_t* codes,
                    int ambiguity_count, const double* ambiguity, const int64_t* weights);

/* substitution.hpp:81-93 raw constructor: q row-major m x m (rows sum to 0),
 * pi root distribution.  reversible != 0 and pi > 0 builds the symmetric
 * eigensystem (substitution.hpp:196-208); otherwise P(t) uses Pade
 * scaling-and-squaring (substitution.hpp:155-156), both on the GPU. */
int pg_set_model(pg_engine* e, int state_count, const double* q, const double* pi, int reversible);
/* substitution.hpp:138-143: raw per-branch generator (non-homogeneous). */
int pg_set_branch_generator(pg_engine* e, int branch, const double* q);

/* substitution.hpp:23-51 (RateCategories::make checks). */
int pg_set_categories(pg_engine* e, int category_count, const double* rates, const double* probs);

/* engine.hpp:116-124: validates size/finiteness/sign; a bit-identical vector
 * keeps the caches valid.  b has 2N-2 entries (index node-1). */
int pg_set_branch_lengths(pg_engine* e, const double* b);
/* Same, reading a DEVICE pointer (no host round trip). */
int pg_set_branch_lengths_device(pg_engine* e, const double* b_device);
int pg_get_branch_lengths(pg_engine* e, double* b);

/* clock.hpp:42-55 / cli.hpp:429-440: calendar durations dt_i = t_i - t_pa(i)
 * used by PG_EVAL_RATE_GRAD (d logL / d r_i = dt_i g_i, b_i = r_i dt_i). */
int pg_set_clock_durations(pg_engine* e, const double* dt);

/* clock.hpp:140-152 and :199-213: the relaxed-clock chain rule from one
 * branch-gradient evaluation at the current lengths b_i = r_i dt_i (cached
 * like pg_evaluate(PG_EVAL_GRAD)), computed on the GPU:
 *   dlog_eps[i] = d logL / d log eps_i = b_i g_i            (2N-2, may be NULL)
 *   *dlog_mu    = d logL / d log mu    = sum_i b_i g_i      (fixed order, may be NULL)
 *   dnode_time[k] = d logL / d t_{N+1+k}
 *                 = r_{N+1+k} g_{N+1+k} [non-root] - sum_children r_c g_c  (N-1, may be NULL)
 * rates[2N-2] are the branch rates r_i = mu eps_i (host); NULL derives them
 * as b_i / dt_i from pg_set_clock_durations.  log_likelihood may be NULL. */
int pg_clock_gradient(pg_engine* e, const double* rates, double* log_likelihood, double* dlog_mu, double* dlog_eps,
                      double* dnode_time);

/* engine.hpp:146-164.  Synchronous: returns when results are in host memory.
 * log_likelihood may be NULL; grad/hess (2N-2 doubles) may be NULL unless the
 * matching flag is set.  With PG_EVAL_RATE_GRAD, grad receives dt_i*g_i and
 * hess dt_i^2*H_ii. */
int pg_evaluate(pg_engine* e, int flags, double* log_likelihood, double* grad, double* hess);

/* Asynchronous variant for multi-GPU sharding: writes [logL, g(2N-2), h(2N-2)]
 * (h only with PG_EVAL_HESS) into out_device on the engine stream; the caller
 * all-reduces it (NCCL) and then calls pg_check_errors. */
int pg_evaluate_device(pg_engine* e, int flags, double* out_device);
int pg_check_errors(pg_engine* e);

/* Run on a caller-provided cudaStream_t (e.g. torch's current stream). */
int pg_set_stream(pg_engine* e, void* cuda_stream);

/* engine.hpp:134-141 debug accessors (needs capture_partials): m x P
 * column-major partials of one (node, category) and the per-pattern log
 * scalers; values are scaled: true partial = partial * exp(scaler). */
int pg_get_partials(pg_engine* e, int node, int category, double* post, double* pre, double* post_scaler,
                    double* pre_scaler);
/* Per-pattern site log-likelihoods of the last evaluation (P doubles). */
int pg_get_site_log_likelihoods(pg_engine* e, double* out);

/* engine.hpp:126-130 instrumentation. */
uint64_t pg_node_visits(const pg_engine* e);
void pg_reset_node_visits(pg_engine* e);
void pg_invalidate_caches(pg_engine* e);

/* Introspection for benchmarks: kernels launched by the last evaluation,
 * average device ms of the walk kernel over the last evaluation, and the
 * launch geometry that evaluation used (the geometry is chosen lazily at the
 * first evaluation after a topology / pattern / model change). */
int pg_engine_info(const pg_engine* e, int* launches, int* total_warps, int* lanes_per_pattern, int* padded_states);
int pg_last_walk_ms(const pg_engine* e, float* walk_ms, float* total_ms);
/* Walk-kernel variant of the current geometry: 0 generic register-tiled
 * walk_kernel<MP,LC>, 1 pipelined 4-state walk4_kernel, 2 DMMA large-state walkm_kernel,
 * 3 level-scheduled walkl_kernel, 4 single-buffered 4-state walk4s_kernel, 5 tensor-core 4-state
 * walk4t_kernel. */
int pg_engine_variant(const pg_engine* e);
/* Per-evaluation CUDA-event timing on the engine stream: returns the number of
 * evaluations recorded since the previous call and the summed device ms of the
 * walk kernel and of whole evaluations, then resets and (dis)arms recording. */
int pg_timing(pg_engine* e, int enable, int* evaluations, double* walk_ms_total, double* eval_ms_total);

/* ---- setup-side formats either side of the path ---- */
/* tree.hpp:144-289 parse_newick: two calls — first with arrays NULL to learn
 * tip_count, then with parent[2N], children[2N*2], branch_length[2N] (index =
 * node, [root] = 0), post_order[2N-1]; labels written NUL-separated into
 * label_buf (tips 1..N). */
int pg_newick_parse(const char* text, int* tip_count, int32_t* parent, int32_t* children, double* branch_length,
                    int32_t* post_order, char* label_buf, int64_t label_cap);

/* alignment.hpp:186-229 from_codes compression, first-occurrence order.
 * codes [ntax][sites] int32 in -1..m-1 (validated).  Returns a handle and the
 * pattern count; pg_compress_result then writes pattern_codes [ntax][P]
 * (int32), weights[P] and site_to_pattern[sites] (each skipped when NULL).  Hashing is
 * multithreaded; the output order is bit-exact with the reference's std::map
 * first-occurrence order. */
int pg_compress_codes(int ntax, int64_t sites, const int32_t* codes, int state_count, void** handle,
                      int* pattern_count);
int pg_compress_result(void* handle, int32_t* pattern_codes, int64_t* weights, int32_t* site_to_pattern);
void pg_compress_free(void* handle);

/* The same compression on the GPU (pg_compress.cu):
 * codes int8 [ntax][sites] (host memory, or device memory on `device` when
 * codes_on_device != 0), values -1..m-1.  Bit-exact with pg_compress_codes:
 * first-occurrence pattern order, int64 weights, site -> pattern map; hash
 * collisions are detected by a full column comparison and re-hashed.
 * pg_compress_result_gpu copies the results to host arrays (any may be NULL)
 * and reports the device time of the compression kernels. */
int pg_compress_codes_gpu(int ntax, int64_t sites, const int8_t* codes, int codes_on_device, int state_count,
                          int device, void** handle, int* pattern_count);
int pg_compress_result_gpu(void* handle, int8_t* pattern_codes, int64_t* weights, int32_t* site_to_pattern,
                           float* device_ms);
void pg_compress_free_gpu(void* handle);

/* alignment.hpp:243-286 forward simulation on the GPU:
 * per site the rate category, then the nodes in pre-order (the reverse of
 * post_order, tree.hpp:76) -- the root from pi, the rest from the row of
 * P(b_node c_l) of the parent's state (substitution.hpp:147-160) -- then a
 * missing tip (-1) with probability gap_fraction per (taxon, site).  The
 * reference draws from one sequential mt19937_64 stream; here draw k of site
 * s is splitmix64 at counter s (3N-1+1) + k of `seed`, so sites are
 * independent (one thread each) and the result is bit-identical with the
 * CPU twin in workloads/ (PGW_SIM_COUNTER).  states: [tip_count][sites] int8
 * in host memory, or in device memory on `device` when states_on_device != 0
 * (e.g. straight into pg_compress_codes_gpu).  device_ms (may be NULL): the
 * simulation kernel's time. */
int pg_simulate_states_gpu(int tip_count, const int32_t* parent, const int32_t* post_order, int state_count,
                           const double* q, const double* pi, int reversible, int category_count,
                           const double* cat_rates, const double* cat_probs, const double* branch_lengths,
                           int64_t sites, uint64_t seed, double gap_fraction, int device, int8_t* states,
                           int states_on_device, float* device_ms);

/* substitution.hpp:55-68 discrete_gamma_categories (bin medians, mean one). */
int pg_discrete_gamma(double alpha, int count, double* rates, double* probs);

#ifdef __cplusplus
}
#endif
#endif /* PHYLOGRAD_B200_H */
