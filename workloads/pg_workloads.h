/*
 * Seeded synthetic workloads for the BASELINE.json configs —
 * input generation only, shared by both bench arms and the tests.
 *
 * This library is deliberately separate from the product library
 * (libphylograd_b200.so): the CPU reference arm of bench.py builds its inputs
 * here and never maps the product code.  It is plain host C++ (no CUDA).
 *
 * Two forward simulators (alignment.hpp:243-286 semantics: per site a rate
 * category, then the root state from pi and every other node from the row of
 * P(b c_l) selected by its parent's state, in pre-order):
 *  - PGW_SIM_REFERENCE: the reference's exact draw order — one
 *    std::mt19937_64(seed) stream and std::uniform_real_distribution<double>
 *    (0,1), category first, then nodes in tree.pre_order, with the linear
 *    cumulative scan of alignment.hpp:258-266.  Sequential; used for the
 *    small configs (C1, C2) so the reference's own simulate_states
 *    regenerates them.
 *  - PGW_SIM_COUNTER: a counter-based per-site stream (draw k of site s =
 *    splitmix64 at counter s D + k of the seed; pg_simulate.hpp), the CPU
 *    twin of the product's GPU simulator pg_simulate_states_gpu (bit-identical
 *    columns).  Used for the 10^5..10^6-column configs (C3-C5).
 *  - PGW_SIM_BLOCKED: independent mt19937_64 streams per block of 4096 sites
 *    (round-1 workloads; kept for reproducing them).
 */
#ifndef PG_WORKLOADS_H
#define PG_WORKLOADS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* PGW_SIM_NONE: tree, model and lengths only (no columns; e.g. to simulate
 * them on the GPU with pg_simulate_states_gpu from the same seed). */
enum pgw_sim { PGW_SIM_BLOCKED = 0, PGW_SIM_REFERENCE = 1, PGW_SIM_COUNTER = 2, PGW_SIM_NONE = 3 };

typedef struct pgw_spec {
  int tips;
  int model_kind;        /* 0 HKY85, 1 GTR, 2 general non-reversible 4-state, 3 AA-20 reversible, 4 GY94 codon */
  int categories;        /* 1 or discrete-gamma count */
  double gamma_alpha;
  int64_t sites;
  double branch_mean;    /* Exp(mean) branch lengths (non-clock configs) */
  int clock;             /* 1: b_i = r_i dt_i with dt ~ Exp(dt_mean), r = rate_scale*exp(N(0, rate_sd^2)) */
  double dt_mean, rate_scale, rate_sd;
  double gap_fraction;   /* Bernoulli per (taxon, site) -> missing */
  uint64_t seed;
  int threads;           /* 0 = hardware concurrency */
  int sim;               /* enum pgw_sim */
} pgw_spec;

const char* pgw_last_error(void);

/* Builds tree, model, simulation and first-occurrence compression. */
int pgw_create(const pgw_spec* spec, void** handle, int* pattern_count, int* state_count);
/* parent[2N], children[2N*2], post_order[2N-1], branch_lengths[2N-2],
 * durations[2N-2] (zeros unless clock), rates[2N-2] (zeros unless clock). */
int pgw_tree(void* handle, int32_t* parent, int32_t* children, int32_t* post_order, double* branch_lengths,
             double* durations, double* rates);
int pgw_model(void* handle, double* q, double* pi, int* reversible, double* cat_rates, double* cat_probs);
/* codes [tips][P] int8 (-1 missing), weights[P]. */
int pgw_patterns(void* handle, int8_t* codes, int64_t* weights);
void pgw_free(void* handle);

/* alignment.hpp:243-286 simulate_states in the reference's draw order (one
 * mt19937_64(seed) stream): tip states [tip_count][sites] (int8).  The tree
 * is given by parent[2N] and post_order[2N-1] (pre-order = its reverse,
 * tree.hpp:76); q row-major m x m; reversible != 0 with pi > 0 uses the
 * symmetric eigensystem, otherwise Pade scaling-and-squaring (substitution.hpp
 * :147-160); branch_lengths[2N-2] (index node-1). */
int pgw_simulate_states(int tip_count, const int32_t* parent, const int32_t* post_order, int state_count,
                        const double* q, const double* pi, int reversible, int category_count,
                        const double* cat_rates, const double* cat_probs, const double* branch_lengths,
                        int64_t sites, uint64_t seed, int8_t* states);

/* The counter-based simulation (PGW_SIM_COUNTER) of raw columns, host side:
 * the same arguments and result as pg_simulate_states_gpu (tip states
 * [tip_count][sites] int8, -1 gap); threads 0 = all cores. */
int pgw_simulate_states_counter(int tip_count, const int32_t* parent, const int32_t* post_order, int state_count,
                                const double* q, const double* pi, int reversible, int category_count,
                                const double* cat_rates, const double* cat_probs, const double* branch_lengths,
                                int64_t sites, uint64_t seed, double gap_fraction, int threads, int8_t* states);

#ifdef __cplusplus
}
#endif
#endif /* PG_WORKLOADS_H */
