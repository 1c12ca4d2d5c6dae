/*
 * pga.h — C ABI of the B200-native Giada–Marsili parallel genetic algorithm
 * (Hendricks, Gebbie & Wilcox, arXiv:1403.4099).
 *
 * Citation keys: P:n = PAPER.md line n; S:n = SPEC.md line n; Q<k> = the
 * reading listed in DESIGN.md §3.  Every entry point below cites the passage
 * that defines the operation it computes.
 *
 * Conventions (all entry points):
 *  - Return 0 (PGA_OK) or a negative PGA_E* code.  Nothing throws, nothing
 *    calls exit().  pga_last_error() gives a thread-local message.
 *  - Pointers are HOST pointers unless the name ends in _device / the
 *    argument is documented as device memory.  Caller buffers are borrowed
 *    only for the duration of the call; outputs are caller-allocated.
 *  - Labels at this boundary are int32 cluster indices 1..N (Eq. 9, P:194-198,
 *    K = N) unless documented as 0-based uint16 device labels.
 *  - A pga_ctx is bound to one CUDA device (one island of the island model)
 *    and must be used by one host thread at a time.  Any CUDA failure returns
 *    PGA_EDEVICE; the ctx must then be destroyed.
 *  - There is no CPU fallback: without a CUDA device every call that needs
 *    one returns PGA_EDEVICE.  Argument validation happens first, so invalid
 *    arguments return PGA_EINVAL even without a device.
 */
#ifndef PGA_H
#define PGA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PGA_OK = 0,
    PGA_EINVAL = -1,    /* invalid argument (message says which) */
    PGA_ENOMEM = -2,    /* device or pinned allocation failed */
    PGA_EDEVICE = -3,   /* CUDA error or no device */
    PGA_ENUMERIC = -4,  /* zero-variance / non-finite column in pga_correlation */
    PGA_ESTATE = -5     /* call not valid in the ctx's current state */
};

enum { PGA_SEL_SUS = 0, PGA_SEL_TOURNAMENT = 1 };   /* P:128; Q10 */
enum { PGA_SCALE_RANK = 0, PGA_SCALE_NONE = 1 };    /* Alg. 1; Q9 */
enum { PGA_REASON_MAX_GENS = 0, PGA_REASON_STALLED = 1 };

typedef struct pga_ctx pga_ctx;

/* GA parameters.  Defaults (pga_params_default) are Table 3. */
typedef struct {
    int32_t  pop_size;      /* individuals on THIS island (this GPU); >= 2, default 1000 */
    int32_t  elite;         /* elites copied unchanged, 0 <= elite < pop_size, default 10 */
    double   p_crossover;   /* per pair (Q11), default 0.9 */
    double   p_mutation;    /* per gene, random replacement (Q13), default 0.1 */
    double   p_kb;          /* share of crossovers that are knowledge-based (Q11/Q12), default 0.9 */
    double   tol;           /* stall tolerance on best L (Q16), default 1e-5; < 0 disables */
    int32_t  stall_gens;    /* default 50 */
    int32_t  max_gens;      /* default 400 */
    int32_t  selection;     /* PGA_SEL_SUS (default) or PGA_SEL_TOURNAMENT */
    int32_t  tournament_k;  /* 1..4, default 2 */
    int32_t  scaling;       /* PGA_SCALE_RANK (default) or PGA_SCALE_NONE.  RANK
                             * (w = 1/sqrt(rank)) is this library's reading Q9 of
                             * Alg. 1's separate "Apply scaling" step; it
                             * deliberately differs from SPEC S:151's identity
                             * scaling, which PGA_SCALE_NONE selects. */
    int32_t  device;        /* CUDA device ordinal, default 0 */
    int32_t  island;        /* this island's id, 0 <= island < n_islands */
    int32_t  n_islands;     /* islands in the run (1 = single population) */
    int32_t  migrate_every; /* migration period M in generations (Q21), default 10 */
    int32_t  migrants;      /* E_m migrants per island per migration, default 10 */
    uint64_t seed;          /* Philox key (Q18) */
} pga_params;

/* Fill *out with the Table 3 defaults.  Host only; no device needed. */
int pga_params_default(pga_params *out);

/* Create a context on p->device: copies the N x N correlation matrix C
 * (row-major fp64, host) to the device and allocates the population.
 * C must be exactly symmetric, |C_ii - 1| <= 1e-12, |C_ij| <= 1 + 1e-9,
 * finite (Eq. 7; reading Q4); otherwise PGA_EINVAL.  2 <= N <= 16384.
 * The ctx owns its copy of C; the caller's buffer may be freed on return.
 * Device buffers come from a per-device memory pool of the library that keeps
 * up to PGA_POOL_KEEP_MB (environment, default 4096) MiB of memory freed by
 * pga_destroy mapped for later contexts in the process. */
int pga_create(const double *C, int32_t N, const pga_params *p, pga_ctx **out);

/* The ctx's sizes (host only, no device call): N, pop_size (this island's
 * population) and the evaluation capacity (pop_size rounded up to 32, the
 * largest P pga_evaluate_device accepts).  Any output pointer may be NULL.
 * Bindings use it to check caller arrays before passing them. */
int pga_get_dims(pga_ctx *ctx, int32_t *N, int64_t *pop_size, int64_t *capacity);

/* Free everything owned by ctx.  NULL-safe. */
void pga_destroy(pga_ctx *ctx);

/* Thread-local message describing the last failure on this thread. */
const char *pga_last_error(void);

/* ---------------------------------------------------------------------
 * Fitness: Eq. 5 (n_s), Eq. 6 (c_s), Eq. 8 (L_c), with readings
 * Q1 (natural log), Q2 (c_s <= n_s contributes 0), Q3 (c_s clamped to
 * n_s^2 - 1e-9).
 * ------------------------------------------------------------------- */

/* labels: host int32 [P][N] row-major, values 1..N (any labelling, not
 * necessarily canonical).  out_L: host fp64 [P].  Any P >= 1 (processed in
 * chunks of the ctx's population capacity).  Values outside 1..N -> PGA_EINVAL. */
int pga_evaluate(pga_ctx *ctx, const int32_t *labels, int64_t P, double *out_L);

/* Device fast path, stream-ordered on `stream` (cudaStream_t, NULL = the
 * ctx's stream; cudaStreamLegacy selects the legacy default stream).  The call uses the ctx's evaluation scratch (staging
 * layouts, fold scratch, block flags and counters), so when `stream` is not
 * the ctx's stream it is joined to it with events in both directions: the
 * launch waits for all work already queued on the ctx's stream, and later
 * ctx work waits for the launch.  Concurrent calls on one ctx are therefore
 * serialised on the device, never interleaved (no wrong-result race).
 * labels_dev: device uint16 [P][N] row-major, 0-based values < N;  L_dev: device fp64 [P];  top_dev: device uint16 [P] or
 * NULL — label of the cluster with the largest Eq. 8 summand, 0xFFFF if none.
 * 1 <= P <= the ctx's capacity (pop_size rounded up to 32).  A label >= N is
 * evaluated as label 0 (that chromosome's L is then meaningless; the others
 * are unaffected). */
int pga_evaluate_device(pga_ctx *ctx, const uint16_t *labels_dev, int64_t P,
                        double *L_dev, uint16_t *top_dev, void *stream);

/* ---------------------------------------------------------------------
 * Genetic algorithm (Alg. 1; operators §3.1; DESIGN.md
 * §3 "GA step" fixes every unspecified detail).  The population stays
 * resident on the device; each call below is stream-ordered and the whole
 * generation runs in this library's kernels.
 * ------------------------------------------------------------------- */

/* Create the initial population from `seed` (Alg. 1 "Create initial
 * population"; Q8) and reset generation, stall and best state. */
int pga_init(pga_ctx *ctx, uint64_t seed);

/* Phase A of one generation: evaluate fitness of all individuals, then
 * (unless this is a migration generation of a multi-island run) update the
 * state and statistics and the termination test (Alg. 1).
 * *is_migration (may be NULL) is set to 1 when the caller must exchange
 * migrants (pga_export_migrants / all-gather / pga_import_migrants) before
 * phase B.  Asynchronous: does not wait for the device. */
int pga_gen_evaluate(pga_ctx *ctx, int32_t *is_migration);

/* Phase B: isolate fittest, elitism, scaling, selection, crossover,
 * mutation, replacement (Alg. 1), then advance the generation.
 * A no-op on the device once the termination flag is set. */
int pga_gen_breed(pga_ctx *ctx);

/* One full generation on a single island (phase A + phase B).  *done is set
 * to 1 if the termination criteria are met (this synchronises the stream).
 * PGA_ESTATE if no population exists or n_islands > 1. */
int pga_generation(pga_ctx *ctx, int32_t *done);

/* Whole GA run on a single island: pga_init(seed), then generations until
 * termination or `gens` generations (gens <= 0: max_gens).  Outputs (host):
 * best_labels [N] canonical 1-based, best_L, gens_run, reason
 * (PGA_REASON_*).  Any output pointer may be NULL. */
int pga_run(pga_ctx *ctx, int32_t gens, uint64_t seed, int32_t *best_labels,
            double *best_L, int32_t *gens_run, int32_t *reason);

/* Poll the device state (synchronises the stream).  Any pointer may be NULL.
 * best_labels: host int32 [N], 1-based canonical labels of the best
 * individual seen so far. */
int pga_get_state(pga_ctx *ctx, int32_t *generation, int32_t *done, int32_t *reason,
                  double *best_L, double *mean_L, int32_t *best_labels);

/* Per-generation best L, host fp64 [n] for generations 0..n-1 (n <= gens run). */
int pga_get_history(pga_ctx *ctx, double *best_L, int32_t n);

/* Copy the current population out (host int32 [pop_size][N], 1-based).  If
 * not NULL, L (host fp64 [pop_size]) and top (host int32 [pop_size], 0-based
 * label of the cluster with the largest Eq. 8 summand, -1 if none) receive
 * the results of the LAST EVALUATION, i.e. of the parents of the current
 * population once a generation has bred. */
int pga_get_population(pga_ctx *ctx, int32_t *labels, double *L, int32_t *top);

/* Replace the population (host int32 [pop_size][N], values 1..N; stored
 * canonicalised) and set the generation counter (resume, S:N/A). */
int pga_set_population(pga_ctx *ctx, const int32_t *labels, int32_t generation);

/* ---------------------------------------------------------------------
 * Island migration (P:147 ZLL2012; reading Q21).  A record
 * is {fp64 L, uint16 top, uint16 labels[N]} padded to pga_migrant_bytes().
 * ------------------------------------------------------------------- */

/* Bytes of one island's send buffer (migrants records). */
int pga_migrant_bytes(pga_ctx *ctx, int64_t *bytes);

/* After pga_gen_evaluate reported a migration generation: write this
 * island's top-`migrants` records (L desc, index asc) to dev_send (device,
 * pga_migrant_bytes()).  Stream-ordered. */
int pga_export_migrants(pga_ctx *ctx, void *dev_send);

/* dev_recv: device buffer holding n_islands send buffers back to back in
 * island order (an all-gather).  The global top-`migrants` under (L desc,
 * island asc, rank asc) replace this island's worst (L asc, index desc); then
 * the statistics / termination step of phase A runs.  Stream-ordered. */
int pga_import_migrants(pga_ctx *ctx, const void *dev_recv, int32_t n_islands);

/* The ctx's cudaStream_t (for ordering collectives with the library). */
int pga_get_stream(pga_ctx *ctx, void **stream);

/* ---------------------------------------------------------------------
 * Eq. 7, Pearson correlation with per-column centring (Q5):
 * returns: host fp64 [T][N] row-major (T observations of N assets).
 * C_out: host fp64 [N][N]; exactly symmetric, unit diagonal.  Zero-variance
 * or non-finite column -> PGA_ENUMERIC.  T >= 2, N >= 1.  Uses `device`.
 * ------------------------------------------------------------------- */
int pga_correlation(const double *returns, int32_t T, int32_t N, double *C_out, int32_t device);

/* Device variant, stream-ordered: X_dev [T][N], C_dev [N][N] (device fp64).
 * Zero variance is reported through *status_dev (device int32, set to
 * nonzero) instead of a return code. */
int pga_correlation_device(const double *X_dev, int32_t T, int32_t N, double *C_dev,
                           int32_t *status_dev, void *stream);

/* ---------------------------------------------------------------------
 * Operator test hooks: run ONE operator of DESIGN.md §3's GA step on
 * explicit host inputs, so the CUDA kernels can be compared bit-for-bit with
 * the oracle given identical inputs.  All arrays are host memory; labels
 * here are 0-based int32; `gen`/`island` select the Philox stream.
 * ------------------------------------------------------------------- */

/* Isolate fittest + scaling + selection: order_out [P] (indices
 * by L desc, index asc) and sel_out [M] parents, M = 2*ceil((P-elite)/2). */
int pga_op_select(const double *L, int64_t P, const pga_params *p, int32_t gen,
                  int32_t island, int32_t *order_out, int32_t *sel_out);

/* Mate pairing (Q10): sigma_out [M], a keyed Feistel permutation of the slots. */
int pga_op_mates(int64_t M, const pga_params *p, int32_t gen, int32_t island,
                 int32_t *sigma_out);

/* Elitism + crossover + mutation + canonicalisation + replacement
 * (P:130-136): pop [P][N] canonical 0-based parents, top [P] (-1 = none),
 * order [P], sel [M], sigma [M]; next_out [P][N] 0-based canonical.
 * p_off = global index of slot 0 (island offset). */
int pga_op_breed(const int32_t *pop, const int32_t *top, const int32_t *order,
                 int64_t P, int32_t N, const int32_t *sel, const int32_t *sigma,
                 const pga_params *p, int32_t gen, int32_t island, int64_t p_off,
                 int32_t *next_out);

/* The label-sparse pass's table-driven natural log (fitness.cu fast_ln) of
 * x[0..n) (host, positive normal values) -> out[n] (host), with the ctx's
 * table; pins its accuracy against libm in the tests. */
int pga_op_fast_ln(pga_ctx *ctx, const double *x, int64_t n, double *out);

/* First-occurrence canonical form (Q7), in place, labels [P][N] 0-based < 2N. */
int pga_op_canonicalize(int32_t *labels, int64_t P, int32_t N, int32_t device);

/* Initial population (Q8): out [P][N] 0-based canonical. */
int pga_op_init(uint64_t seed, int32_t N, int64_t P, int64_t p_off, int32_t island,
                int32_t device, int32_t *out);

/* Label-sparse fitness.  Before the dense sweep, each
 * block of 32 chromosomes is checked: if every chromosome in it needs at
 * most theta * N(N-1)/2 pair updates (sum over clusters of n_s(n_s-1)/2),
 * the block is evaluated from its clusters directly (counting sort by
 * label, L2 gathers of C for the pairs inside each cluster) and skipped by
 * the dense sweep.  The result is the same Eq. 5/6/8 value (within the
 * parity tolerance; deterministic).  theta in [0, 1]; 0 = always dense,
 * 1 = sparse whenever N <= 2048; negative = automatic, the default: 0 for
 * N < 64, else 0.25 with the cluster cache on (pga_set_cluster_cache) and
 * 0.04 with it off.  The
 * pass is cheaper than the dense sweep up to about 4% of the pairs when
 * every pair is gathered, and up to a quarter when most clusters are cache
 * hits, as in GA generations.  During a GA run the check
 * stops once a generation had no sparse block (the population only gets
 * denser); pga_init / pga_set_population re-arm it.  Host only. */
int pga_set_sparse_threshold(pga_ctx *ctx, double theta);

/* Cluster cache of the label-sparse pass (on by default; N <= 2048).  c_s
 * (Eq. 6) depends only on the member set of cluster s, and a GA generation
 * repeats almost every cluster of the one before (elites are copied,
 * knowledge-based crossover transplants whole clusters, mutation moves a
 * few genes).  Clusters with at least 4 members are keyed by two 64-bit
 * Zobrist sums of their members plus n_s, and their exact 64-bit
 * fixed-point c_s is kept in a device hash table (64 slots per chromosome,
 * PGA_CC_PER overrides; 2^12..2^22 slots of 32 B; cleared by the pass itself when half full).  A
 * hit replaces the cluster's n_s(n_s-1)/2 gathers.  Results are
 * bit-identical with the cache on or off (a wrong hit needs a 128-bit key
 * collision).  on: 0 = off, else on.  Host only. */
int pga_set_cluster_cache(pga_ctx *ctx, int32_t on);

/* Cluster-cache occupancy (measurement and tests; synchronises): slots
 * filled since the last clear, table size in slots (0 when the ctx has no
 * cache, N > 2048), and how many times the table was cleared (a launch
 * clears it when more than half the slots are filled).  Any pointer may be
 * NULL. */
int pga_cache_stats(pga_ctx *ctx, int64_t *fill, int64_t *slots, int64_t *clears);

/* ---------------------------------------------------------------------
 * Replicated master-slave across GPUs.  The paper's
 * own parallel model (§3.2): ONE population, fitness evaluated
 * by the slaves, operators on the master.  Here every GPU holds a replica
 * of the population and runs the same deterministic operators, and the
 * fitness evaluation is sharded over the GPUs.  Every rank creates its ctx
 * with the same C and params (n_islands = 1) and calls pga_init with the
 * same seed.  Per generation:
 *   pga_rep_evaluate(this rank's shard) -> all-gather L and top over the
 *   ranks (the caller, e.g. NCCL) -> pga_rep_commit(full vectors) ->
 *   pga_gen_breed.
 * The replicas stay bit-identical and the run equals pga_run on one GPU:
 * a chromosome's fitness does not depend on which launch evaluated it.
 * ------------------------------------------------------------------- */

/* Fitness (Eq. 5/6/8) of chromosomes [begin, end) of the current
 * population.  begin must be a multiple of 32 and end <= pop_size.  L_dev
 * (fp64 [end - begin]) and top_dev (uint16 [end - begin]: 0-based label of
 * the largest Eq. 8 summand, 0xFFFF = none) are device buffers.
 * Stream-ordered on the ctx's stream (pga_get_stream). */
int pga_rep_evaluate(pga_ctx *ctx, int64_t begin, int64_t end, double *L_dev, uint16_t *top_dev);

/* Install the gathered fitness of the whole population (device fp64
 * [pop_size] and uint16 [pop_size], in chromosome order) and run the
 * statistics / termination step of Alg. 1 (Q16, Q17) -- the part
 * of pga_gen_evaluate after the fitness kernel.  Stream-ordered. */
int pga_rep_commit(pga_ctx *ctx, const double *L_dev, const uint16_t *top_dev);

/* ---------------------------------------------------------------------
 * Batched GA: many small, independent clustering
 * problems in ONE kernel launch.  This is the paper's own test workload
 * (1760 correlation matrices of 18 JSE stocks, each clustered by its
 * own PGA run with the Table 3 configuration; timed per matrix in Table 4,
 * P:356-375).  One CTA per matrix keeps C, both populations, L, and the
 * selection state in shared memory for the whole run.
 *
 * Matrix b runs exactly the single-population GA of pga_run (Alg. 1
 * P:208-234 with DESIGN.md §3's operators, one island, island id 0, global
 * index offset 0) under the seed params->seed + b.  The oracle equivalent is
 * orc_run(C_b, seed + b, n_islands = 1).
 *
 * C            fp64 [B][N][N], each exactly symmetric with unit diagonal
 *              (checked for host input; device input is trusted).
 * B            number of matrices, 1 <= B <= 2^20.
 * N            2 <= N <= 32 (one gene per lane).
 * params       pop_size 2..2048; the shared-memory footprint
 *              (pga_batch_smem_bytes) must fit one CTA; n_islands must be 1;
 *              device selects the GPU.
 * on_device    0: every array is host memory and the call is synchronous.
 *              1: every array is device memory on params->device and the call
 *              is stream-ordered on `stream` (NULL = legacy default stream).
 * best_labels  int32 [B][N], 1-based canonical best labelling per matrix.
 * best_L       fp64 [B], its Eq. 8 likelihood.
 * gens         int32 [B], generations evaluated.
 * reason       int32 [B], PGA_REASON_*.
 * history      fp64 [B][max_gens] per-generation best L, or NULL.  Entries
 *              past gens[b] are 0 (host) / untouched (device).
 * Any of best_labels .. history may be NULL except best_L.
 * ------------------------------------------------------------------- */
int pga_batch_run(const double *C, int32_t B, int32_t N, const pga_params *params,
                  int32_t on_device, int32_t *best_labels, double *best_L, int32_t *gens,
                  int32_t *reason, double *history, void *stream);

/* Shared memory one CTA of pga_batch_run needs for (N, pop_size, elite);
 * PGA_EINVAL if it exceeds the device's per-block opt-in limit. */
int pga_batch_smem_bytes(int32_t N, int32_t pop_size, int32_t elite, int32_t device,
                         int64_t *bytes);

/* Test hooks of the batched kernel (host memory, 0-based labels):
 * pga_batch_op_evaluate: Eq. 8 for labels [B][P][N] (values 0..2N) against
 *   C [B][N][N] -> L [B][P], top [B][P] (-1 = none), as pga_evaluate.
 * pga_batch_op_step: one generation's operators (order, scaling, selection,
 *   mates, crossover, mutation, canonicalisation, elitism) of every matrix,
 *   given its canonical population pop [B][P][N], L [B][P] and top [B][P],
 *   at generation `gen` -> next [B][P][N]; matrix b uses seed + b. */
int pga_batch_op_evaluate(const double *C, int32_t B, int32_t N, const int32_t *labels,
                          int32_t P, int32_t device, double *L, int32_t *top);
int pga_batch_op_step(int32_t B, int32_t N, const pga_params *params, const int32_t *pop,
                      const double *L, const int32_t *top, int32_t gen, int32_t *next);

/* ---------------------------------------------------------------------
 * Correlation stream: the paper's pre-processing
 * (§4.2.5; operations as SPEC S:279-301, readings Q31-Q33) on the
 * device, producing the windows the batched GA clusters ("fast online
 * intraday correlation matrix estimation").
 *   EWMA:   d = x_t - m; cov <- lambda cov + (1-lambda) d d^T;
 *           m <- lambda m + (1-lambda) x_t; zero initial state.
 *   After observation t = warm-1 + b*stride (b = 0 .. B-1) the state is
 *   emitted as a correlation matrix C_ij = cov_ij / sqrt(cov_ii cov_jj)
 *   and, if q >= 0, cleaned: eigenvalues inside the Marchenko-Pastur band
 *   [(1-sqrt q)^2, (1+sqrt q)^2] are replaced by their mean (trace
 *   preserving), C' = V diag(w') V^T, renormalised to a unit diagonal
 *   from its upper triangle (exactly symmetric).  q == 0 selects the
 *   SPEC's q = N (1 - lambda) (effective sample 1/(1-lambda)); q < 0
 *   disables cleaning.
 * X       fp64 [T][N] returns, row-major.   1 <= N <= 64, 0 < lambda < 1,
 *         warm >= 1, stride >= 1, T >= warm.
 * C_out   fp64 [B][N][N], B = pga_stream_count(T, warm, stride).
 * on_device 0: X, C_out host, synchronous; a non-positive variance at an
 *         emission -> PGA_ENUMERIC (and *status = 1 if status != NULL).
 *         1: X, C_out, status device memory on `device`; the call is
 *         ASYNCHRONOUS and stream-ordered: it enqueues the kernels and the
 *         stream-ordered release of its scratch (cudaFreeAsync) on `stream`
 *         and returns; C_out and *status (caller-zeroed, set to 1 on a
 *         non-positive variance) are valid only once `stream` has reached
 *         that point (synchronise it, or order later work on it).
 * The EWMA recurrences and the uncleaned correlation are computed without
 * FMA contraction in the SPEC's operation order (bit-identical to a plain
 * fp64 evaluation); the cleaning uses a two-sided Jacobi eigensolver.
 * ------------------------------------------------------------------- */
int pga_stream_count(int32_t T, int32_t warm, int32_t stride);
int pga_corr_stream(const double *X, int32_t T, int32_t N, double lambda, int32_t warm,
                    int32_t stride, double q, int32_t on_device, double *C_out, int32_t *status,
                    int32_t device, void *stream);

/* Number of this library's kernel launches issued so far in this process
 * (for the bench's gpu_launches claim). */
int64_t pga_launch_count(void);

/* Device-side invariant checks (test infrastructure; the substitute for
 * compute-sanitizer, which the GPU pool does not allow): in a library built
 * with -DPGA_DEVICE_CHECKS, the number of index/range invariants of the hot
 * kernels found violated so far in this process (0 = clean; synchronises
 * with the device).  -1 in the product build (checks compiled out); -2 on a
 * CUDA error. */
int64_t pga_debug_violations(void);

/* Kernel timing with CUDA events on the ctx's stream (measurement only).
 * pga_profile_enable(ctx, level): level 1 records, for every generation
 * launched through pga_gen_evaluate / pga_gen_breed, 3 events (fitness
 * kernel start/end, generation end); level 2 records every phase boundary
 * (9 events, ~3 us of overhead per generation); 0 stops and clears.
 * pga_profile_read synchronises and returns the SUMS in milliseconds of the
 * dense fitness kernel (sweep_ms: sweep + fused fold), of the label-sparse
 * pre-pass (fold_ms; pga_set_sparse_threshold) and of whole generations, and
 * the number of generations recorded.  pga_profile_sparse_blocks returns how
 * many 32-chromosome blocks the pre-pass evaluated since profiling was
 * enabled (the dense kernel skipped those). */
int pga_profile_enable(pga_ctx *ctx, int32_t on);
int pga_profile_read(pga_ctx *ctx, double *sweep_ms, double *fold_ms, double *gen_ms,
                     int32_t *count);
int pga_profile_sparse_blocks(pga_ctx *ctx, int64_t *sparse_blocks);
/* Same, plus the off-diagonal C entries the pre-pass gathered (sum over its
 * chromosomes' clusters of n_s(n_s-1)/2); gathered may be NULL. */
int pga_profile_sparse(pga_ctx *ctx, int64_t *sparse_blocks, int64_t *gathered);
/* Cluster-cache hits since profiling was enabled, and the off-diagonal pair
 * updates they replaced (pga_set_cluster_cache).  Synchronises. */
int pga_profile_cache(pga_ctx *ctx, int64_t *hits, int64_t *saved);

/* Level-2 profiling: per-phase AVERAGE milliseconds, ms[PGA_PROF_PHASES]:
 * 0 dense fitness kernel (sweep + fused fold), 1 label-sparse pre-pass, 2 statistics/termination
 * (in non-migration generations also the order sort and the selection, which run beside the
 * statistics since round 2), 3 order sort, 4 scaling+selection, 5 mate pairing (~0 then: only
 * the phase marks), 6 breed, 7 advance (fused into the breed's last CTA since round 2: ~0). */
#define PGA_PROF_PHASES 8
int pga_profile_phases(pga_ctx *ctx, double *ms, int32_t *count);

#ifdef __cplusplus
}
#endif

#endif /* PGA_H */
