/*
 * oracle.c — the CPU ORACLE for the Giada–Marsili PGA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1403_4099_b200/, libpga.so) never links, imports
 * or calls it, and shares no code, header, table or constant generator with
 * it.  Plain, slow, obviously-correct C: fp64, sequential loops, no blocking,
 * no fusion, no SIMD intrinsics.
 *
 * Citation keys: P:n = PAPER.md line n (arXiv:1403.4099, Hendricks, Gebbie &
 * Wilcox); S:n = SPEC.md line n; Q<k> = reading k listed in DESIGN.md §3
 * (taken from SURVEY.md §8(c)).
 *
 * Parity status per function:
 *   orc_philox4x32_10     pinned (Random123 known-answer vectors)
 *   orc_cluster_stats     pinned (numpy one-hot diag(Z^T C Z); closed forms)
 *   orc_log_likelihood    pinned (closed forms: pair, triple, planted block;
 *                         singleton/identity zeros; brute-force argmax)
 *                         -- GPU parity unpinned near the c_s -> n_s^2 clamp
 *                            (Q3); the clamp itself is pinned by properties
 *                            (tests/test_oracle_fitness.py)
 *   orc_canonicalize      pinned (idempotence, first-occurrence invariants)
 *   orc_brute_force       pinned (Bell numbers 1..10)
 *   orc_select / mates    pinned (SUS worked examples S:153-155, expected-copies
 *                         identity, tournament brute force)
 *   orc_breed             pinned (identity cases S:163-164, binomial mean)
 *                         -- knowledge-based crossover is a reconstruction
 *                            (Q12): parity vs the paper UNPINNED
 *   orc_pearson           pinned (numpy corrcoef)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_TAG_INIT 1u
#define ORC_TAG_SUS  2u
#define ORC_TAG_PERM 3u
#define ORC_TAG_TOUR 4u
#define ORC_TAG_XO   5u
#define ORC_TAG_MUT  6u
#define ORC_TAG_MUTV 7u

/* ------------------------------------------------------------------------
 * Philox4x32-10 (Salmon, Moraes, Dror & Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3").  The paper does not name an RNG (Q18); DESIGN.md §3
 * fixes this counter-based generator so the GPU and the oracle draw the same
 * stream.  Written out round by round.
 * ---------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    int round;
    for (round = 0; round < 10; round++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (round < 9) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The counter layout of DESIGN.md §3 (RNG): key = (seed_lo, seed_hi),
 * counter = (c0, c1, generation, tag | island << 8). */
static void draw(uint64_t seed, uint32_t tag, uint32_t island, uint32_t gen,
                 uint32_t c0, uint32_t c1, uint32_t out[4])
{
    uint32_t ctr[4], key[2];
    ctr[0] = c0;
    ctr[1] = c1;
    ctr[2] = gen;
    ctr[3] = tag | (island << 8);
    key[0] = (uint32_t)(seed & 0xFFFFFFFFu);
    key[1] = (uint32_t)(seed >> 32);
    orc_philox4x32_10(ctr, key, out);
}

/* Integer in [0, n): floor(x * n / 2^32) (Q18). */
static uint32_t scale_u32(uint32_t x, uint32_t n)
{
    return (uint32_t)(((uint64_t)x * (uint64_t)n) >> 32);
}

/* Probability p as an integer threshold on a uniform u32: event iff x < thr. */
static uint64_t prob_threshold(double p)
{
    if (p >= 1.0) return (uint64_t)1 << 32;
    if (p <= 0.0) return 0;
    return (uint64_t)llround(p * 4294967296.0);
}

/* ------------------------------------------------------------------------
 * Eq. 5 and Eq. 6: cluster sizes and intra-cluster correlation,
 * by definition: a full N x N double loop in row-major order, diagonal
 * included.  labels are 0-based and < K.
 * ---------------------------------------------------------------------- */
void orc_cluster_stats(const double *C, int32_t N, const int32_t *s, int32_t K,
                       int64_t *n_out, double *c_out)
{
    int32_t i, j, k;
    for (k = 0; k < K; k++) { n_out[k] = 0; c_out[k] = 0.0; }
    for (i = 0; i < N; i++) n_out[s[i]] += 1;                 /* Eq. 5 */
    for (i = 0; i < N; i++)
        for (j = 0; j < N; j++)
            if (s[i] == s[j]) c_out[s[i]] += C[(int64_t)i * N + j];   /* Eq. 6 */
}

/* One cluster's summand of Eq. 8, natural log (Q1).
 * Q2: clusters with c_s <= n_s contribute 0 (constrained MLE g* in [0,1],
 *     Eq. 4; "L_c = 0 for clusters of objects that are uncorrelated",
 *     P:111).
 * Q3: c_s is clamped to n_s^2 - 1e-9 before the second log. */
double orc_cluster_term(int64_t n_s, double c_s)
{
    double n = (double)n_s;
    double n2, ch;
    if (n_s < 2) return 0.0;                 /* Eq. 8 sums over n_s > 1 only */
    if (c_s <= n) return 0.0;                /* Q2 */
    n2 = n * n;
    ch = c_s;
    if (ch > n2 - 1e-9) ch = n2 - 1e-9;      /* Q3 */
    return log(n / ch) + (n - 1.0) * log((n2 - n) / (n2 - ch));
}

static int32_t max_label(const int32_t *s, int32_t N)
{
    int32_t i, m = 0;
    for (i = 0; i < N; i++) if (s[i] > m) m = s[i];
    return m;
}

/* Eq. 8: L_c = 1/2 sum_{s: n_s > 1} f_s, summed by ascending s.
 * top_out (may be NULL) receives the label with the largest f_s > 0
 * (smallest label wins ties), or -1 if every f_s is 0 (KB
 * crossover input). */
double orc_log_likelihood(const double *C, int32_t N, const int32_t *s, int32_t *top_out)
{
    int32_t K = max_label(s, N) + 1;
    int64_t *n = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
    double *c = (double *)malloc(sizeof(double) * (size_t)K);
    double sum = 0.0, best_f = 0.0;
    int32_t k, top = -1;
    orc_cluster_stats(C, N, s, K, n, c);
    for (k = 0; k < K; k++) {
        if (n[k] >= 2) {
            double f = orc_cluster_term(n[k], c[k]);
            sum += f;
            if (f > best_f) { best_f = f; top = k; }
        }
    }
    free(n);
    free(c);
    if (top_out) *top_out = top;
    return 0.5 * sum;
}

/* Fitness of a population: labels [P][N] row-major.  nthreads > 1 splits the
 * chromosomes with a static stride (each chromosome is still evaluated by
 * the same sequential definition, so the result does not depend on it). */
typedef struct {
    const double *C; int32_t N; const int32_t *labels; int64_t P;
    double *L; int32_t *top; int t, nt;
} eval_job;

static void *eval_worker(void *arg)
{
    eval_job *j = (eval_job *)arg;
    int64_t p;
    for (p = j->t; p < j->P; p += j->nt) {
        int32_t tp;
        j->L[p] = orc_log_likelihood(j->C, j->N, j->labels + p * j->N, &tp);
        if (j->top) j->top[p] = tp;
    }
    return NULL;
}

void orc_evaluate(const double *C, int32_t N, const int32_t *labels, int64_t P,
                  double *L, int32_t *top, int32_t nthreads)
{
    int t;
    if (nthreads <= 1) {
        eval_job j = {C, N, labels, P, L, top, 0, 1};
        eval_worker(&j);
        return;
    }
    {
        pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
        eval_job *jobs = (eval_job *)malloc(sizeof(eval_job) * (size_t)nthreads);
        for (t = 0; t < nthreads; t++) {
            eval_job j = {C, N, labels, P, L, top, t, nthreads};
            jobs[t] = j;
            pthread_create(&th[t], NULL, eval_worker, &jobs[t]);
        }
        for (t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
        free(th);
        free(jobs);
    }
}

/* First-occurrence canonical form (Q7): the label of gene 0 becomes 0,
 * each new cluster takes the next unused integer.  In place, one chromosome. */
void orc_canonicalize(int32_t *s, int32_t N)
{
    int32_t K = max_label(s, N) + 1;
    int32_t *map = (int32_t *)malloc(sizeof(int32_t) * (size_t)K);
    int32_t i, next = 0;
    for (i = 0; i < K; i++) map[i] = -1;
    for (i = 0; i < N; i++) {
        if (map[s[i]] < 0) map[s[i]] = next++;
        s[i] = map[s[i]];
    }
    free(map);
}

void orc_canonicalize_batch(int32_t *labels, int64_t P, int32_t N)
{
    int64_t p;
    for (p = 0; p < P; p++) orc_canonicalize(labels + p * N, N);
}

/* ------------------------------------------------------------------------
 * Exhaustive maximisation over all set partitions: restricted
 * growth strings a[0]=0, a[i] <= 1 + max(a[0..i-1]), visited in
 * lexicographic order.  Ties keep the first (smallest) string (Q19).
 * Returns the number of partitions visited (Bell(N)) or -1 if N > 12.
 * ---------------------------------------------------------------------- */
int64_t orc_brute_force(const double *C, int32_t N, int32_t *best, double *best_L)
{
    int32_t a[16], m[16];
    int64_t count = 0;
    double bL = -1.0;
    int32_t i;
    if (N < 1 || N > 12) return -1;
    for (i = 0; i < N; i++) { a[i] = 0; m[i] = 0; }
    for (;;) {
        double L = orc_log_likelihood(C, N, a, NULL);
        count++;
        if (L > bL) {
            bL = L;
            for (i = 0; i < N; i++) best[i] = a[i];
        }
        /* next restricted growth string: m[i] = max(a[0..i-1]) */
        i = N - 1;
        while (i > 0 && a[i] == m[i] + 1) i--;
        if (i == 0) break;
        a[i] += 1;
        {
            int32_t k;
            for (k = i + 1; k < N; k++) {
                a[k] = 0;
                m[k] = (m[k - 1] > a[k - 1]) ? m[k - 1] : a[k - 1];
            }
        }
    }
    *best_L = bL;
    return count;
}

/* ------------------------------------------------------------------------
 * Genetic operators (Alg. 1; §3.1; Table 3),
 * exactly as DESIGN.md §3 (GA step) specifies.
 * ---------------------------------------------------------------------- */

/* Initial population (Alg. 1 "Create initial population"; Q8):
 * gene i of chromosome p_global: scale(Philox(INIT; i>>2, p_global)[i&3], N)
 * with generation field 0xFFFFFFFF, then canonicalised. */
void orc_init_population(uint64_t seed, int32_t N, int64_t P, int64_t p_off,
                         uint32_t island, int32_t *out)
{
    int64_t p;
    int32_t i;
    for (p = 0; p < P; p++) {
        for (i = 0; i < N; i++) {
            uint32_t x[4];
            draw(seed, ORC_TAG_INIT, island, 0xFFFFFFFFu, (uint32_t)(i >> 2),
                 (uint32_t)(p_off + p), x);
            out[p * N + i] = (int32_t)scale_u32(x[i & 3], (uint32_t)N);
        }
        orc_canonicalize(out + p * N, N);
    }
}

typedef struct { double L; int32_t idx; } lkey;

/* (L desc, idx asc) */
static int cmp_lkey(const void *a, const void *b)
{
    const lkey *x = (const lkey *)a, *y = (const lkey *)b;
    if (x->L > y->L) return -1;
    if (x->L < y->L) return 1;
    return (x->idx < y->idx) ? -1 : (x->idx > y->idx);
}

/* order[r] = index of the individual with rank r+1 under (L desc, idx asc)
 * ("Isolate fittest individuals"). */
void orc_order(const double *L, int32_t P, int32_t *order)
{
    lkey *k = (lkey *)malloc(sizeof(lkey) * (size_t)P);
    int32_t i;
    for (i = 0; i < P; i++) { k[i].L = L[i]; k[i].idx = i; }
    qsort(k, (size_t)P, sizeof(lkey), cmp_lkey);
    for (i = 0; i < P; i++) order[i] = k[i].idx;
    free(k);
}

static int32_t ceil_log2(int64_t x)
{
    int32_t b = 0;
    while (((int64_t)1 << b) < x) b++;
    return b;
}

int32_t orc_num_offspring(int32_t P, int32_t E)
{
    return 2 * ((P - E + 1) / 2);
}

/* Scaling + selection (Alg. 1 "Apply scaling", "selection").
 * scaling 0 = RANK (w = 1/sqrt(rank), Q9), 1 = NONE (w = L).
 * selection 0 = SUS (Baker's stochastic universal sampling with
 * integer-quantised segments), 1 = tournament of size tour_k (Q10).
 * order: from orc_order.  sel_out: M = orc_num_offspring(P, E) parents. */
void orc_select(const double *L, const int32_t *order, int32_t P, int32_t E,
                int32_t selection, int32_t tour_k, int32_t scaling,
                uint64_t seed, uint32_t gen, uint32_t island, int32_t *sel_out)
{
    int32_t M = orc_num_offspring(P, E);
    int32_t m, i;
    if (selection == 1) {
        for (m = 0; m < M; m++) {
            uint32_t x[4];
            int32_t best, t;
            draw(seed, ORC_TAG_TOUR, island, gen, (uint32_t)m, 0u, x);
            best = (int32_t)scale_u32(x[0], (uint32_t)P);
            for (t = 1; t < tour_k; t++) {
                int32_t c = (int32_t)scale_u32(x[t], (uint32_t)P);
                if (L[c] > L[best] || (L[c] == L[best] && c < best)) best = c;
            }
            sel_out[m] = best;
        }
        return;
    }
    {
        double *w = (double *)malloc(sizeof(double) * (size_t)P);
        int32_t *rank = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
        double wmax = 0.0;
        for (i = 0; i < P; i++) rank[order[i]] = i + 1;
        for (i = 0; i < P; i++) {
            if (scaling == 0) w[i] = 1.0 / sqrt((double)rank[i]);
            else w[i] = L[i];
            if (i == 0 || w[i] > wmax) wmax = w[i];
        }
        if (!(wmax > 0.0)) {
            /* all-zero fitness: uniform fallback */
            for (m = 0; m < M; m++) {
                uint32_t x[4];
                draw(seed, ORC_TAG_SUS, island, gen, (uint32_t)m, 0u, x);
                sel_out[m] = (int32_t)scale_u32(x[0], (uint32_t)P);
            }
        } else {
            int32_t B = 62 - ceil_log2(P);
            uint64_t *prefix = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)P);
            uint64_t Q = 0, step, start, u;
            uint32_t x[4];
            for (i = 0; i < P; i++) {
                double r = w[i] / wmax;
                uint64_t q = (r > 0.0) ? (uint64_t)floor(ldexp(r, B)) : 0;
                Q += q;
                prefix[i] = Q;                      /* inclusive prefix */
            }
            step = Q / (uint64_t)M;
            draw(seed, ORC_TAG_SUS, island, gen, 0u, 0xFFFFFFFFu, x);
            u = ((uint64_t)x[0] << 32) | (uint64_t)x[1];
            start = (uint64_t)(((unsigned __int128)u * (unsigned __int128)step) >> 64);
            i = 0;
            for (m = 0; m < M; m++) {
                uint64_t ptr = start + (uint64_t)m * step;
                while (prefix[i] <= ptr) i++;        /* min{i : prefix_i > ptr} */
                sel_out[m] = i;
            }
            free(prefix);
        }
        free(w);
        free(rank);
    }
}

/* Mate pairing (unspecified in the paper, Q10): sigma is a keyed pseudo-
 * random permutation of the M offspring slots -- a 4-round Feistel network
 * on h+h bits (2^(2h) >= M) with round function Philox(PERM; R, round)[0],
 * cycle-walked back into [0, M); pair k = (sigma[2k], sigma[2k+1]). */
static uint32_t feistel_perm(uint32_t m, uint32_t M, uint64_t seed, uint32_t gen, uint32_t island)
{
    int32_t h = (ceil_log2(M) + 1) / 2;
    uint32_t mask, x = m;
    if (h < 1) h = 1;
    mask = (1u << h) - 1u;
    do {
        uint32_t Lh = x >> h, R = x & mask;
        int r;
        for (r = 0; r < 4; r++) {
            uint32_t f[4], t;
            draw(seed, ORC_TAG_PERM, island, gen, R, (uint32_t)r, f);
            t = R;
            R = Lh ^ (f[0] & mask);
            Lh = t;
        }
        x = (Lh << h) | R;
    } while (x >= M);
    return x;
}

void orc_mates(int32_t M, uint64_t seed, uint32_t gen, uint32_t island, int32_t *sigma)
{
    int32_t m;
    for (m = 0; m < M; m++)
        sigma[m] = (int32_t)feistel_perm((uint32_t)m, (uint32_t)M, seed, gen, island);
}

/* Crossover (Table 3; Q11, Q12), mutation
 * (Table 3; Q13, Q14), canonicalisation and replacement
 * (Q15) for every pair; elites are copied unchanged.
 * pop: [P][N] canonical parents; top[p] = KB top label (-1 = none);
 * sel: M parents; sigma: mate order; next: [P][N] output. */
void orc_breed(const int32_t *pop, const int32_t *top, const int32_t *order,
               int32_t P, int32_t N, int32_t E, const int32_t *sel,
               const int32_t *sigma, double p_c, double p_m, double p_kb,
               uint64_t seed, uint32_t gen, uint32_t island, int64_t p_off,
               int32_t *next)
{
    int32_t M = orc_num_offspring(P, E);
    uint64_t thr_c = prob_threshold(p_c), thr_kb = prob_threshold(p_kb);
    uint64_t thr_m = prob_threshold(p_m);
    int32_t *A = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
    int32_t *Bc = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
    int32_t e, k, i, c;
    for (e = 0; e < E; e++)
        memcpy(next + (int64_t)e * N, pop + (int64_t)order[e] * N, sizeof(int32_t) * (size_t)N);
    for (k = 0; k < M / 2; k++) {
        int32_t a = sel[sigma[2 * k]], b = sel[sigma[2 * k + 1]];
        const int32_t *pa = pop + (int64_t)a * N, *pb = pop + (int64_t)b * N;
        uint32_t x[4];
        draw(seed, ORC_TAG_XO, island, gen, (uint32_t)k, 0u, x);
        if ((uint64_t)x[0] >= thr_c) {
            memcpy(A, pa, sizeof(int32_t) * (size_t)N);
            memcpy(Bc, pb, sizeof(int32_t) * (size_t)N);
        } else if ((uint64_t)x[1] < thr_kb) {
            /* knowledge-based: transplant the other parent's top cluster as a
             * fresh label N (SPEC S:195 reconstruction, Q12) */
            for (i = 0; i < N; i++) {
                A[i] = (top[b] >= 0 && pb[i] == top[b]) ? N : pa[i];
                Bc[i] = (top[a] >= 0 && pa[i] == top[a]) ? N : pb[i];
            }
        } else {
            int32_t cut = 1 + (int32_t)scale_u32(x[2], (uint32_t)(N - 1));
            for (i = 0; i < N; i++) {
                A[i] = (i < cut) ? pa[i] : pb[i];
                Bc[i] = (i < cut) ? pb[i] : pa[i];
            }
        }
        for (c = 0; c < 2; c++) {
            int32_t o = E + 2 * k + c;
            int32_t *child = (c == 0) ? A : Bc;
            uint32_t og = (uint32_t)(p_off + o);
            for (i = 0; i < N; i++) {
                uint32_t u[4];
                draw(seed, ORC_TAG_MUT, island, gen, (uint32_t)(i >> 2), og, u);
                if ((uint64_t)u[i & 3] < thr_m) {
                    uint32_t v[4];
                    draw(seed, ORC_TAG_MUTV, island, gen, (uint32_t)(i >> 2), og, v);
                    child[i] = (int32_t)scale_u32(v[i & 3], (uint32_t)N);
                }
            }
            orc_canonicalize(child, N);
            if (o < P) memcpy(next + (int64_t)o * N, child, sizeof(int32_t) * (size_t)N);
        }
    }
    free(A);
    free(Bc);
}

/* Parameters (Table 3 defaults).  The oracle's own struct. */
typedef struct {
    int32_t pop;          /* individuals per island */
    int32_t elite;        /* 10 */
    double p_c;           /* 0.9 */
    double p_m;           /* 0.1 per gene (Q13) */
    double p_kb;          /* 0.9 */
    double tol;           /* 1e-5; < 0 disables stall termination */
    int32_t stall_gens;   /* 50 */
    int32_t max_gens;     /* 400 */
    int32_t selection;    /* 0 SUS, 1 tournament */
    int32_t tour_k;       /* 2 */
    int32_t scaling;      /* 0 RANK, 1 NONE */
    int32_t n_islands;    /* 1 */
    int32_t migrate_every;/* 10 */
    int32_t migrants;     /* 10 */
    uint64_t seed;
} orc_params;

/* One generation's operators (elitism .. replacement) given the evaluated
 * population; next receives the new population. */
void orc_step(const orc_params *pp, int32_t N, const int32_t *pop, const double *L,
              const int32_t *top, uint32_t gen, uint32_t island, int64_t p_off,
              int32_t *next)
{
    int32_t P = pp->pop, E = pp->elite;
    int32_t M = orc_num_offspring(P, E);
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
    int32_t *sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)M);
    int32_t *sigma = (int32_t *)malloc(sizeof(int32_t) * (size_t)M);
    orc_order(L, P, order);
    orc_select(L, order, P, E, pp->selection, pp->tour_k, pp->scaling, pp->seed, gen,
               island, sel);
    orc_mates(M, pp->seed, gen, island, sigma);
    orc_breed(pop, top, order, P, N, E, sel, sigma, pp->p_c, pp->p_m, pp->p_kb,
              pp->seed, gen, island, p_off, next);
    free(order);
    free(sel);
    free(sigma);
}

/* Elite migration between islands (P:147 ZLL2012; Q21):
 * every island offers its top `migrants` (L desc, idx asc); the global top
 * `migrants` under (L desc, island asc, rank asc) replace each island's
 * worst `migrants` (L asc, idx desc).  pops/Ls/tops: arrays of G pointers. */
void orc_migrate(int32_t G, int32_t P, int32_t N, int32_t Em, int32_t **pops,
                 double **Ls, int32_t **tops)
{
    int32_t total = G * Em, g, r, j;
    int32_t *cand_isl = (int32_t *)malloc(sizeof(int32_t) * (size_t)total);
    int32_t *cand_idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)total);
    double *cand_L = (double *)malloc(sizeof(double) * (size_t)total);
    int32_t *chosen = (int32_t *)malloc(sizeof(int32_t) * (size_t)Em);
    int32_t *mig_lab = (int32_t *)malloc(sizeof(int32_t) * (size_t)Em * (size_t)N);
    double *mig_L = (double *)malloc(sizeof(double) * (size_t)Em);
    int32_t *mig_top = (int32_t *)malloc(sizeof(int32_t) * (size_t)Em);
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
    int32_t *used = (int32_t *)calloc((size_t)total, sizeof(int32_t));
    for (g = 0; g < G; g++) {
        orc_order(Ls[g], P, order);
        for (r = 0; r < Em; r++) {
            cand_isl[g * Em + r] = g;
            cand_idx[g * Em + r] = order[r];
            cand_L[g * Em + r] = Ls[g][order[r]];
        }
    }
    /* selection of the global top Em by (L desc, island asc, rank asc):
     * candidates are stored in (island, rank) order, so a strict '>' scan
     * keeps the earliest among equals. */
    for (r = 0; r < Em; r++) {
        int32_t b = -1;
        for (j = 0; j < total; j++) {
            if (used[j]) continue;
            if (b < 0 || cand_L[j] > cand_L[b]) b = j;
        }
        used[b] = 1;
        chosen[r] = b;
    }
    for (r = 0; r < Em; r++) {
        int32_t b = chosen[r];
        memcpy(mig_lab + (int64_t)r * N, pops[cand_isl[b]] + (int64_t)cand_idx[b] * N,
               sizeof(int32_t) * (size_t)N);
        mig_L[r] = cand_L[b];
        mig_top[r] = tops[cand_isl[b]][cand_idx[b]];
    }
    for (g = 0; g < G; g++) {
        orc_order(Ls[g], P, order);
        for (r = 0; r < Em; r++) {
            int32_t w = order[P - 1 - r];            /* r-th worst */
            memcpy(pops[g] + (int64_t)w * N, mig_lab + (int64_t)r * N,
                   sizeof(int32_t) * (size_t)N);
            Ls[g][w] = mig_L[r];
            tops[g][w] = mig_top[r];
        }
    }
    free(cand_isl); free(cand_idx); free(cand_L); free(chosen);
    free(mig_lab); free(mig_L); free(mig_top); free(order); free(used);
}

/* Full GA (Alg. 1) on G islands simulated in sequence.  For G == 1 the stall
 * rule is checked every generation; for G > 1 it is checked only at
 * migration generations on the global best (Q16/Q21).
 * best_labels [N], best_L, gens_run, reason (0 max_gens, 1 stalled).
 * history (may be NULL): best L of every generation (island-global). */
int32_t orc_run(const double *C, int32_t N, const orc_params *pp,
                int32_t *best_labels, double *best_L, int32_t *gens_run,
                int32_t *reason, double *history, int32_t nthreads)
{
    int32_t G = pp->n_islands, P = pp->pop, g, isl, i;
    int32_t **pop = (int32_t **)malloc(sizeof(int32_t *) * (size_t)G);
    int32_t **nxt = (int32_t **)malloc(sizeof(int32_t *) * (size_t)G);
    double **L = (double **)malloc(sizeof(double *) * (size_t)G);
    int32_t **top = (int32_t **)malloc(sizeof(int32_t *) * (size_t)G);
    double best_ever = -1.0, prev_best = 0.0;
    int32_t stall = 0, stop = 0;
    if (N < 2 || P < 2 || pp->elite < 0 || pp->elite >= P || G < 1) return -1;
    for (isl = 0; isl < G; isl++) {
        pop[isl] = (int32_t *)malloc(sizeof(int32_t) * (size_t)P * (size_t)N);
        nxt[isl] = (int32_t *)malloc(sizeof(int32_t) * (size_t)P * (size_t)N);
        L[isl] = (double *)malloc(sizeof(double) * (size_t)P);
        top[isl] = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
        orc_init_population(pp->seed, N, P, (int64_t)isl * P, (uint32_t)isl, pop[isl]);
    }
    *reason = 0;
    for (g = 0; !stop; g++) {
        double gbest = -1.0;
        int32_t gbest_isl = 0, gbest_idx = 0;
        int migrate_now = (G > 1) && ((g + 1) % pp->migrate_every == 0);
        for (isl = 0; isl < G; isl++)
            orc_evaluate(C, N, pop[isl], P, L[isl], top[isl], nthreads);
        if (migrate_now)
            orc_migrate(G, P, N, pp->migrants, pop, L, top);
        for (isl = 0; isl < G; isl++)
            for (i = 0; i < P; i++)
                if (L[isl][i] > gbest) { gbest = L[isl][i]; gbest_isl = isl; gbest_idx = i; }
        if (history) history[g] = gbest;
        if (gbest > best_ever) {
            best_ever = gbest;
            memcpy(best_labels, pop[gbest_isl] + (int64_t)gbest_idx * N, sizeof(int32_t) * (size_t)N);
        }
        if (G == 1) {
            if (g > 0) {
                if (gbest - prev_best < pp->tol) stall++;
                else stall = 0;
            }
            prev_best = gbest;
        } else if (migrate_now) {
            if (g + 1 > pp->migrate_every) {
                if (gbest - prev_best < pp->tol) stall += pp->migrate_every;
                else stall = 0;
            }
            prev_best = gbest;
        }
        if (pp->tol >= 0.0 && stall >= pp->stall_gens) { stop = 1; *reason = 1; }
        if (g + 1 >= pp->max_gens) stop = 1;
        if (stop) { *gens_run = g + 1; break; }
        for (isl = 0; isl < G; isl++) {
            int32_t *t;
            orc_step(pp, N, pop[isl], L[isl], top[isl], (uint32_t)g, (uint32_t)isl,
                     (int64_t)isl * P, nxt[isl]);
            t = pop[isl]; pop[isl] = nxt[isl]; nxt[isl] = t;
        }
    }
    *best_L = best_ever;
    for (isl = 0; isl < G; isl++) { free(pop[isl]); free(nxt[isl]); free(L[isl]); free(top[isl]); }
    free(pop); free(nxt); free(L); free(top);
    return 0;
}

/* ------------------------------------------------------------------------
 * Eq. 7, Pearson correlation with per-column centring (Q5):
 * X is [T][N] row-major (T observations of N assets).  Two passes: mean,
 * then centred inner products; C_ii := 1, lower triangle mirrored from the
 * upper.  Returns -1 if a column has zero variance or X is not finite.
 * ---------------------------------------------------------------------- */
int32_t orc_pearson(const double *X, int32_t T, int32_t N, double *C)
{
    double *mean = (double *)calloc((size_t)N, sizeof(double));
    double *norm = (double *)calloc((size_t)N, sizeof(double));
    int32_t i, j, t, rc = 0;
    for (t = 0; t < T; t++)
        for (i = 0; i < N; i++) {
            double v = X[(int64_t)t * N + i];
            if (!isfinite(v)) rc = -1;
            mean[i] += v;
        }
    for (i = 0; i < N; i++) mean[i] /= (double)T;
    for (i = 0; i < N; i++) {
        double s = 0.0;
        for (t = 0; t < T; t++) {
            double d = X[(int64_t)t * N + i] - mean[i];
            s += d * d;
        }
        norm[i] = sqrt(s);
        if (!(norm[i] > 0.0)) rc = -1;
    }
    if (rc == 0) {
        for (i = 0; i < N; i++) {
            C[(int64_t)i * N + i] = 1.0;
            for (j = i + 1; j < N; j++) {
                double s = 0.0;
                for (t = 0; t < T; t++)
                    s += (X[(int64_t)t * N + i] - mean[i]) * (X[(int64_t)t * N + j] - mean[j]);
                C[(int64_t)i * N + j] = s / (norm[i] * norm[j]);
                C[(int64_t)j * N + i] = C[(int64_t)i * N + j];
            }
        }
    }
    free(mean);
    free(norm);
    return rc;
}
