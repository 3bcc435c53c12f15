/*
 * qap_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-file CPU restatement of the reference's swap-delta hot path
 * (package `qapsolve` under /root/reference/pkg/src/qapsolve).  It exists to
 * check the CUDA path; it is never linked, imported or called by the product
 * (paper_2307_11248_b200/).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function here
 * against (a) the reference's literal known answers (toy2 costs 13/17, delta
 * +4, the tenure table) and (b) golden vectors produced by running the
 * reference itself in the build container (tests/golden/make_golden.py), and
 * -- when oracle/_ref/_kernels*.so (the reference's own Cython kernel compiled
 * from /root/reference) is present -- against that library directly.
 *
 * Every function cites the reference lines it restates.  All arithmetic is
 * int64 / uint64 exactly as in the reference (`ctypedef long long i64`,
 * _kernels.pyx:15; 64-bit masking in rng.py:9-20).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;
typedef uint64_t u64;

#define ORC_GAMMA 0x9E3779B97F4A7C15ULL

/* ------------------------------------------------------------------ RNG -- */

/* rng.py:15-20  mix64: Stafford variant 13 finaliser on 64-bit words. */
u64 orc_mix64(u64 z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.py:35-37  SplitMix64.next64: advance by GAMMA, output mix64(state). */
u64 orc_next64(u64 *state)
{
    *state += ORC_GAMMA;
    return orc_mix64(*state);
}

/* rng.py:39-47  randbelow: rejection sampling against
 * limit = 2^64 - (2^64 mod bound).  In 64-bit words: rem = (-bound) % bound
 * equals 2^64 mod bound, and r < limit  <=>  r <= UINT64_MAX - rem. */
u64 orc_randbelow(u64 *state, u64 bound)
{
    u64 rem = (0ULL - bound) % bound;
    u64 last_ok = UINT64_MAX - rem;
    for (;;) {
        u64 r = orc_next64(state);
        if (r <= last_ok)
            return r % bound;
    }
}

/* rng.py:62-70  derive_seed: mix64(master + GAMMA*(index+1)) mod 2^64. */
u64 orc_derive_seed(u64 master_seed, u64 start_index)
{
    return orc_mix64(master_seed + ORC_GAMMA * (start_index + 1ULL));
}

/* core.py:81-87 + rng.py:55-59  identity then Fisher-Yates from the top:
 * for i = n-1 .. 1: j = randbelow(i+1); swap(seq[i], seq[j]). */
void orc_random_permutation(int n, u64 *state, i64 *perm)
{
    for (int i = 0; i < n; ++i)
        perm[i] = i;
    for (int i = n - 1; i >= 1; --i) {
        u64 j = orc_randbelow(state, (u64)i + 1ULL);
        i64 t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
    }
}

/* tabu.py:40-46  tenure_bounds: low = max(1, n//10), high = max(low, ceil(.33 n)). */
void orc_tenure_bounds(int n, i64 *low, i64 *high)
{
    i64 lo = n / 10;
    if (lo < 1) lo = 1;
    i64 hi = (33 * (i64)n + 99) / 100;
    if (hi < lo) hi = lo;
    *low = lo;
    *high = hi;
}

/* tabu.py:184-186 + rng.py:49-52  one randint(low, high) per potential
 * iteration, drawn after the shuffle; a draw is consumed even if low == high. */
void orc_draw_tenures(u64 *state, i64 low, i64 high, int iterations, i64 *tenures)
{
    u64 span = (u64)(high - low + 1);
    for (int c = 0; c < iterations; ++c)
        tenures[c] = low + (i64)orc_randbelow(state, span);
}

/* instance.py:194-209  random_instance: row-major fill, flow first then
 * distance, zero diagonal, off-diagonal low + randbelow(high-low+1). */
void orc_random_instance(int n, u64 *state, i64 low, i64 high, i64 *flow, i64 *dist)
{
    u64 span = (u64)(high - low + 1);
    i64 *mats[2] = {flow, dist};
    for (int m = 0; m < 2; ++m)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                mats[m][(size_t)i * n + j] = (i == j) ? 0 : low + (i64)orc_randbelow(state, span);
}

/* ----------------------------------------------------------- cost core -- */

/* _kernels.pyx:18-24  full cost = sum_i sum_j F[p_i, p_j] * D[i, j]. */
i64 orc_full_cost(int n, const i64 *F, const i64 *D, const i64 *p)
{
    i64 total = 0;
    for (int i = 0; i < n; ++i) {
        const i64 *frow = F + (size_t)p[i] * n;
        const i64 *drow = D + (size_t)i * n;
        for (int j = 0; j < n; ++j)
            total += frow[p[j]] * drow[j];
    }
    return total;
}

/* _kernels.pyx:27-41  O(n) exchange delta for locations i < j: direct term,
 * diagonal term, then the k-loop over every other location. */
i64 orc_delta(int n, const i64 *F, const i64 *D, const i64 *p, int i, int j)
{
#define F_(a, b) F[(size_t)(a) * n + (b)]
#define D_(a, b) D[(size_t)(a) * n + (b)]
    i64 pi = p[i], pj = p[j];
    i64 acc = (D_(j, i) - D_(i, j)) * (F_(pi, pj) - F_(pj, pi))
            + (F_(pj, pj) - F_(pi, pi)) * (D_(i, i) - D_(j, j));
    for (int k = 0; k < n; ++k) {
        if (k == i || k == j)
            continue;
        i64 pk = p[k];
        acc += (D_(j, k) - D_(i, k)) * (F_(pi, pk) - F_(pj, pk))
             + (D_(k, j) - D_(k, i)) * (F_(pk, pi) - F_(pk, pj));
    }
    return acc;
#undef F_
#undef D_
}

/* _kernels.pyx:58-70  all n(n-1)/2 deltas in lexicographic (i, j) order. */
void orc_all_deltas(int n, const i64 *F, const i64 *D, const i64 *p, i64 *out)
{
    size_t k = 0;
    for (int i = 0; i < n - 1; ++i)
        for (int j = i + 1; j < n; ++j)
            out[k++] = orc_delta(n, F, D, p, i, j);
}

/* ----------------------------------------------------------------- 2opt -- */

/* _kernels.pyx:73-118  two_opt_run: every step takes the lexicographically
 * first minimum-delta move (strict <, :104), applies it unconditionally
 * (:108-111), tracks best on strict < (:112-114), logs (i, j, delta).
 * `perm0` is not modified (:77).  Outputs: best[n], cur[n], move_*[iterations]. */
void orc_two_opt_run(int n, const i64 *F, const i64 *D, const i64 *perm0, int iterations,
                     i64 *best, i64 *best_cost_out, i64 *cur, i64 *cur_cost_out,
                     i64 *move_i, i64 *move_j, i64 *move_delta)
{
    memcpy(cur, perm0, sizeof(i64) * (size_t)n);
    memcpy(best, perm0, sizeof(i64) * (size_t)n);
    i64 cost = orc_full_cost(n, F, D, cur);
    i64 best_cost = cost;
    for (int step = 0; step < iterations; ++step) {
        int bi = 0, bj = 1;
        i64 bd = orc_delta(n, F, D, cur, 0, 1);
        for (int i = 0; i < n - 1; ++i)
            for (int j = i + 1; j < n; ++j) {
                if (i == 0 && j == 1)
                    continue;
                i64 d = orc_delta(n, F, D, cur, i, j);
                if (d < bd) {
                    bd = d;
                    bi = i;
                    bj = j;
                }
            }
        i64 t = cur[bi];
        cur[bi] = cur[bj];
        cur[bj] = t;
        cost += bd;
        if (cost < best_cost) {
            best_cost = cost;
            memcpy(best, cur, sizeof(i64) * (size_t)n);
        }
        if (move_i) move_i[step] = bi;
        if (move_j) move_j[step] = bj;
        if (move_delta) move_delta[step] = bd;
    }
    *best_cost_out = best_cost;
    *cur_cost_out = cost;
}

/* ----------------------------------------------------------------- tabu -- */

/* _kernels.pyx:121-197  tabu_run.  Iteration counter c runs 1..iterations.
 *   admissible(i,j)  <=>  cells[i][j] <= c  ||  cost + delta < best_cost   (:162)
 *   choose the lexicographically first minimum delta among admissible   (:163-167)
 *   none admissible -> stopped_early, steps_done = c-1                   (:168-170)
 *   was_tabu = cells[bi][bj] > c                                         (:171)
 *   swap; cost += bd; cells[bi][bj] = c + tenures[c-1]; cells[bj][bi] += 1 (:172-178)
 *   best on strict <                                                      (:179-181)
 *   trail row (bi, bj, bd, was_tabu, was_tabu, t)                         (:182-187)
 * `cells` is n*n, zero-initialised here (:137).  Trail pointers may be NULL.
 * Returns steps_done. */
int orc_tabu_run(int n, const i64 *F, const i64 *D, const i64 *perm0, int iterations,
                 const i64 *tenures,
                 i64 *best, i64 *best_cost_out, i64 *cur, i64 *cur_cost_out,
                 i64 *cells, int *stopped_early_out,
                 i64 *t_i, i64 *t_j, i64 *t_delta, i64 *t_tabu, i64 *t_asp, i64 *t_tenure)
{
    memcpy(cur, perm0, sizeof(i64) * (size_t)n);
    memcpy(best, perm0, sizeof(i64) * (size_t)n);
    memset(cells, 0, sizeof(i64) * (size_t)n * (size_t)n);
    i64 cost = orc_full_cost(n, F, D, cur);
    i64 best_cost = cost;
    int steps_done = 0, stopped = 0;
    for (int c = 1; c <= iterations; ++c) {
        int found = 0, bi = 0, bj = 0;
        i64 bd = 0;
        for (int i = 0; i < n - 1; ++i)
            for (int j = i + 1; j < n; ++j) {
                i64 d = orc_delta(n, F, D, cur, i, j);
                if (cells[(size_t)i * n + j] <= c || cost + d < best_cost) {
                    if (!found || d < bd) {
                        found = 1;
                        bd = d;
                        bi = i;
                        bj = j;
                    }
                }
            }
        if (!found) {
            stopped = 1;
            break;
        }
        int was_tabu = cells[(size_t)bi * n + bj] > c;
        i64 t = cur[bi];
        cur[bi] = cur[bj];
        cur[bj] = t;
        cost += bd;
        i64 ten = tenures[c - 1];
        cells[(size_t)bi * n + bj] = c + ten;
        cells[(size_t)bj * n + bi] += 1;
        if (cost < best_cost) {
            best_cost = cost;
            memcpy(best, cur, sizeof(i64) * (size_t)n);
        }
        if (t_i) t_i[c - 1] = bi;
        if (t_j) t_j[c - 1] = bj;
        if (t_delta) t_delta[c - 1] = bd;
        if (t_tabu) t_tabu[c - 1] = was_tabu;
        if (t_asp) t_asp[c - 1] = was_tabu;
        if (t_tenure) t_tenure[c - 1] = ten;
        steps_done = c;
    }
    *best_cost_out = best_cost;
    *cur_cost_out = cost;
    *stopped_early_out = stopped;
    return steps_done;
}

/* ----------------------------------------------------------- multistart -- */

/* multistart.py:86-93 (run_start) -> two_opt.py:64-69 / tabu.py:178-189:
 * state = derive_seed(master, index); shuffle; (tabu only) draw `iterations`
 * tenures; run the kernel; keep the best permutation and cost.
 * algo: 0 = 2opt, 1 = tabu.  Returns the best cost of this start. */
i64 orc_run_start(int n, const i64 *F, const i64 *D, int algo, u64 master_seed, u64 index,
                  int iterations, i64 ten_low, i64 ten_high, i64 *best_perm,
                  i64 *work /* >= 2n + n*n + iterations words */)
{
    u64 state = orc_derive_seed(master_seed, index);
    i64 *start = work;
    i64 *cur = work + n;
    i64 *cells = work + 2 * (size_t)n;
    i64 *tenures = cells + (size_t)n * n;
    i64 best_cost = 0, cur_cost = 0;
    orc_random_permutation(n, &state, start);
    if (algo == 1) {
        int stopped = 0;
        orc_draw_tenures(&state, ten_low, ten_high, iterations, tenures);
        orc_tabu_run(n, F, D, start, iterations, tenures, best_perm, &best_cost, cur, &cur_cost,
                     cells, &stopped, NULL, NULL, NULL, NULL, NULL, NULL);
    } else {
        orc_two_opt_run(n, F, D, start, iterations, best_perm, &best_cost, cur, &cur_cost,
                        NULL, NULL, NULL);
    }
    return best_cost;
}

/* multistart.py:121-172  run_multistart: starts first_index .. first_index+count-1,
 * per_start_costs[k] = best cost of start first_index+k; winner = minimum cost,
 * ties to the lowest start index (:114 strict <, :156 key (cost, index)).
 * `threads` > 1 spreads starts over OpenMP threads (the reference uses a
 * process pool, :141-150; the result is scheduling-independent by construction).
 * Returns 0, or -1 if scratch memory could not be allocated. */
int orc_multistart(int n, const i64 *F, const i64 *D, int algo, u64 master_seed,
                   u64 first_index, int count, int iterations, i64 ten_low, i64 ten_high,
                   int threads, i64 *per_start_costs, i64 *best_cost_out, i64 *best_index_out,
                   i64 *best_perm_out)
{
    int failed = 0;
    size_t work_words = 2 * (size_t)n + (size_t)n * n + (size_t)iterations;
    i64 win_cost = 0, win_index = -1;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
#endif
    {
        i64 *work = (i64 *)malloc(sizeof(i64) * work_words);
        i64 *perm = (i64 *)malloc(sizeof(i64) * (size_t)n);
        i64 *my_perm = (i64 *)malloc(sizeof(i64) * (size_t)n);
        i64 my_cost = 0, my_index = -1;
        if (!work || !perm || !my_perm) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            failed = 1;
        } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
            for (int k = 0; k < count; ++k) {
                u64 index = first_index + (u64)k;
                i64 c = orc_run_start(n, F, D, algo, master_seed, index, iterations, ten_low,
                                      ten_high, perm, work);
                per_start_costs[k] = c;
                if (my_index < 0 || c < my_cost || (c == my_cost && (i64)index < my_index)) {
                    my_cost = c;
                    my_index = (i64)index;
                    memcpy(my_perm, perm, sizeof(i64) * (size_t)n);
                }
            }
#ifdef _OPENMP
#pragma omp critical
#endif
            {
                if (my_index >= 0 &&
                    (win_index < 0 || my_cost < win_cost ||
                     (my_cost == win_cost && my_index < win_index))) {
                    win_cost = my_cost;
                    win_index = my_index;
                    memcpy(best_perm_out, my_perm, sizeof(i64) * (size_t)n);
                }
            }
        }
        free(work);
        free(perm);
        free(my_perm);
    }
    if (failed)
        return -1;
    *best_cost_out = win_cost;
    *best_index_out = win_index;
    return 0;
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
