/*
 * qapb.h -- C ABI of libqapb.so, the B200 (sm_100a) implementation of the QAP
 * swap-delta hot path.
 *
 * This is the drop-in boundary for the reference's kernel-backend plugin
 * interface: the module object `qapsolve.backend.kernels`
 * (/root/reference/pkg/src/qapsolve/backend.py:16-29) whose members are
 *     full_cost   (_kernels.pyx:48-55)
 *     all_deltas  (_kernels.pyx:58-70)
 *     two_opt_run (_kernels.pyx:73-118)
 *     tabu_run    (_kernels.pyx:121-197)
 * plus the multi-start map/reduce that sits directly on top of them
 * (multistart.py:86-172: run_start / _run_chunk / run_multistart).
 *
 * Conventions
 *   - Every function returns a status code (QAPB_OK == 0).  No exceptions cross
 *     the boundary; qapb_last_error() returns a thread-local message.
 *   - All matrices, permutations and result arrays are int64, C-contiguous,
 *     0-based, exactly the layout the reference kernels take and return
 *     (`ctypedef long long i64`, _kernels.pyx:15).
 *   - Functions without a suffix take DEVICE pointers (e.g. torch
 *     `tensor.data_ptr()`), enqueue work on `stream` (a cudaStream_t passed as
 *     void*, NULL = default stream) and return without synchronising.  The
 *     caller owns all buffers; inputs are never written (_kernels.pyx:77,125).
 *   - `_host` variants take HOST pointers, perform the host<->device copies
 *     themselves and return after the result is in host memory.  They are what
 *     a ctypes/NumPy binding of `kernels.*` calls.
 *   - There is no CPU fallback: without a CUDA device every call fails with
 *     QAPB_ERR_CUDA.
 *   - A handle is bound to one device and owns a scratch workspace: it must not be
 *     used from two threads at the same time, nor have launches in flight on two
 *     streams at once (create one handle per stream for that).
 */
#ifndef QAPB_H
#define QAPB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QAPB_OK 0
#define QAPB_ERR_INVALID 1     /* bad argument          -> DomainError (errors.py:31) */
#define QAPB_ERR_CUDA 2        /* CUDA runtime failure  -> QapError    (errors.py:4)  */
#define QAPB_ERR_NOMEM 3       /* allocation failure    -> QapError                   */
#define QAPB_ERR_UNSUPPORTED 4 /* outside supported range (n > 1020, |entry| >= 2^30) */

#define QAPB_ALGO_2OPT 0
#define QAPB_ALGO_TABU 1

typedef struct qapb_handle qapb_handle;

/* Properties chosen for an instance at qapb_create time. */
typedef struct qapb_info {
    int32_t n;              /* instance size                                         */
    int32_t device;         /* CUDA device ordinal                                    */
    int32_t acc_bits;       /* 32 or 64: width of the on-chip delta state             */
    int32_t symmetric;      /* 1 if flow and distance are both symmetric              */
    int32_t threads;        /* CTA size of the search kernel                          */
    int32_t units_per_thread;
    int32_t storage;        /* 0: placement matrix in shared memory, 1: in L2/global,
                               2: placement matrix and tabu masks in L2/global,
                               3: hybrid kernel (registers + shared memory),
                               4: one warp per search (n <= 32; `threads` / 32 searches per
                                  CTA, twice that at n <= 16)                            */
    int32_t smem_bytes;     /* dynamic shared memory per CTA                          */
    int32_t ctas_per_sm;    /* resident searches per SM (occupancy query)             */
    int32_t sm_count;
    int64_t delta_bound;    /* proven bound on |delta| used to pick acc_bits          */
} qapb_info;

int qapb_version(void);
const char *qapb_last_error(void);
int qapb_device_count(int *count);

/* Upload an instance (host int64 n*n matrices: flow, distance -- the argument
 * order of every reference kernel) to `device`, analyse value ranges and pick
 * the kernel configuration.  Replaces the per-call `_as_matrix` conversions of
 * _kernels.pyx:44-45. */
int qapb_create(int n, const int64_t *flow, const int64_t *dist, int device, qapb_handle **out);
int qapb_destroy(qapb_handle *h);
int qapb_get_info(const qapb_handle *h, qapb_info *info);

/* kernels.full_cost (_kernels.pyx:48-55), batched: costs[b] = cost(perms[b,:]). */
int qapb_full_cost(qapb_handle *h, const int64_t *perms, int batch, int64_t *costs, void *stream);

/* kernels.all_deltas (_kernels.pyx:58-70), batched:
 * deltas[b, k] for the n(n-1)/2 moves in lexicographic (i, j) order. */
int qapb_all_deltas(qapb_handle *h, const int64_t *perms, int batch, int64_t *deltas, void *stream);

/* kernels.two_opt_run (_kernels.pyx:73-118), batched over `batch` starts.
 * best/cur: [batch, n]; best_cost/cur_cost: [batch];
 * move_i/move_j/move_delta: [batch, iterations], may be NULL together. */
int qapb_two_opt(qapb_handle *h, const int64_t *perms, int batch, int iterations,
                 int64_t *best, int64_t *best_cost, int64_t *cur, int64_t *cur_cost,
                 int64_t *move_i, int64_t *move_j, int64_t *move_delta, void *stream);

/* kernels.tabu_run (_kernels.pyx:121-197), batched.  tenures: [batch, iterations]
 * (tenures[b, c-1] belongs to the move accepted at iteration c, tabu.py:182-186).
 * Any int64 tenure with |c + tenure| < 2^31 is honoured (zero / negative: the cell
 * is never tabu); qapb_tabu_host refuses others, the device entry does not look.
 * cells: [batch, n, n] or NULL (upper triangle expiry, lower triangle counts);
 * stopped_early/steps_done: [batch] (0/1 and count);
 * trail_*: [batch, iterations] or NULL together; entries past steps_done are
 * left untouched.  The reference's `aspirated_flag` trail equals `tabu_flag`
 * (_kernels.pyx:185-186) so one array is produced. */
int qapb_tabu(qapb_handle *h, const int64_t *perms, int batch, int iterations,
              const int64_t *tenures, int64_t *best, int64_t *best_cost, int64_t *cur,
              int64_t *cur_cost, int64_t *cells, int64_t *stopped_early, int64_t *steps_done,
              int64_t *trail_i, int64_t *trail_j, int64_t *trail_delta, int64_t *trail_tabu,
              void *stream);

/* run_multistart's map + local reduce (multistart.py:86-118) for the starts
 * [first_index, first_index + count): each start derives its SplitMix64 state
 * on the device (rng.py:62-70), shuffles (core.py:81-87), draws its tenure
 * stream (tabu.py:184-186) and runs `iterations` steps.
 *   per_start_costs: [count]  best cost of each start
 *   best_key:        [2]      {min cost, its global start index}; ties -> lowest
 *                             index (multistart.py:114,156)
 *   best_perm:       [n]      best permutation of that start
 * ten_low/ten_high are ignored for QAPB_ALGO_2OPT. */
int qapb_multistart(qapb_handle *h, int algo, uint64_t master_seed, uint64_t first_index,
                    int count, int iterations, int64_t ten_low, int64_t ten_high,
                    int64_t *per_start_costs, int64_t *best_key, int64_t *best_perm,
                    void *stream);

/* The same map for an explicit list of starts: start b runs from the SplitMix64 state
 * seeds[b] (what rng.py:62-70 `derive_seed(master, index)` returns), so one launch can serve
 * several (master_seed, index range) runs at once -- the repetitions `master_seed + rep` of
 * cli.py:113-115 and the seeds axis `+ 7919 * idx` of cli.py:168-175.  No reduction is done:
 *   per_start_costs: [count]    best cost of each start
 *   best_perms:      [count,n]  best permutation of each start */
int qapb_multistart_seeds(qapb_handle *h, int algo, const uint64_t *seeds, int count, int iterations,
                          int64_t ten_low, int64_t ten_high, int64_t *per_start_costs,
                          int64_t *best_perms, void *stream);

/* qapb_multistart_seeds with each start's trajectory recorded: move_i/move_j/move_delta are
 * [count, iterations] (rows past steps_done[b] are left untouched; a tabu start can stop early,
 * _kernels.pyx:168-170).  The best cost after any shorter budget v is then
 *   c0 + min(0, min prefix sums of move_delta[b, :v])   with c0 = per_start_costs[b] - min(0, min prefix sums),
 * because the tenure stream of a run does not depend on its budget (tabu.py:184-186 draws it after the
 * start permutation, in order) -- so the `neighborhoods` sweep of cli.py:162-166 over increasing
 * iteration counts is ONE run at the largest count. */
int qapb_multistart_trace(qapb_handle *h, int algo, const uint64_t *seeds, int count, int iterations,
                          int64_t ten_low, int64_t ten_high, int64_t *per_start_costs,
                          int64_t *best_perms, int64_t *steps_done, int64_t *move_i, int64_t *move_j,
                          int64_t *move_delta, void *stream);

/* Host-buffer variants (synchronous; copies inside). */
int qapb_full_cost_host(qapb_handle *h, const int64_t *perms, int batch, int64_t *costs);
int qapb_all_deltas_host(qapb_handle *h, const int64_t *perms, int batch, int64_t *deltas);
int qapb_two_opt_host(qapb_handle *h, const int64_t *perms, int batch, int iterations,
                      int64_t *best, int64_t *best_cost, int64_t *cur, int64_t *cur_cost,
                      int64_t *move_i, int64_t *move_j, int64_t *move_delta);
int qapb_tabu_host(qapb_handle *h, const int64_t *perms, int batch, int iterations,
                   const int64_t *tenures, int64_t *best, int64_t *best_cost, int64_t *cur,
                   int64_t *cur_cost, int64_t *cells, int64_t *stopped_early,
                   int64_t *steps_done, int64_t *trail_i, int64_t *trail_j,
                   int64_t *trail_delta, int64_t *trail_tabu);
int qapb_multistart_host(qapb_handle *h, int algo, uint64_t master_seed, uint64_t first_index,
                         int count, int iterations, int64_t ten_low, int64_t ten_high,
                         int64_t *per_start_costs, int64_t *best_key, int64_t *best_perm);

int qapb_multistart_seeds_host(qapb_handle *h, int algo, const uint64_t *seeds, int count,
                               int iterations, int64_t ten_low, int64_t ten_high,
                               int64_t *per_start_costs, int64_t *best_perms);

int qapb_multistart_trace_host(qapb_handle *h, int algo, const uint64_t *seeds, int count,
                               int iterations, int64_t ten_low, int64_t ten_high,
                               int64_t *per_start_costs, int64_t *best_perms, int64_t *steps_done,
                               int64_t *move_i, int64_t *move_j, int64_t *move_delta);

/* Launch-configuration tuning (the GPU counterpart of the (N, t, b) space of tuner.py:28-78: here a
 * configuration is how one search is laid out on an SM).  `qapb_plan_candidates` lists the plans of
 * the register/shared-memory kernel that fit this instance as rows {register units per thread,
 * threads carrying off-diagonal units, shared-memory units per thread, diagonal blocks in shared
 * memory (0/1)} -- register units 0 names the one-warp-per-search kernel (n <= 32, the default there); {1, T, 0, 0} at
 * n > 128 is the register-only plan with one search per SM (n <= 176, two symmetric matrices; the default there); `qapb_set_plan` re-plans the handle with one of them (results are identical under
 * every plan; only the speed differs).  Instances served by the generic kernel have no candidates.
 * Instances with 64-bit deltas at n = 129..152 are re-planned by `qapb_multistart` itself according to the batch
 * size (at most one search per SM: register-only) until `qapb_set_plan` names a plan. */
int qapb_plan_candidates(qapb_handle *h, int32_t *plans /* [cap][4] */, int cap, int *count);
int qapb_set_plan(qapb_handle *h, int reg_units, int unit_threads, int smem_units, int diag_in_smem);

/* Time of the most recent search-kernel launch sequence on this handle, in
 * milliseconds between CUDA events recorded on the launching stream
 * (valid after the stream has been synchronised).  Used by bench.py for the
 * roofline figure. */
int qapb_last_kernel_ms(qapb_handle *h, float *ms);

/* Sum of steps_done over the starts of the most recent qapb_multistart on this handle (synchronises
 * with that launch).  A tabu start can stop early (_kernels.pyx:168-170), so the number of move
 * evaluations of a run is this sum times n(n-1)/2, not starts x iterations. */
int qapb_last_total_steps(qapb_handle *h, int64_t *steps);

/* Integer-pipe peak probe: runs a dependent-chain-free IMAD/IADD3 loop on every
 * SM and reports lane-operations per second (the roofline denominator SURVEY.md
 * section 8d asks to be measured on the box).  `kind`: 0 = IMAD only,
 * 1 = IADD3 only, 2 = mixed 1:1. */
int qapb_probe_int_peak(int device, int kind, double *ops_per_sec);

/* Shared-memory bandwidth probe: conflict-free 128-bit loads on every SM, bytes per second (the
 * shared-memory roofline denominator of SURVEY.md section 8d). */
int qapb_probe_smem_peak(int device, double *bytes_per_sec);

#ifdef __cplusplus
}
#endif
#endif /* QAPB_H */
