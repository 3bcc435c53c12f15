// qapb.cu -- C ABI (include/qapb.h) over the sm_100a search kernels.
//
// Host responsibilities: value-range analysis of the instance (int32 vs int64
// on-chip state), packing (zero-diagonal int32 copies of F, D and their
// transposes, padded to a multiple of 4), kernel configuration (CTA size, units
// per thread, where the placement matrix lives), workspace and launches.
#include "../../include/qapb.h"
#include "search_kernel.cuh"
#include "build_kernels.cuh"
#include "search_hybrid.cuh"
#include "search_warp.cuh"

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

using namespace qapb;

int g_attr_smem(int device);  // opt-in shared memory per block of a device seen by qapb_create
static cudaError_t ensure_smem_optin(const void *kern, int device, unsigned bytes);
static thread_local std::string g_err;
static int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}
#define CU(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(QAPB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct qapb_handle {
    int n = 0, nb = 0, npad = 0, device = 0;
    int acc_bits = 32, symmetric = 0;
    int sym_mode = 0;  // generic kernel: 0 two products per entry, 1 both symmetric, 2 D only, 3 F only
    int nunits = 0, noff = 0, threads = 0, upt = 0, storage = 0;
    int lb_class = 0;  // 0: <=384 threads, 2 CTAs/SM register budget; 1: <=512 threads
    int toff = 0, us = 0, exp_in_smem = 1;         // hybrid plan
    int staged = 0, fits_i16 = 0;                  // int16 copies of D/F staged in shared memory
    int dsm = 0;                                   // hybrid: diagonal blocks in shared memory (no dedicated warps)
    int dd = 0;                                    // hybrid: diagonal blocks paired in the registers of the threads after the last unit
    int ow = 0;                                    // hybrid: the search is one warp (n <= 32 with dd)
    int wide = 0;                                  // hybrid: unsigned 32-bit state with 64-bit deltas (acc_bits holds the STATE width, 32)
    int wk = 0;                                    // lanes per search (32, or 16 at n <= 16) of the warp kernel (search_warp.cuh; n <= 32), 0 = other plans
    int wpc = 1;                                   // ... warps per CTA
    // 64-bit deltas at n > 128: the default plan (two searches per SM, part of the state in shared memory) wins when both
    // slots of every SM are taken; a batch of at most one search per SM runs faster on the register-only plan (tai150b,
    // 148 starts: 477 against 356 G evals/s).  qapb_multistart switches between the two by batch size unless the caller
    // chose a plan itself (qapb_set_plan) -- results are identical under every plan.
    int have_alt = 0, user_plan = 0, def_plan[4] = {0, 0, 0, 0}, alt_plan[4] = {0, 0, 0, 0};
    unsigned smem_bytes = 0;
    int ctas_per_sm = 0, sm_count = 0;
    long long delta_bound = 0;
    int32_t *dF = nullptr, *dFT = nullptr, *dD = nullptr, *dDT = nullptr, *dfd = nullptr, *ddd = nullptr;
    uint16_t *dunit = nullptr;
    void *arena = nullptr;  // one block holding all of the above
    size_t arena_bytes = 0;
    void *ws = nullptr;
    size_t ws_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int have_timing = 0;
    int force_seq_rng = 0;
    size_t steps_total_off = (size_t)-1;  // workspace offset of the last multistart's summed steps_done
};

typedef void (*kern_t)(const SearchParams);
#ifndef QAPB_DEV_REGS
#define QAPB_DEV_REGS 88
#endif
#ifdef QAPB_DEV_ONLY
// development build (seconds instead of minutes): only one instantiation, -DQAPB_DEV_ONLY=<preset>
#if QAPB_DEV_ONLY == 1   // tai100a / sko100 multi-start tabu (staged one-register-unit plan)
#define QAPB_DEV_ARGS 1, true, 1, false, true, 80, false, false, false
#elif QAPB_DEV_ONLY == 2 // tai256c multi-start tabu (shared-memory units, DSM)
#define QAPB_DEV_ARGS 1, true, 2, true, false, 128, true, false, false
#elif QAPB_DEV_ONLY == 4 // preset 1 with paired diagonal blocks (DD), 64 registers
#define QAPB_DEV_ARGS 1, true, 1, false, true, 64, false, false, false, true
#elif QAPB_DEV_ONLY == 7 // preset 1 at 56 registers (three 352-thread CTAs per SM)
#define QAPB_DEV_ARGS 1, true, 1, false, true, 56, false, false, false
#elif QAPB_DEV_ONLY == 6 // DD at 80 registers
#define QAPB_DEV_ARGS 1, true, 1, false, true, 80, false, false, false, true
#elif QAPB_DEV_ONLY == 8 // one-warp searches (n <= 32), multi-start tabu
#define QAPB_DEV_ARGS 1, true, 1, false, false, 64, false, false, false, true, true
#elif QAPB_DEV_ONLY == 9 // tai150b: 64-bit deltas over unsigned 32-bit state, shared-memory plan with DSM, one symmetric matrix
#define QAPB_DEV_ARGS 2, false, 2, true, false, 128, true, false, true, false, false, true
#elif QAPB_DEV_ONLY == 12 // preset 1 at 88 registers (still two 352-thread CTAs per SM)
#ifndef QAPB_DEV_REGS
#define QAPB_DEV_REGS 88
#endif
#define QAPB_DEV_ARGS 1, true, 1, false, true, QAPB_DEV_REGS, false, false, false
#elif QAPB_DEV_ONLY == 13 // one-warp searches at 80 registers (25 per SM)
#define QAPB_DEV_ARGS 1, true, 1, false, false, 80, false, false, false, true, true
#elif QAPB_DEV_ONLY == 14 // one-warp searches at 96 registers (21 per SM)
#define QAPB_DEV_ARGS 1, true, 1, false, false, 96, false, false, false, true, true
#elif QAPB_DEV_ONLY == 15 // preset 9 without the recording code (multi-start only)
#define QAPB_DEV_ARGS 2, false, 2, true, false, 128, true, false, false, false, false, true
#elif QAPB_DEV_ONLY == 5 // recording instantiation of preset 4
#define QAPB_DEV_ARGS 1, true, 1, false, true, 64, false, false, true, true
#elif QAPB_DEV_ONLY == 3 // recording instantiation of preset 1 (single-run entries: parity tests)
#define QAPB_DEV_ARGS 1, true, 1, false, true, 80
#elif QAPB_DEV_ONLY == 40 // ONE register unit + shared-memory units, DSM, multi-start tabu (n = 129..256: QAPB_PLAN=1,512,3,1 + QAPB_UR1_SMEM=1)
#define QAPB_DEV_ARGS 1, true, 1, true, false, QAPB_DEV_REGS, true, false, false
#elif QAPB_DEV_ONLY == 41 // ... with 64-bit deltas, one symmetric matrix (tai150b: QAPB_PLAN=1,256,2,1)
#define QAPB_DEV_ARGS 2, false, 1, true, false, QAPB_DEV_REGS, true, false, false, false, false, true
#elif QAPB_DEV_ONLY == 42 // register-only plan at n = 129..180 (size class 256), one search per SM, multi-start tabu
#define QAPB_DEV_ARGS 1, true, 1, false, false, QAPB_DEV_REGS, false, false, false, false, false, false, true
#elif QAPB_DEV_ONLY == 43 // ... with 64-bit deltas, one symmetric matrix (tai150b)
#define QAPB_DEV_ARGS 2, false, 1, false, false, 80, false, false, false, false, false, true, true
#elif QAPB_DEV_ONLY == 20 // one warp per search (search_warp.cuh), symmetric, multi-start tabu
#define QAPB_DEV_WARP 1, false, false, 32
#elif QAPB_DEV_ONLY == 21 // ... recording instantiation
#define QAPB_DEV_WARP 1, false, true, 32
#elif QAPB_DEV_ONLY == 22 // ... multi-start 2opt
#define QAPB_DEV_WARP 1, true, false, 32
#elif QAPB_DEV_ONLY == 23 // ... asymmetric recording instantiation
#define QAPB_DEV_WARP 0, false, true, 32
#elif QAPB_DEV_ONLY == 24 // ... two searches per warp (n <= 16), multi-start tabu
#define QAPB_DEV_WARP 1, false, false, 16
#elif QAPB_DEV_ONLY == 25 // ... two searches per warp, recording instantiation
#define QAPB_DEV_WARP 1, false, true, 16
#elif QAPB_DEV_ONLY == 26 // ... two searches per warp, asymmetric recording instantiation
#define QAPB_DEV_WARP 0, false, true, 16
#endif
#ifdef QAPB_DEV_WARP
#define QAPB_DEV_KERNEL qap_search_warp_kernel<QAPB_DEV_WARP>
#else
#define QAPB_DEV_KERNEL qap_search_hybrid_kernel<QAPB_DEV_ARGS>
#endif
static kern_t pick_kernel(int, int, int) { return (kern_t) QAPB_DEV_KERNEL; }
static kern_t pick_hybrid_kernel(int, int, int) { return (kern_t) QAPB_DEV_KERNEL; }
static kern_t multistart_kernel(int, int, int, int, int) { return (kern_t) QAPB_DEV_KERNEL; }
static kern_t pick_wide_kernel(int, int) { return (kern_t) QAPB_DEV_KERNEL; }
static kern_t pick_warp_kernel(int, int, int, int) { return (kern_t) QAPB_DEV_KERNEL; }
static kern_t pick_np256_kernel(int, int, int) { return (kern_t) QAPB_DEV_KERNEL; }
static kern_t pick_wide_np256_kernel(int) { return (kern_t) QAPB_DEV_KERNEL; }
#else
static kern_t pick_kernel(int acc_bits, int storage, int lb_class)
{
#define K(A, S, MT, MB) (kern_t) qap_search_kernel<A, S, MT, MB>
    static kern_t tab[2][3][2] = {
        {{K(int32_t, 0, 384, 2), K(int32_t, 0, 512, 1)}, {K(int32_t, 1, 384, 2), K(int32_t, 1, 512, 1)},
         {K(int32_t, 2, 384, 2), K(int32_t, 2, 512, 1)}},
        {{K(int64_t, 0, 384, 1), K(int64_t, 0, 512, 1)}, {K(int64_t, 1, 384, 1), K(int64_t, 1, 512, 1)},
         {K(int64_t, 2, 384, 1), K(int64_t, 2, 512, 1)}},
    };
#undef K
    return tab[acc_bits == 64][storage][lb_class];
}

// WIDE instantiations (unsigned 32-bit state, 64-bit deltas; never packed): the one-register-unit plan without /
// with staged matrices and the shared-memory plan with DSM.
static kern_t pick_wide_kernel(int symm, int plan)
{
#define KW(S) {(kern_t) qap_search_hybrid_kernel<S, false, 1, false, false, 80, false, false, true, false, false, true>, \
               (kern_t) qap_search_hybrid_kernel<S, false, 1, false, true, 80, false, false, true, false, false, true>,  \
               (kern_t) qap_search_hybrid_kernel<S, false, 2, true, false, 128, true, false, true, false, false, true>,  \
               (kern_t) qap_search_hybrid_kernel<S, false, 1, true, false, 128, true, false, true, false, false, true>}
    static kern_t tab[3][4] = {KW(0), KW(1), KW(2)};
#undef KW
    return tab[symm][plan == 9 ? 3 : plan == 5 ? 2 : plan];
}

static kern_t pick_hybrid_kernel(int symm, int packed, int plan)
{
    // symm: 0 both matrices asymmetric, 1 both symmetric, 2 exactly one symmetric (plans 0, 1, 5 only)
    // plan 0: register-only (n <= 128), 80 registers/thread (two 352-thread CTAs per SM at n = 100)
    // plan 1: the same with int16 copies of D and F staged in shared memory
    // plan 2: two register units + shared-memory units per thread, 128 registers (n <= 256)
    // plan 3/4: two register units per thread on half the threads, 112 registers (109 <= n <= 120:
    //           two CTAs per SM where plan 0/1 would fit only one), without / with int16 staging
    // plan 5: plan 2 with the diagonal blocks in shared memory (no dedicated diagonal warps)
    // plan 6/7: plan 0/1 with the diagonal blocks paired in the threads after the last unit (DD), 64 registers
    // plan 8: plan 6 as ONE warp (n <= 32): warp barriers, 32 searches per SM
    // plan 9: plan 5 with ONE register unit per thread (the rest in shared memory): no spills at 128 registers --
    //         instantiated for two symmetric matrices with packed keys (tai256c: 846 -> 887 G evals/s) and for 64-bit deltas
    if (plan == 9) return (kern_t) qap_search_hybrid_kernel<1, true, 1, true, false, 128, true>;
#define KH(S, PK) {(kern_t) qap_search_hybrid_kernel<S, PK, 1, false, false, 80>, \
                   (kern_t) qap_search_hybrid_kernel<S, PK, 1, false, true, 80>,  \
                   (kern_t) qap_search_hybrid_kernel<S, PK, 2, true, false, 128>,  \
                   (kern_t) qap_search_hybrid_kernel<S, PK, 2, false, false, 112>, \
                   (kern_t) qap_search_hybrid_kernel<S, PK, 2, false, true, 112>, \
                   (kern_t) qap_search_hybrid_kernel<S, PK, 2, true, false, 128, true>,  \
                   (kern_t) qap_search_hybrid_kernel<S, PK, 1, false, false, 64, false, false, true, true>, \
                   (kern_t) qap_search_hybrid_kernel<S, PK, 1, false, true, 64, false, false, true, true>, \
                   (kern_t) qap_search_hybrid_kernel<S, PK, 1, false, false, 64, false, false, true, true, true>}
#define KH2(PK) {(kern_t) qap_search_hybrid_kernel<2, PK, 1, false, false, 80>, \
                 (kern_t) qap_search_hybrid_kernel<2, PK, 1, false, true, 80>,  \
                 nullptr, nullptr, nullptr,                                     \
                 (kern_t) qap_search_hybrid_kernel<2, PK, 2, true, false, 128, true>,  \
                 (kern_t) qap_search_hybrid_kernel<2, PK, 1, false, false, 64, false, false, true, true>, \
                 (kern_t) qap_search_hybrid_kernel<2, PK, 1, false, true, 64, false, false, true, true>, \
                 (kern_t) qap_search_hybrid_kernel<2, PK, 1, false, false, 64, false, false, true, true, true>}
    static kern_t tab[3][2][9] = {{KH(0, false), KH(0, true)}, {KH(1, false), KH(1, true)}, {KH2(false), KH2(true)}};
#undef KH
#undef KH2
    kern_t k = tab[symm][packed != 0][plan];
    return k ? k : tab[0][packed != 0][plan];  // no one-symmetric-matrix instantiation of this plan: two products
}
// Multi-start instantiations of the two plans the benchmarks use (the staged one-register-unit plan and
// the shared-memory plan with DSM; packed keys; both matrices symmetric or neither): no trail / cells
// code, and for 2opt a selection without tabu bits.  null = use the common kernel.
// (regs88: the staged one-register-unit plan compiled for 88 instead of 80 registers -- ptxas schedules the pass
// with more values in flight: n = 100 tabu 852 -> 878, 2opt 895 -> 918, sko100 812 -> 836 G evals/s -- used when it
// costs no resident CTA, and for two symmetric matrices only: the two-product kernel LOSES at 88 (rand100 670 -> 467).)
static kern_t multistart_kernel(int symm, int packed, int plan, int two_opt, int regs88)
{
    if (!packed || symm > 1) return nullptr;
    if (plan == 9)
        return two_opt ? (kern_t) qap_search_hybrid_kernel<1, true, 1, true, false, 128, true, true, false>
                       : (kern_t) qap_search_hybrid_kernel<1, true, 1, true, false, 128, true, false, false>;
#define KM(S, NT) (plan == 1 ? ((regs88 && S == 1) ? (kern_t) qap_search_hybrid_kernel<1, true, 1, false, true, 88, false, NT, false> \
                                       : (kern_t) qap_search_hybrid_kernel<S, true, 1, false, true, 80, false, NT, false>) \
                   : plan == 7 ? (kern_t) qap_search_hybrid_kernel<S, true, 1, false, true, 64, false, NT, false, true> \
                   : plan == 8 ? (kern_t) qap_search_hybrid_kernel<S, true, 1, false, false, 64, false, NT, false, true, true> \
                             : (kern_t) qap_search_hybrid_kernel<S, true, 2, true, false, 128, true, NT, false>)
    if (plan != 1 && plan != 5 && plan != 7 && plan != 8) return nullptr;
    if (two_opt) return symm ? KM(1, true) : KM(0, true);
    return symm ? KM(1, false) : KM(0, false);
#undef KM
}
// One warp per search (search_warp.cuh): recording instantiations for the single-run entries, and multi-start
// instantiations (tabu / 2opt) without the recording code.
static kern_t pick_warp_kernel(int symm, int multistart, int two_opt, int lanes)
{
#define KW3(G) {{(kern_t) qap_search_warp_kernel<0, false, true, G>, (kern_t) qap_search_warp_kernel<0, false, false, G>, \
                 (kern_t) qap_search_warp_kernel<0, true, false, G>},                                                     \
                {(kern_t) qap_search_warp_kernel<1, false, true, G>, (kern_t) qap_search_warp_kernel<1, false, false, G>, \
                 (kern_t) qap_search_warp_kernel<1, true, false, G>}}
    static kern_t tab[2][2][3] = {KW3(32), KW3(16)};
#undef KW3
    return tab[lanes == 16][symm != 0][!multistart ? 0 : two_opt ? 2 : 1];
}
// Register-only plan at n = 129..176 (NP256: the n <= 128 kernel in layout size class 256), ONE search per SM on
// noff + 64 threads: 80 registers up to 800 threads (n <= 152; +3 % over 72), 72 up to 896 (n <= 164), 64 up to 1024 (n <= 176).  Two symmetric matrices
// with packed keys; recording / multi-start tabu / multi-start 2opt instantiations.
static kern_t pick_np256_kernel(int multistart, int two_opt, int regs)
{
#define KN(R) {(kern_t) qap_search_hybrid_kernel<1, true, 1, false, false, R, false, false, true, false, false, false, true>,  \
               (kern_t) qap_search_hybrid_kernel<1, true, 1, false, false, R, false, false, false, false, false, false, true>, \
               (kern_t) qap_search_hybrid_kernel<1, true, 1, false, false, R, false, true, false, false, false, false, true>}
    static kern_t tab[3][3] = {KN(80), KN(72), KN(64)};
#undef KN
    return tab[regs == 64 ? 2 : regs == 72 ? 1 : 0][!multistart ? 0 : two_opt ? 2 : 1];
}
// ... with 64-bit deltas (80 registers, at most 800 threads: n <= 152), per symmetry class
static kern_t pick_wide_np256_kernel(int symm)
{
#define KWN(S) (kern_t) qap_search_hybrid_kernel<S, false, 1, false, false, 80, false, false, true, false, false, true, true>
    static kern_t tab[3] = {KWN(0), KWN(1), KWN(2)};
#undef KWN
    return tab[symm];
}
#endif

// Resident CTAs per SM of `k` at this handle's CTA size and shared memory (cached: the query costs more than
// packing a small instance).
static int kernel_occupancy(const void *k, const qapb_handle *h)
{
    struct Key { const void *k; int threads; unsigned smem; int device; int occ; };
    static std::mutex mu;
    static std::vector<Key> seen;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const Key &e : seen)
            if (e.k == k && e.threads == h->threads && e.smem == h->smem_bytes && e.device == h->device) return e.occ;
    }
    int occ = 0;
    if (ensure_smem_optin(k, h->device, h->smem_bytes) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, h->threads, h->smem_bytes) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    std::lock_guard<std::mutex> lk(mu);
    seen.push_back({k, h->threads, h->smem_bytes, h->device, occ});
    return occ;
}

static kern_t handle_kernel(const qapb_handle *h, int multistart = 0, int two_opt = 0)
{
    // packed (delta, slot) keys need |delta|*16 + 15 < 2^31
    const int packed = h->delta_bound < ((1LL << 27) - 1);
    int plan = h->us > 0 ? 2 : (h->upt == 2 ? (h->staged ? 4 : 3) : (h->staged ? 1 : 0));
    if (h->dsm) plan = h->upt == 1 ? 9 : 5;
    if (h->dd) plan = h->ow ? 8 : h->staged ? 7 : 6;
    const int symm = h->symmetric ? 1 : (h->sym_mode >= 2 ? 2 : 0);
    if (h->storage == 3 && h->wk) return pick_warp_kernel(h->symmetric ? 1 : 0, multistart, two_opt, h->wk);
    if (h->storage == 3 && h->npad > 128 && h->us == 0 && h->wide) return pick_wide_np256_kernel(symm);
    if (h->storage == 3 && h->npad > 128 && h->us == 0) return pick_np256_kernel(multistart, two_opt, h->threads <= 800 ? 80 : h->threads <= 896 ? 72 : 64);
    if (h->storage == 3 && h->wide) return pick_wide_kernel(symm, plan);
    if (multistart && h->storage == 3) {
        // 88 registers per thread where that keeps as many CTAs resident as 80 do (asked of the runtime)
        kern_t k80 = multistart_kernel(symm, packed, plan, two_opt, 0);
        kern_t k88 = (k80 && plan == 1 && symm == 1 && !getenv("QAPB_NO_REGS88")) ? multistart_kernel(symm, packed, plan, two_opt, 1) : nullptr;
        if (k88 && k88 != k80 && kernel_occupancy((const void *)k88, h) >= kernel_occupancy((const void *)k80, h)) return k88;
        if (k80) return k80;
    }
    return h->storage == 3 ? pick_hybrid_kernel(symm, packed, plan)
                           : pick_kernel(h->acc_bits, h->storage, h->lb_class);
}

// Split of the off-diagonal units of one search between registers (UR per thread) and shared
// memory (US per thread) for the hybrid kernel.  Returns false if the instance does not fit.
static bool try_hybrid_plan(qapb_handle *h, unsigned smem_cap, int ur, int toff, int us, int dsm = 0,
                            unsigned smem_target = 0)
{
    const int nb = h->nb, dw = (nb + 31) / 32;
    if (ur == 0) {
        // one warp per search, the whole state in the warp's slice of shared memory (search_warp.cuh): n <= 32,
        // int32 state with packed selection keys
        if (h->npad > 32 || h->wide || h->acc_bits != 32 || h->delta_bound >= ((1LL << 27) - 1)) return false;
        int wpc = 4;  // warps per CTA: they share nothing but the address table (launch_search takes fewer for small batches)
        if (const char *e = getenv("QAPB_WPC")) wpc = std::min(8, std::max(1, atoi(e)));
        const int lanes = (h->npad <= 16 && !getenv("QAPB_NO_HALFWARP")) ? 16 : 32;  // lanes per search
        h->wk = lanes; h->wpc = wpc;
        h->staged = 0; h->dsm = 0; h->dd = 0; h->ow = 0;
        h->upt = 1; h->toff = 32; h->us = 0; h->exp_in_smem = 1;
        h->threads = 32 * wpc;
        h->lb_class = 0;
        h->smem_bytes = wk_smem_bytes(lanes, wpc);
        return h->smem_bytes <= smem_cap;
    }
    const int dd = dsm == 2;  // diagonal blocks paired in registers: no dedicated warps, toff counts every thread
    if (dd) dsm = 0;
    if (h->wide && (dd || (ur == 2 && !dsm))) return false;  // 64-bit deltas: plans 0 / 1 / 5 only
    if (dd && !(ur == 1 && us == 0 && toff >= h->noff + (nb + 1) / 2)) return false;
    const int threads = (dsm || dd) ? toff : toff + 32 * dw;
    // the instantiated shapes: two register units, or one for 64-bit deltas / two symmetric matrices with packed keys
    const bool ur1_smem = ur == 1 && (h->wide || (h->symmetric && h->delta_bound < ((1LL << 27) - 1)));
    if (dsm && !((ur == 2 || ur1_smem) && us > 0)) return false;
    if (dsm && threads < nb) return false;
    if ((long long)(ur + us) * toff < h->noff) return false;
    if (threads > 1024 || (us > 0 && threads > 512) || (us == 0 && ur == 2 && threads > 608)) return false;
    int exp_in_smem = 1;
    const int ow = dd && threads == 32 && h->npad <= 32;  // the whole search is one warp
    HybLayout L = make_hyb_layout(h->npad, nb, toff, us, 1, 0, 1, dsm, ow);
    // keep the expiry array in shared memory only while it does not cost a resident CTA -- and not at all when
    // the matrices cannot be staged as int16 (entries above 32767: tai*b flows): the publish phase then reads
    // rows of D and F through L1, which is what is left of the 228 KB after the shared-memory carve-out; with
    // the expiries (touched only when a pair is set or expires) in L2, tai150b runs at 434 instead of 376 G evals/s
    if ((L.total > (smem_target ? smem_target : smem_cap) || !h->fits_i16) && us > 0) {
        exp_in_smem = 0;
        L = make_hyb_layout(h->npad, nb, toff, us, 0, 0, 1, dsm);
    }
    if (L.total > smem_cap) return false;
    if (threads < h->n) return false;  // the publish phase maps one location per thread
    // layout size class 256 goes with shared-memory units -- or with the register-only plan of one search per SM (NP256)
    const bool reg_only_256 = h->npad > 128 && us == 0 && ur == 1 && !dsm && !dd;
    // the instantiated shapes: two symmetric matrices with packed keys, or 64-bit deltas on at most 800 threads
    if (reg_only_256 && !(toff >= h->noff && (h->wide ? toff + 32 * dw <= 800 : (h->symmetric && h->delta_bound < ((1LL << 27) - 1))))) return false;
    if (h->npad > 128 && !reg_only_256 && !(us > 0 && (ur == 2 || (ur == 1 && dsm)))) return false;
    if (h->npad <= 128 && us > 0) return false;
    int staged = 0;
    if (us == 0 && h->fits_i16 && !ow && !reg_only_256 && !getenv("QAPB_NO_STAGE")) {
        // stage while two CTAs per SM still fit
        HybLayout Ls = make_hyb_layout(h->npad, nb, toff, us, exp_in_smem, 1, h->symmetric, dsm);
        if (Ls.total <= std::min(smem_cap, ((dsm || dd) ? 74u : 110u) * 1024u)) { staged = 1; L = Ls; }
    }
    h->staged = staged;
    h->dsm = dsm;
    h->dd = dd;
    h->ow = ow;
    h->wk = 0; h->wpc = 1;
    h->upt = ur; h->toff = toff; h->us = us; h->exp_in_smem = exp_in_smem;
    h->threads = threads;
    h->lb_class = 0;
    h->smem_bytes = L.total;
    return true;
}

static int hybrid_occupancy(const qapb_handle *h) { return kernel_occupancy((const void *)handle_kernel(h), h); }

// Split of the off-diagonal units of one search between registers (UR per thread) and shared
// memory (US per thread) for the hybrid kernel.  Returns false if the instance does not fit.
//   n <= 128: one register unit per thread (80 registers) if two such CTAs fit an SM (n <= 108),
//             else two register units per thread on half the threads (112 registers) if THAT
//             gives two CTAs per SM (n <= 120), else one unit per thread;
//   n <= 256: two register units + shared-memory units per thread, one CTA per SM.
static bool plan_hybrid(qapb_handle *h, unsigned smem_cap)
{
    const int nb = h->nb, noff = h->noff;
    h->storage = 3;  // handle_kernel() dispatches on it
    if (const char *pl = getenv("QAPB_PLAN")) {  // development override: "UR,Toff,US"
        int a, b, c, d = 0, e = 0;
        if (sscanf(pl, "%d,%d,%d,%d,%d", &a, &b, &c, &d, &e) >= 3 && (a == 1 || a == 2) && b % 32 == 0 && b >= 0 && c >= 0)
            return try_hybrid_plan(h, smem_cap, a, b, c, d, (unsigned)e * 1024u);
    }
    // n <= 32: one warp per search (no block barriers, no register-indexed fix-ups)
    if (!getenv("QAPB_NO_WARP") && try_hybrid_plan(h, smem_cap, 0, 32, 0)) return true;
    if (nb > 32 && !h->wide && !getenv("QAPB_NO_REGONLY256")) {
        // n = 129..176, two symmetric matrices, packed keys: the register-only kernel of n <= 128 on ONE search per SM
        // (noff + 64 threads, 72 / 64 registers, no spills, no shared-memory units): tabu 296 x 640 at n = 132 / 144 /
        // 148 / 152 / 156 / 160 / 164 / 176: 736 / 811 / 835 / 842 / 832 / 854 / 873 / 898 G evals/s against 653 / 714 /
        // 736 / 762 / 759 / 684 / 683 / 732 for the shared-memory plans with two searches per SM
        const int tro = (noff + 31) / 32 * 32;
        if (tro + 64 <= 1024 && try_hybrid_plan(h, smem_cap, 1, tro, 0) && hybrid_occupancy(h) >= 1) return true;
    }
    if (nb > 32) {
        // n = 129..256: every warp on off-diagonal units (two in registers + the rest in shared memory per
        // thread), the diagonal blocks in shared memory with the last nb threads (DSM).  Preferred: 256
        // threads with the expiry array in L2 if that keeps TWO searches resident per SM (n <= ~190:
        // 545 / 559 / 616 G evals/s at n = 144 / 160 / 180 against 420 / 376 / 442 for the dedicated-
        // diagonal-warp plan); else all 512 threads on one search (4 units per thread at n = 256
        // instead of 4 or 5 on 14 of 16 warps: 710 -> 750 G evals/s).
        if (!getenv("QAPB_NO_DSM") || h->wide) {
            const bool ur1 = !getenv("QAPB_NO_UR1");
            // 64-bit deltas: ONE register unit per thread keeps the 128-register kernel free of spills (tai150b:
            // 428 -> 484 G evals/s with two searches per SM)
            if (h->wide && ur1 && try_hybrid_plan(h, smem_cap, 1, 256, std::max(1, (noff - 256 + 255) / 256), 1, 113u * 1024u) &&
                hybrid_occupancy(h) >= 2)
                return true;
            // two symmetric matrices with packed keys (the instantiated shape of plan 9), n <= 156: one register unit
            // + at most TWO shared-memory units per thread still leaves room for two searches per SM, and the
            // spill-free kernel beats the two-register-unit one (G evals/s at 296 x 640, n = 132 / 144 / 148 / 156:
            // 600 / 665 / 677 / 584 -> 652 / 713 / 735 / 760).  Three shared-memory units (n >= 157) cost the second
            // resident search (n = 160: 497 against 684), and wider CTAs at 96 registers gain 1-2 % only.
            const int us1s = std::max(1, (noff - 256 + 255) / 256);
            if (!h->wide && ur1 && us1s <= 2 && try_hybrid_plan(h, smem_cap, 1, 256, us1s, 1, 113u * 1024u) &&
                hybrid_occupancy(h) >= 2)
                return true;
            const int us2 = std::max(1, (noff - 2 * 256 + 255) / 256);
            if (try_hybrid_plan(h, smem_cap, 2, 256, us2, 1, 113u * 1024u) && hybrid_occupancy(h) >= 2) return true;
            // one search per SM: one register unit per thread where that shape is instantiated and fits (n = 200:
            // 678 -> 701, n = 256: 846 -> 887 G evals/s), else two
            if (!h->wide && ur1 && try_hybrid_plan(h, smem_cap, 1, 512, std::max(1, (noff - 512 + 511) / 512), 1)) return true;
            const int us1 = std::max(1, (noff - 2 * 512 + 511) / 512);
            if (try_hybrid_plan(h, smem_cap, 2, 512, us1, 1)) return true;
        }
        if (h->wide) return false;  // (no 64-bit-delta instantiation of the dedicated-diagonal-warp plan)
        const int toff = std::min(448, ((noff + 3) / 4 + 31) / 32 * 32);
        const int us = std::max(0, (noff - 2 * toff + toff - 1) / toff);
        return try_hybrid_plan(h, smem_cap, 2, toff, us);
    }
    const int t1 = (noff + 31) / 32 * 32, t2 = ((noff + 1) / 2 + 31) / 32 * 32;
    const int td = (noff + (nb + 1) / 2 + 31) / 32 * 32;
    // paired diagonal blocks (three searches per SM at n = 100) are a candidate plan, not the default: the
    // warp that carries them runs an off-diagonal pass AND two diagonal passes, and the other warps wait
    // for it at barrier 1 (580 against 800 G evals/s at n = 100)
    const char *dd_env = getenv("QAPB_DD");
    if (h->wide) return try_hybrid_plan(h, smem_cap, 1, t1, 0);  // 64-bit deltas: the one-register-unit plan only
    if (dd_env && dd_env[0] == '1' && try_hybrid_plan(h, smem_cap, 1, td, 0, 2)) return true;
    // n <= 32: the paired-diagonal plan is ONE warp per search (no block barriers, 32 searches per SM).  A
    // candidate, not the default: it wins only on large batches (393 against 337 G evals/s at 4736 starts of
    // n = 30) and loses on the BASELINE configurations (271 against 318 G at 1776 starts; a single start takes
    // 2.1 us per iteration against 1.2)
    const char *ow_env = getenv("QAPB_OW");
    if (td == 32 && h->npad <= 32 && ow_env && ow_env[0] == '1' && try_hybrid_plan(h, smem_cap, 1, td, 0, 2)) return true;
    if (!try_hybrid_plan(h, smem_cap, 1, t1, 0)) return false;
    if (hybrid_occupancy(h) >= 2 || t2 < 32) return true;
    const qapb_handle one = *h;
    if (try_hybrid_plan(h, smem_cap, 2, t2, 0) && hybrid_occupancy(h) >= 2) return true;
    *h = one;
    return true;
}

// Candidate hybrid plans of an instance: {ur, toff, us, dsm} rows, the default choice first.
static std::vector<std::array<int, 4>> hybrid_candidates(const qapb_handle *h)
{
    std::vector<std::array<int, 4>> out;
    const int nb = h->nb, noff = h->noff;
    auto add = [&](int ur, int toff, int us, int dsm) {
        if (toff < 32 && !(toff == 0 && noff == 0)) return;
        for (const auto &c : out)
            if (c[0] == ur && c[1] == toff && c[2] == us && c[3] == dsm) return;
        out.push_back({ur, toff, us, dsm});
    };
    if (h->npad <= 32 && !h->wide && h->acc_bits == 32 && h->delta_bound < ((1LL << 27) - 1)) out.push_back({0, 32, 0, 0});
    if (nb > 32) {
        for (int t : {256, 384, 512}) add(2, t, std::max(1, (noff - 2 * t + t - 1) / t), 1);
        for (int t : {256, 512}) add(1, t, std::max(1, (noff - t + t - 1) / t), 1);  // (kept if the shape is instantiated for the instance)
        if ((noff + 31) / 32 * 32 + 64 <= 1024) add(1, (noff + 31) / 32 * 32, 0, 0);  // register-only, one search per SM (likewise)
        const int toff = std::min(448, ((noff + 3) / 4 + 31) / 32 * 32);
        if (!h->wide) add(2, toff, std::max(0, (noff - 2 * toff + toff - 1) / toff), 0);
    } else {
        if (!h->wide) add(1, (noff + (nb + 1) / 2 + 31) / 32 * 32, 0, 2);
        add(1, (noff + 31) / 32 * 32, 0, 0);
        if (!h->wide) add(2, ((noff + 1) / 2 + 31) / 32 * 32, 0, 0);
    }
    return out;
}

static unsigned device_smem_cap(int device) { return (unsigned)g_attr_smem(device); }

extern "C" int qapb_version(void) { return 1; }
extern "C" const char *qapb_last_error(void) { return g_err.c_str(); }
extern "C" int qapb_device_count(int *count)
{
    if (!count) return fail(QAPB_ERR_INVALID, "count is NULL");
    CU(cudaGetDeviceCount(count));
    return QAPB_OK;
}

// ---- process-wide device block cache --------------------------------------------------
// cudaMalloc/cudaFree cost far more than a whole search launch on small instances, so
// blocks released by qapb_destroy are kept (per device, bounded) and handed out again.
namespace {
struct Block { void *p; size_t bytes; int device; };
std::mutex g_pool_mu;
std::vector<Block> g_pool;
size_t g_pool_bytes = 0;
const size_t POOL_MAX_BYTES = (size_t)4 << 30;
const size_t POOL_MAX_BLOCKS = 64;

void *pool_alloc(int device, size_t need, size_t *got)
{
    need = (need + 65535) / 65536 * 65536;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        int best = -1;
        for (int k = 0; k < (int)g_pool.size(); ++k)
            if (g_pool[k].device == device && g_pool[k].bytes >= need && g_pool[k].bytes <= 2 * need + 65536 &&
                (best < 0 || g_pool[k].bytes < g_pool[best].bytes))
                best = k;
        if (best >= 0) {
            Block b = g_pool[best];
            g_pool.erase(g_pool.begin() + best);
            g_pool_bytes -= b.bytes;
            *got = b.bytes;
            return b.p;
        }
    }
    void *p = nullptr;
    if (cudaMalloc(&p, need) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    *got = need;
    return p;
}

void pool_free(int device, void *p, size_t bytes)
{
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back({p, bytes, device});
    g_pool_bytes += bytes;
    while (g_pool.size() > POOL_MAX_BLOCKS || g_pool_bytes > POOL_MAX_BYTES) {
        Block b = g_pool.front();
        g_pool.erase(g_pool.begin());
        g_pool_bytes -= b.bytes;
        cudaSetDevice(b.device);
        cudaFree(b.p);
    }
}

// pinned host staging buffer for instance uploads (one copy per qapb_create)
std::mutex g_stage_mu;
void *g_stage = nullptr;
size_t g_stage_bytes = 0;

struct DevAttr { int valid = 0, sm_count = 0, smem_optin = 0; };
DevAttr g_attr[64];
}  // namespace
int g_attr_smem(int device) { return g_attr[device & 63].smem_optin; }

// Opt-in dynamic shared memory of a kernel instantiation: several handles (and host threads) share one
// instantiation, so the attribute only ever grows -- set to the maximum requested so far, under a mutex.
static cudaError_t ensure_smem_optin(const void *kern, int device, unsigned bytes)
{
    struct Key { const void *k; int device; unsigned bytes; };
    static std::mutex mu;
    static std::vector<Key> seen;
    std::lock_guard<std::mutex> lk(mu);
    for (Key &e : seen)
        if (e.k == kern && e.device == device) {
            if (e.bytes >= bytes) return cudaSuccess;
            cudaError_t rc = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
            if (rc == cudaSuccess) e.bytes = bytes;
            return rc;
        }
    cudaError_t rc = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (rc == cudaSuccess) seen.push_back({kern, device, bytes});
    return rc;
}

static int ensure_ws(qapb_handle *h, size_t bytes)
{
    if (bytes <= h->ws_bytes) return QAPB_OK;
    // launches of this handle that are still in flight write the old workspace: wait before recycling it
    if (h->have_timing) CU(cudaEventSynchronize(h->ev1));
    pool_free(h->device, h->ws, h->ws_bytes);
    h->ws = nullptr;
    h->ws_bytes = 0;
    h->steps_total_off = (size_t)-1;
    size_t want = bytes + bytes / 4 + 4096, got = 0;
    h->ws = pool_alloc(h->device, want, &got);
    if (!h->ws) return fail(QAPB_ERR_NOMEM, "workspace allocation of " + std::to_string(want) + " bytes failed");
    h->ws_bytes = got;
    return QAPB_OK;
}

// Upper bound on |M[a][b]| and |h[a]| over all permutations: rearrangement inequality on sorted
// absolute rows/columns, plus the direct and diagonal terms.
//   level 0: 2 n max|D| max|F|                                   O(n^2)
//   level 1: sorted row/column of D against the elementwise maximum ("envelope") of the
//            sorted rows/columns of F                            O(n^2 log n)
//   level 2: sorted row/column of D against every sorted row/column of F      O(n^3)
static double placement_bound(int n, const std::vector<long long> &F0, const std::vector<long long> &D0,
                              const std::vector<long long> &fd, const std::vector<long long> &dd, int level)
{
    long long maxF = 0, maxD = 0, maxfd = 0, maxdd = 0;
    for (long long v : F0) maxF = std::max(maxF, std::llabs(v));
    for (long long v : D0) maxD = std::max(maxD, std::llabs(v));
    for (long long v : fd) maxfd = std::max(maxfd, std::llabs(v));
    for (long long v : dd) maxdd = std::max(maxdd, std::llabs(v));
    double extra = 2.0 * (double)maxD * (double)maxF + (double)maxfd * (double)maxdd;
    if (level == 0) return 2.0 * n * (double)maxD * (double)maxF + extra;
    std::vector<std::vector<double>> dr(n), dc(n), fr(n), fc(n);
    for (int a = 0; a < n; ++a) {
        dr[a].resize(n); dc[a].resize(n); fr[a].resize(n); fc[a].resize(n);
        for (int k = 0; k < n; ++k) {
            dr[a][k] = (double)std::llabs(D0[(size_t)a * n + k]);
            dc[a][k] = (double)std::llabs(D0[(size_t)k * n + a]);
            fr[a][k] = (double)std::llabs(F0[(size_t)a * n + k]);
            fc[a][k] = (double)std::llabs(F0[(size_t)k * n + a]);
        }
        std::sort(dr[a].begin(), dr[a].end(), std::greater<double>());
        std::sort(dc[a].begin(), dc[a].end(), std::greater<double>());
        std::sort(fr[a].begin(), fr[a].end(), std::greater<double>());
        std::sort(fc[a].begin(), fc[a].end(), std::greater<double>());
    }
    double best = 0;
    if (level == 1) {
        std::vector<double> er(n, 0.0), ec(n, 0.0);
        for (int u = 0; u < n; ++u)
            for (int k = 0; k < n; ++k) { er[k] = std::max(er[k], fr[u][k]); ec[k] = std::max(ec[k], fc[u][k]); }
        for (int a = 0; a < n; ++a) {
            double s = 0;
            for (int k = 0; k < n; ++k) s += dr[a][k] * er[k] + dc[a][k] * ec[k];
            best = std::max(best, s);
        }
        return best + extra;
    }
    for (int a = 0; a < n; ++a)
        for (int u = 0; u < n; ++u) {
            double s = 0;
            for (int k = 0; k < n; ++k) s += dr[a][k] * fr[u][k] + dc[a][k] * fc[u][k];
            best = std::max(best, s);
        }
    return best + extra;
}

// Unit table of a handle: entry uid = I | J << 8 for the off-diagonal units (uid < noff), then the nb diagonal
// blocks.  The generic kernel addresses units by formula (locate()), so its table is lexicographic.  The
// hybrid kernel is table-driven, and there the order decides which WARPS touch block row/column R or S of a
// move: the 4n entries on those rows/columns are fixed in divergent regions that a warp executes when any of
// its units touches the block, and in lexicographic order nearly every warp does (a warp spans one or two
// block rows I and all the columns J > I).  Greedy clustering -- grow a vertex set of the complete graph on
// the blocks, taking each time the block with the most unassigned edges into the set -- gives every warp a
// near-clique: n = 100 (25 blocks, 10 warps) 4.4 warps per block instead of ~9.
static void fill_unit_table(const qapb_handle *h, uint16_t *units)
{
    const int nb = h->nb, noff = h->noff;
    int u = 0;
    // Measured (G evals/s, clustered vs lexicographic): n = 100 852 vs 831, n = 160 682 vs 661 -- but n = 64 683
    // vs 718 and n = 256 (one 512-thread search per SM) 786 vs 843: a clique's blocks sit at arbitrary
    // shared-memory banks, where a lexicographic warp reads one broadcast block and consecutive ones, and
    // with few warps (n <= 76) or every warp busy anyway (512 threads) the conflicts cost more than the
    // skipped regions save.  Hence only the two-searches-per-SM plans from 20 blocks up.
    const char *cl_env = getenv("QAPB_CLUSTER");  // development: 0 / 1 overrides the rule
    const bool by_rule = h->nb >= 20 && h->threads <= 384;
    const bool clustered = h->storage == 3 && !getenv("QAPB_NO_CLUSTER") && (cl_env ? cl_env[0] == '1' : by_rule);
    if (!clustered) {
        for (int I = 0; I < nb; ++I)
            for (int J = I + 1; J < nb; ++J) units[u++] = (uint16_t)(I | (J << 8));
    } else {
        // slots of warp w: uid = k * toff + 32 w + lane for every unit slot k of a thread (registers, then
        // shared memory); its capacity = the slots below noff
        const int toff = std::max(32, h->toff), K = std::max(1, h->upt + h->us), W = toff / 32;
        std::vector<char> rem((size_t)nb * nb, 0);
        std::vector<int> deg(nb, nb - 1);
        for (int I = 0; I < nb; ++I)
            for (int J = 0; J < nb; ++J) rem[(size_t)I * nb + J] = I != J;
        for (int q = 0; q < noff; ++q) units[q] = 0xffffu;
        for (int w = 0; w < W; ++w) {
            std::vector<int> slots;
            for (int k = 0; k < K; ++k)
                for (int l = 0; l < 32; ++l)
                    if (k * toff + 32 * w + l < noff) slots.push_back(k * toff + 32 * w + l);
            std::vector<int> S;
            size_t used = 0;
            while (used < slots.size()) {
                int best = -1, binto = -1, bdeg = -1;
                for (int v = 0; v < nb; ++v) {
                    if (deg[v] == 0 || std::find(S.begin(), S.end(), v) != S.end()) continue;
                    int into = 0;
                    for (int x : S) into += rem[(size_t)v * nb + x];
                    if (into > binto || (into == binto && deg[v] > bdeg)) { best = v; binto = into; bdeg = deg[v]; }
                }
                if (best < 0) break;
                for (int x : S) {
                    if (used >= slots.size()) break;
                    if (!rem[(size_t)best * nb + x]) continue;
                    rem[(size_t)best * nb + x] = rem[(size_t)x * nb + best] = 0;
                    --deg[best]; --deg[x];
                    const int I = std::min(best, x), J = std::max(best, x);
                    units[slots[used++]] = (uint16_t)(I | (J << 8));
                }
                S.push_back(best);
            }
        }
        u = noff;
    }
    for (int I = 0; I < nb; ++I) units[u++] = (uint16_t)(I | (I << 8));
}

extern "C" int qapb_create(int n, const int64_t *flow, const int64_t *dist, int device, qapb_handle **out)
{
    if (!out) return fail(QAPB_ERR_INVALID, "out is NULL");
    *out = nullptr;
    if (n < 2) return fail(QAPB_ERR_INVALID, "instance size must be >= 2, got " + std::to_string(n));
    if (!flow || !dist) return fail(QAPB_ERR_INVALID, "matrix pointer is NULL");
    if (n > 1020) return fail(QAPB_ERR_UNSUPPORTED, "n > 1020 is not supported");
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(QAPB_ERR_INVALID, "device " + std::to_string(device) + " out of range (" + std::to_string(ndev) + " devices)");
    CU(cudaSetDevice(device));

    const int nb = (n + 3) / 4, npad = nb * 4;
    std::vector<long long> F0((size_t)n * n), D0((size_t)n * n), fd(n), dd(n);
    bool sym = true, symF = true, symD = true, fits16 = true, nonneg = true;
    long long maxF0 = 0, maxD0 = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            long long f = flow[(size_t)i * n + j], d = dist[(size_t)i * n + j];
            if (std::llabs(f) >= (1LL << 30) || std::llabs(d) >= (1LL << 30))
                return fail(QAPB_ERR_UNSUPPORTED, "matrix entries must satisfy |x| < 2^30");
            if (f < 0 || d < 0) nonneg = false;
            if (i == j) { fd[i] = f; dd[i] = d; f = 0; d = 0; }
            if (std::llabs(f) > 32767 || std::llabs(d) > 32767) fits16 = false;
            F0[(size_t)i * n + j] = f;
            D0[(size_t)i * n + j] = d;
            maxF0 = std::max(maxF0, std::llabs(f));
            maxD0 = std::max(maxD0, std::llabs(d));
            if (i != j && flow[(size_t)i * n + j] != flow[(size_t)j * n + i]) symF = false;
            if (i != j && dist[(size_t)i * n + j] != dist[(size_t)j * n + i]) symD = false;
        }
    sym = symF && symD;

    qapb_handle *h = new qapb_handle();
    h->n = n; h->nb = nb; h->npad = npad; h->device = device; h->symmetric = sym ? 1 : 0;
    // one symmetric matrix is enough for a single-product rank-2 update: D = D^T gives a == c, so
    // a[i] b[j] + c[i] e[j] = a[i] (b[j] + e[j]); F = F^T gives b == e.  The summed vector must fit int32.
    h->sym_mode = sym ? 1 : (symD && maxF0 < (1LL << 29)) ? 2 : (symF && maxD0 < (1LL << 29)) ? 3 : 0;
    h->fits_i16 = fits16 ? 1 : 0;

    // accumulator width: |delta| <= 4 * bound must stay below 2^31-1 for the int32 state
    const double lim32 = 2147483647.0 / 4.0 - 8.0;
    // the cheap envelope bound also decides packed selection keys (|delta| < 2^27); the O(n^3) one
    // is only worth its time when it can still rescue the int32 state
    double bnd = placement_bound(n, F0, D0, fd, dd, 0);
    if (4.0 * bnd >= (double)((1LL << 27) - 1)) bnd = std::min(bnd, placement_bound(n, F0, D0, fd, dd, 1));
    if (bnd >= lim32) bnd = std::min(bnd, placement_bound(n, F0, D0, fd, dd, 2));
    h->acc_bits = bnd < lim32 ? 32 : 64;
    if (bnd >= 9.0e18 / 4.0) {
        delete h;
        return fail(QAPB_ERR_UNSUPPORTED, "delta bound exceeds int64");
    }
    h->delta_bound = (long long)std::min(4.0 * bnd, 9.0e18);

    // units and CTA shape
    h->noff = nb * (nb - 1) / 2;
    h->nunits = h->noff + nb;
    if (device < 64 && !g_attr[device].valid) {
        CU(cudaDeviceGetAttribute(&g_attr[device].sm_count, cudaDevAttrMultiProcessorCount, device));
        CU(cudaDeviceGetAttribute(&g_attr[device].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        g_attr[device].valid = 1;
    }
    h->sm_count = g_attr[device & 63].sm_count;
    const unsigned smem_cap = (unsigned)g_attr[device & 63].smem_optin;
    const int acc_bytes = h->acc_bits / 8;
    // generic kernel: at most 384 threads, several units per thread (measured: two units per
    // thread on 384 threads beat one unit per thread on 768 at n = 150, int64 state)
    int upt = (h->nunits + 383) / 384;
    if (upt < 1) upt = 1;
    int threads = ((h->nunits + upt - 1) / upt + 31) / 32 * 32;
    if (threads < 32) threads = 32;
    if (threads < ((n + 31) / 32) * 32 && ((n + 31) / 32) * 32 <= 384) threads = ((n + 31) / 32) * 32;
    h->upt = upt;
    h->threads = threads;
    h->lb_class = threads <= 384 ? 0 : 1;
    int storage = 0;
    const char *force = getenv("QAPB_FORCE_GENERIC");
    const bool forced_generic = force && force[0] == '1';
    // 64-bit deltas over UNSIGNED 32-bit state (search_hybrid.cuh, WIDE): the bound exceeds int32, but with
    // non-negative entries every M[i][j] and h[i] is a cost in [0, bound] and bound < 2^32 (4.0e9 admitted: the
    // pad constant needs the margin) -- tai*b shapes.  The state, the build kernels and the workspace are then
    // 32-bit, and the instance runs on the register / shared-memory plans instead of the generic kernel.
    if (h->acc_bits == 64 && nonneg && bnd < 4.0e9 && nb <= 64 && !forced_generic && !getenv("QAPB_NO_WIDE")) {
        const qapb_handle saved = *h;
        h->acc_bits = 32;
        h->wide = 1;
        if (plan_hybrid(h, smem_cap)) storage = 3;
        else *h = saved;
    }
    if (storage == 3) {
    } else if (h->acc_bits == 32 && nb <= 64 && !forced_generic && plan_hybrid(h, smem_cap)) {
        storage = 3;
    } else {
        // generic kernel: M in shared memory when it fits, else in an L2-resident workspace, else
        // (n > ~700) the per-unit tabu masks too
        const char *fs = getenv("QAPB_FORCE_STORAGE");  // development: 1 or 2
        storage = -1;
        for (int k = (fs && (fs[0] == '1' || fs[0] == '2')) ? fs[0] - '0' : 0; k < 3; ++k) {
            SmemLayout L = make_layout(npad, h->nunits, threads, upt, acc_bytes, k);
            if (L.total <= smem_cap) { h->smem_bytes = L.total; storage = k; break; }
        }
        if (storage < 0) {
            delete h;
            return fail(QAPB_ERR_UNSUPPORTED, "instance too large for shared-memory vectors");
        }
    }
    h->storage = storage;
    if (storage == 3 && h->wide && h->npad > 128 && !h->dd && !getenv("QAPB_NO_AUTOPLAN")) {
        qapb_handle probe = *h;
        const int tro = (h->noff + 31) / 32 * 32;
        if (h->us > 0 && try_hybrid_plan(&probe, smem_cap, 1, tro, 0, 0) && hybrid_occupancy(&probe) >= 1) {
            h->have_alt = 1;
            h->def_plan[0] = h->upt; h->def_plan[1] = h->toff; h->def_plan[2] = h->us; h->def_plan[3] = h->dsm;
            h->alt_plan[0] = 1; h->alt_plan[1] = tro; h->alt_plan[2] = 0; h->alt_plan[3] = 0;
        }
    }

    // device copies: one arena, filled in a pinned staging buffer and uploaded with one copy
    const size_t mb = (size_t)npad * npad * sizeof(int32_t), vb = (size_t)npad * sizeof(int32_t);
    const size_t ub = ((size_t)h->nunits * sizeof(uint16_t) + 15) / 16 * 16;
    const size_t total = 4 * mb + 2 * vb + ub;
    cudaError_t e = cudaSuccess;
    h->arena = pool_alloc(device, total, &h->arena_bytes);
    if (!h->arena) {
        delete h;
        return fail(QAPB_ERR_NOMEM, "instance allocation of " + std::to_string(total) + " bytes failed");
    }
    {
        std::lock_guard<std::mutex> lk(g_stage_mu);
        if (g_stage_bytes < total) {
            if (g_stage) cudaFreeHost(g_stage);
            g_stage = nullptr;
            g_stage_bytes = 0;
            e = cudaHostAlloc(&g_stage, total + total / 2, cudaHostAllocDefault);
            if (e == cudaSuccess) g_stage_bytes = total + total / 2;
        }
        if (e == cudaSuccess) {
            memset(g_stage, 0, total);
            int32_t *pF = (int32_t *)g_stage, *pFT = pF + (size_t)npad * npad, *pD = pFT + (size_t)npad * npad,
                    *pDT = pD + (size_t)npad * npad, *pfd = pDT + (size_t)npad * npad, *pdd = pfd + npad;
            uint16_t *units = (uint16_t *)(pdd + npad);
            for (int i = 0; i < n; ++i) {
                pfd[i] = (int32_t)fd[i];
                pdd[i] = (int32_t)dd[i];
                for (int j = 0; j < n; ++j) {
                    const int32_t f = (int32_t)F0[(size_t)i * n + j], d = (int32_t)D0[(size_t)i * n + j];
                    pF[(size_t)i * npad + j] = f;
                    pFT[(size_t)j * npad + i] = f;
                    pD[(size_t)i * npad + j] = d;
                    pDT[(size_t)j * npad + i] = d;
                }
            }
            fill_unit_table(h, units);
            e = cudaMemcpy(h->arena, g_stage, total, cudaMemcpyHostToDevice);
        }
    }
    h->dF = (int32_t *)h->arena;
    h->dFT = h->dF + (size_t)npad * npad;
    h->dD = h->dFT + (size_t)npad * npad;
    h->dDT = h->dD + (size_t)npad * npad;
    h->dfd = h->dDT + (size_t)npad * npad;
    h->ddd = h->dfd + npad;
    h->dunit = (uint16_t *)(h->ddd + npad);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev1);
    kern_t kern = handle_kernel(h);
    if (e == cudaSuccess) e = ensure_smem_optin((const void *)kern, device, h->smem_bytes);
    if (e != cudaSuccess) {
        std::string msg = std::string("instance upload failed: ") + cudaGetErrorString(e);
        qapb_destroy(h);
        return fail(QAPB_ERR_CUDA, msg);
    }
    *out = h;
    return QAPB_OK;
}

extern "C" int qapb_destroy(qapb_handle *h)
{
    if (!h) return QAPB_OK;
    cudaSetDevice(h->device);
    // pending work on this handle's buffers must finish before another handle may reuse them
    if (h->have_timing) cudaEventSynchronize(h->ev1);
    pool_free(h->device, h->arena, h->arena_bytes);
    pool_free(h->device, h->ws, h->ws_bytes);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    delete h;
    return QAPB_OK;
}

extern "C" int qapb_get_info(const qapb_handle *h, qapb_info *info)
{
    if (!h || !info) return fail(QAPB_ERR_INVALID, "NULL argument");
    if (h->ctas_per_sm == 0) {
        qapb_handle *hm = const_cast<qapb_handle *>(h);
        cudaSetDevice(h->device);
        ensure_smem_optin((const void *)handle_kernel(h), h->device, h->smem_bytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hm->ctas_per_sm, (const void *)handle_kernel(h), h->threads, h->smem_bytes);
    }
    info->n = h->n; info->device = h->device; info->acc_bits = h->wide ? 64 : h->acc_bits; info->symmetric = h->symmetric;
    info->threads = h->threads; info->units_per_thread = h->upt; info->storage = h->wk ? 4 : h->storage;
    info->smem_bytes = (int32_t)h->smem_bytes; info->ctas_per_sm = h->ctas_per_sm; info->sm_count = h->sm_count;
    info->delta_bound = h->delta_bound;
    return QAPB_OK;
}

// development hook (not in the public header): phase-cycle counters of CTA 0 of the next launches
static long long *g_dbg = nullptr;
extern "C" int qapb_debug_phase_cycles(long long *out18)
{
    if (!g_dbg) { if (cudaMalloc(&g_dbg, 18 * sizeof(long long)) != cudaSuccess) return QAPB_ERR_NOMEM; cudaMemset(g_dbg, 0, 18 * sizeof(long long)); return QAPB_OK; }
    cudaDeviceSynchronize();
    cudaMemcpy(out18, g_dbg, 18 * sizeof(long long), cudaMemcpyDeviceToHost);
    return QAPB_OK;
}

// test hook (not declared in the public header): force the sequential RNG path
extern "C" int qapb_debug_force_seq_rng(qapb_handle *h, int on)
{
    if (!h) return fail(QAPB_ERR_INVALID, "NULL handle");
    h->force_seq_rng = on;
    return QAPB_OK;
}

static void base_params(const qapb_handle *h, SearchParams &P)
{
    memset(&P, 0, sizeof(P));
    P.n = h->n; P.nb = h->nb; P.npad = h->npad; P.nunits = h->nunits; P.noff = h->noff; P.upt = h->upt;
    P.symmetric = h->sym_mode;  // 0 none, 1 both, 2 distance only, 3 flow only
    P.force_seq_rng = h->force_seq_rng;
    P.one = 1;
    P.sixteen = 16;
    P.F = h->dF; P.FT = h->dFT; P.D = h->dD; P.DT = h->dDT; P.fd = h->dfd; P.dd = h->ddd;
    P.unit_ij = h->dunit;
    P.dbg = g_dbg;
}

// Workspace of one launch: [caller head | M (storage 1) | tabu expiries | start permutations |
// stream states | initial h | initial M], every block 256-byte aligned.
struct WsPlan {
    size_t offM, offT, offPerm, offState, offInitH, offInitM, total;
    size_t m_elems, x_elems;
};
static WsPlan plan_ws(const qapb_handle *h, int batch, size_t head)
{
    auto up = [](size_t v) { return (v + 255) / 256 * 256; };
    const size_t acc_bytes = h->acc_bits / 8, np = (size_t)h->npad;
    WsPlan w;
    w.m_elems = (size_t)h->upt * 8 * h->threads * 4;
    w.x_elems = (size_t)h->nunits * 16 + (h->storage == 2 ? (size_t)2 * h->upt * h->threads : 0);
    size_t o = up(head);
    w.offM = o;
    if (h->storage == 1 || h->storage == 2) o += up(w.m_elems * acc_bytes * batch);
    w.offT = o;
    if (h->storage != 3 || !h->exp_in_smem) o += up(w.x_elems * sizeof(int32_t) * batch);
    w.offPerm = o;  o += up(np * 4 * batch);
    w.offState = o; o += up((size_t)8 * batch);
    w.offInitH = o; o += up(np * acc_bytes * batch);
    w.offInitM = o; o += up(np * np * acc_bytes * batch);
    w.total = o;
    return w;
}

// qap_start_kernel + qap_build_m_kernel for `batch` permutations (caller-provided or device-drawn)
static int launch_build(qapb_handle *h, const WsPlan &w, int batch, int rng, int force_seq, unsigned long long master_seed,
                        unsigned long long first_index, const unsigned long long *seeds, const int64_t *perms,
                        cudaStream_t st, BuildParams &BP, StartParams &SP, int64_t *emit_deltas = nullptr,
                        int *emitted = nullptr)
{
    if (emitted) *emitted = 0;
    const size_t np = (size_t)h->npad;
    SP.n = h->n; SP.npad = h->npad; SP.rng = rng; SP.force_seq_rng = force_seq;
    SP.master_seed = master_seed; SP.first_index = first_index; SP.seeds = seeds; SP.perms = perms;
    SP.perm32 = (int32_t *)((char *)h->ws + w.offPerm);
    SP.state = (unsigned long long *)((char *)h->ws + w.offState);
    qap_start_kernel<<<batch, 128, 2 * np * sizeof(int32_t), st>>>(SP);
    CU(cudaGetLastError());
    BP.n = h->n; BP.npad = h->npad; BP.symmetric = h->symmetric;
    BP.F = h->dF; BP.FT = h->dFT; BP.D = h->dD; BP.DT = h->dDT; BP.fd = h->dfd; BP.dd = h->ddd;
    BP.perm32 = SP.perm32;
    BP.M = (char *)h->ws + w.offInitM;
    BP.h = (char *)h->ws + w.offInitH;
    if (h->npad <= 128 && !getenv("QAPB_BUILD_TILED")) {
        // one CTA per permutation: D^T and the gathered F staged once, 8 x 4 register tiles over all k
        const int cgs = h->npad / 4, rgs = (h->npad + 7) / 8;
        const unsigned nt = (unsigned)((cgs * rgs + 31) / 32 * 32);
        const size_t acc = h->acc_bits / 8;
        const size_t dyn_build = (2 * (np * np + 8) + np) * sizeof(int32_t);
        const size_t dyn = emit_deltas ? std::max(dyn_build, (np * (np + 1) + np) * acc + 16) : dyn_build;
#define QAPB_WHOLE2(A, E, T, B)                                                                                  \
    do {                                                                                                         \
        const void *kf = (const void *)qap_build_m_whole_kernel<A, E, T, B>;                                     \
        CU(ensure_smem_optin(kf, h->device, (unsigned)dyn));                                                     \
        CU(cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared)); \
        qap_build_m_whole_kernel<A, E, T, B><<<batch, nt, dyn, st>>>(BP, emit_deltas);                           \
    } while (0)
#define QAPB_WHOLE(A, E)                                                                                         \
    do {                                                                                                         \
        if (nt <= 352 && sizeof(A) == 4) QAPB_WHOLE2(A, E, 352, 2); else QAPB_WHOLE2(A, E, 544, 1);              \
    } while (0)
        if (h->acc_bits == 64) { if (emit_deltas) QAPB_WHOLE(int64_t, true); else QAPB_WHOLE(int64_t, false); }
        else { if (emit_deltas) QAPB_WHOLE(int32_t, true); else QAPB_WHOLE(int32_t, false); }
#undef QAPB_WHOLE
#undef QAPB_WHOLE2
        CU(cudaGetLastError());
        if (emitted) *emitted = emit_deltas != nullptr;  // the deltas have been written: no emission kernel needed
        return QAPB_OK;
    }
    const int bt = build_tile(h->npad), tiles = (h->npad + bt - 1) / bt;
    const unsigned grid = (unsigned)(tiles * tiles) * (unsigned)batch;
    const unsigned nt = (unsigned)(((bt / 4) * (bt / 4) + 31) / 32 * 32);
    const size_t dyn = np * sizeof(int32_t);
#define QAPB_BUILD(A, B) qap_build_m_kernel<A, B><<<grid, nt, dyn, st>>>(BP)
    if (h->acc_bits == 64) { if (bt == 64) QAPB_BUILD(int64_t, 64); else if (bt == 52) QAPB_BUILD(int64_t, 52); else QAPB_BUILD(int64_t, 32); }
    else { if (bt == 64) QAPB_BUILD(int32_t, 64); else if (bt == 52) QAPB_BUILD(int32_t, 52); else QAPB_BUILD(int32_t, 32); }
#undef QAPB_BUILD
    CU(cudaGetLastError());
    return QAPB_OK;
}

// Launch start + build + search kernels for `batch` starts.  `extra_ws` bytes are reserved at
// the start of the workspace for the caller (multistart keeps best perms there).
static int launch_search(qapb_handle *h, SearchParams &P, int batch, size_t extra_ws, cudaStream_t st, bool first_wave = true)
{
    const WsPlan w = plan_ws(h, batch, extra_ws);
    int rc = ensure_ws(h, w.total);
    if (rc) return rc;
    P.gM = (char *)h->ws + w.offM;
    P.gT = (char *)h->ws + w.offT;
    P.gM_stride = w.m_elems;
    P.gT_stride = w.x_elems;
    const bool records = P.tr_i || P.cells;
    kern_t kern = handle_kernel(h, P.rng && !records, P.mode == MODE_TWO_OPT);
    if (h->storage == 3) {
        P.hlay = make_hyb_layout(h->npad, h->nb, h->toff, h->us, h->exp_in_smem, h->staged, h->symmetric, h->dsm, h->ow);
        P.staged = h->staged; P.dsm = h->dsm;
        P.toff = h->toff; P.us = h->us; P.exp_in_smem = h->exp_in_smem;
    } else {
        P.lay = make_layout(h->npad, h->nunits, h->threads, h->upt, h->acc_bits / 8, h->storage);
        P.inv_t = (unsigned)(((1ULL << 32) + (unsigned)h->threads - 1) / (unsigned)h->threads);
    }
    // several handles share one kernel instantiation: its opt-in size is the maximum requested so far
    CU(ensure_smem_optin((const void *)kern, h->device, h->smem_bytes));
    if (first_wave) CU(cudaEventRecord(h->ev0, st));
    // start permutations (+ stream state), then M and h as one batched tiled integer product
    BuildParams BP;
    StartParams SP;
    if (!h->wk) {  // (the warp kernel draws its start and builds its placement matrix itself)
        rc = launch_build(h, w, batch, P.rng, P.force_seq_rng, P.master_seed, P.first_index, P.seeds, P.perms, st, BP, SP);
        if (rc) return rc;
        P.perm32 = SP.perm32; P.start_state = SP.state; P.initM = BP.M; P.initH = BP.h;
    }
    P.batch = batch;
    if (h->wk) {
        // searches share nothing: pack as many warps into a CTA as still leaves every SM a CTA
        const int per_warp = 32 / h->wk;
        int wpc = h->wpc;
        while (wpc > 1 && (batch + wpc * per_warp - 1) / (wpc * per_warp) < 2 * h->sm_count) wpc >>= 1;
        const int per_cta = wpc * per_warp;
        kern<<<(batch + per_cta - 1) / per_cta, 32 * wpc, wk_smem_bytes(h->wk, wpc), st>>>(P);
    } else {
        kern<<<batch, h->threads, h->smem_bytes, st>>>(P);
    }
    CU(cudaGetLastError());
    CU(cudaEventRecord(h->ev1, st));
    h->have_timing = 1;
    return QAPB_OK;
}

static int check_common(qapb_handle *h, int batch)
{
    if (!h) return fail(QAPB_ERR_INVALID, "NULL handle");
    if (batch < 1) return fail(QAPB_ERR_INVALID, "batch must be >= 1, got " + std::to_string(batch));
    CU(cudaSetDevice(h->device));
    return QAPB_OK;
}

extern "C" int qapb_full_cost(qapb_handle *h, const int64_t *perms, int batch, int64_t *costs, void *stream)
{
    int rc = check_common(h, batch);
    if (rc) return rc;
    if (!perms || !costs) return fail(QAPB_ERR_INVALID, "NULL buffer");
    qap_full_cost_kernel<<<batch, 256, h->npad * sizeof(int32_t), (cudaStream_t)stream>>>(
        h->n, h->npad, h->dF, h->dD, h->dfd, h->ddd, perms, costs);
    CU(cudaGetLastError());
    CU(cudaEventRecord(h->ev1, (cudaStream_t)stream));  // qapb_destroy waits for it before recycling the arena
    if (!h->have_timing) { CU(cudaEventRecord(h->ev0, (cudaStream_t)stream)); h->have_timing = 1; }
    return QAPB_OK;
}

extern "C" int qapb_all_deltas(qapb_handle *h, const int64_t *perms, int batch, int64_t *deltas, void *stream)
{
    int rc = check_common(h, batch);
    if (rc) return rc;
    if (!perms || !deltas) return fail(QAPB_ERR_INVALID, "NULL buffer");
    // the full evaluator as a tiled contraction (qap_build_m_kernel) + emission
    cudaStream_t st = (cudaStream_t)stream;
    // (a WIDE handle keeps 32-bit state, but the deltas themselves need 64 bits: build M in int64 here)
    qapb_handle hv = *h;
    if (h->wide) { hv.acc_bits = 64; hv.wide = 0; }
    const WsPlan w = plan_ws(&hv, batch, 0);
    rc = ensure_ws(h, w.total);
    if (rc) return rc;
    hv.ws = h->ws; hv.ws_bytes = h->ws_bytes;
    CU(cudaEventRecord(h->ev0, st));
    BuildParams BP;
    StartParams SP;
    int emitted = 0;
    rc = launch_build(&hv, w, batch, 0, 0, 0, 0, nullptr, perms, st, BP, SP, deltas, &emitted);
    if (rc) return rc;
    if (!emitted) {  // tiled build (n > 128): M and h are in the workspace, emit from there
        const dim3 grid(batch, std::min(h->n - 1, 64));
        if (hv.acc_bits == 64) qap_emit_deltas_kernel<int64_t><<<grid, 256, 0, st>>>(h->n, h->npad, BP.M, BP.h, deltas);
        else qap_emit_deltas_kernel<int32_t><<<grid, 256, 0, st>>>(h->n, h->npad, BP.M, BP.h, deltas);
        CU(cudaGetLastError());
    }
    CU(cudaEventRecord(h->ev1, st));
    h->have_timing = 1;
    return QAPB_OK;
}

extern "C" int qapb_two_opt(qapb_handle *h, const int64_t *perms, int batch, int iterations, int64_t *best,
                            int64_t *best_cost, int64_t *cur, int64_t *cur_cost, int64_t *move_i,
                            int64_t *move_j, int64_t *move_delta, void *stream)
{
    int rc = check_common(h, batch);
    if (rc) return rc;
    if (iterations < 1) return fail(QAPB_ERR_INVALID, "iterations must be >= 1, got " + std::to_string(iterations));
    if (!perms || !best || !best_cost || !cur || !cur_cost) return fail(QAPB_ERR_INVALID, "NULL buffer");
    if ((move_i || move_j || move_delta) && !(move_i && move_j && move_delta))
        return fail(QAPB_ERR_INVALID, "move_i/move_j/move_delta must be given together");
    SearchParams P;
    base_params(h, P);
    P.mode = MODE_TWO_OPT;
    P.iterations = iterations;
    P.perms = perms;
    P.best = best; P.best_cost = best_cost; P.cur = cur; P.cur_cost = cur_cost;
    P.tr_i = move_i; P.tr_j = move_j; P.tr_d = move_delta;
    return launch_search(h, P, batch, 0, (cudaStream_t)stream);
}

extern "C" int qapb_tabu(qapb_handle *h, const int64_t *perms, int batch, int iterations, const int64_t *tenures,
                         int64_t *best, int64_t *best_cost, int64_t *cur, int64_t *cur_cost, int64_t *cells,
                         int64_t *stopped_early, int64_t *steps_done, int64_t *trail_i, int64_t *trail_j,
                         int64_t *trail_delta, int64_t *trail_tabu, void *stream)
{
    int rc = check_common(h, batch);
    if (rc) return rc;
    if (iterations < 1) return fail(QAPB_ERR_INVALID, "iterations must be >= 1, got " + std::to_string(iterations));
    if (!perms || !tenures || !best || !best_cost || !cur || !cur_cost) return fail(QAPB_ERR_INVALID, "NULL buffer");
    if ((trail_i || trail_j || trail_delta || trail_tabu) && !(trail_i && trail_j && trail_delta && trail_tabu))
        return fail(QAPB_ERR_INVALID, "trail arrays must be given together");
    SearchParams P;
    base_params(h, P);
    P.mode = MODE_TABU;
    P.iterations = iterations;
    P.perms = perms;
    P.tenures = tenures;
    P.best = best; P.best_cost = best_cost; P.cur = cur; P.cur_cost = cur_cost;
    P.cells = cells; P.stopped = stopped_early; P.steps = steps_done;
    P.tr_i = trail_i; P.tr_j = trail_j; P.tr_d = trail_delta; P.tr_tabu = trail_tabu;
    return launch_search(h, P, batch, 0, (cudaStream_t)stream);
}

static int apply_plan(qapb_handle *h, int reg_units, int unit_threads, int smem_units, int diag_in_smem);

extern "C" int qapb_multistart(qapb_handle *h, int algo, uint64_t master_seed, uint64_t first_index, int count,
                               int iterations, int64_t ten_low, int64_t ten_high, int64_t *per_start_costs,
                               int64_t *best_key, int64_t *best_perm, void *stream)
{
    int rc = check_common(h, count);
    if (rc) return rc;
    if (algo != QAPB_ALGO_2OPT && algo != QAPB_ALGO_TABU) return fail(QAPB_ERR_INVALID, "unknown algorithm " + std::to_string(algo));
    if (iterations < 1) return fail(QAPB_ERR_INVALID, "iterations must be >= 1, got " + std::to_string(iterations));
    if (algo == QAPB_ALGO_TABU && !(1 <= ten_low && ten_low <= ten_high))
        return fail(QAPB_ERR_INVALID, "invalid tenure interval [" + std::to_string(ten_low) + ", " + std::to_string(ten_high) + "]");
    if (algo == QAPB_ALGO_TABU && (double)iterations + (double)ten_high >= 2147483647.0)
        return fail(QAPB_ERR_UNSUPPORTED, "iterations + tenure must fit int32");
    if (!per_start_costs || !best_key || !best_perm) return fail(QAPB_ERR_INVALID, "NULL buffer");
    if (h->have_alt && !h->user_plan) {
        // at most one search per SM: the register-only plan; more: the default (see qapb_handle::have_alt)
        const int *want = count <= h->sm_count ? h->alt_plan : h->def_plan;
        if (want[0] != h->upt || want[1] != h->toff || want[2] != h->us || want[3] != h->dsm) {
            rc = apply_plan(h, want[0], want[1], want[2], want[3]);
            if (rc) return rc;
        }
    }
    const int n = h->n;
    // workspace head: best perms [count,n], cur perms [count,n], cur costs [count], steps [count], total steps [1]
    const size_t perm_bytes = (size_t)count * n * sizeof(int64_t);
    const size_t head = 2 * perm_bytes + 2 * (size_t)count * sizeof(int64_t) + 16;
    SearchParams P;
    base_params(h, P);
    P.mode = algo == QAPB_ALGO_TABU ? MODE_TABU : MODE_TWO_OPT;
    P.rng = 1;
    P.iterations = iterations;
    P.master_seed = master_seed;
    P.first_index = first_index;
    P.ten_lo = ten_low;
    P.ten_hi = ten_high;
    // The per-start workspace (initial M, permutations, M in L2 for large n) grows with the batch: the reference's
    // default of 6144 starts on a large int64 instance would ask for tens of GB.  The starts are therefore run in
    // waves sized to a memory budget (free memory / 2, at most 8 GiB; QAPB_WAVE_BYTES overrides), each a whole number
    // of resident CTA sets; per-start results land in the caller's arrays at their offsets and one reduction
    // follows.  A batch that fits (every benchmark shape) is a single wave.
    size_t budget = (size_t)8 << 30, free_b = 0, total_b = 0;
    const size_t need = plan_ws(h, count, head).total;
    // (cudaMemGetInfo costs milliseconds: only batches of a GiB and more, that do not fit the workspace the
    // handle already holds, ask)
    if (need > h->ws_bytes && need > ((size_t)1 << 30) && cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
        budget = std::min(budget, (free_b + h->ws_bytes) / 2);
    if (const char *wb = getenv("QAPB_WAVE_BYTES")) budget = (size_t)strtoull(wb, nullptr, 10);
    int wave = count;
    if (need > budget) {
        const size_t per_start = (plan_ws(h, 1024, head).total - plan_ws(h, 0, head).total) / 1024 + 1;
        const size_t room = budget > plan_ws(h, 0, head).total ? budget - plan_ws(h, 0, head).total : 0;
        const int set = std::max(1, h->sm_count * std::max(1, h->ctas_per_sm ? h->ctas_per_sm : 1));
        wave = (int)std::min<size_t>((size_t)count, std::max<size_t>(1, room / per_start));
        if (wave > set) wave -= wave % set;
    }
    // size the whole workspace first so the head pointers stay valid
    rc = ensure_ws(h, plan_ws(h, wave, head).total);
    if (rc) return rc;
    int64_t *w_best = (int64_t *)h->ws;
    int64_t *w_cur = (int64_t *)((char *)h->ws + perm_bytes);
    int64_t *w_curcost = (int64_t *)((char *)h->ws + 2 * perm_bytes);
    int64_t *w_steps = w_curcost + count;
    for (int off = 0; off < count; off += wave) {
        const int cnt = std::min(wave, count - off);
        P.first_index = first_index + (uint64_t)off;
        P.best = w_best + (size_t)off * n; P.best_cost = per_start_costs + off; P.cur = w_cur + (size_t)off * n;
        P.cur_cost = w_curcost + off;
        P.steps = w_steps + off;
        rc = launch_search(h, P, cnt, head, (cudaStream_t)stream, off == 0);
        if (rc) return rc;
    }
    h->steps_total_off = (size_t)((char *)(w_steps + count) - (char *)h->ws);
    qap_pick_best_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(count, n, first_index, per_start_costs, w_best, best_key, best_perm,
                                                               w_steps, w_steps + count);
    CU(cudaGetLastError());
    CU(cudaEventRecord(h->ev1, (cudaStream_t)stream));
    return QAPB_OK;
}

static int check_multistart_args(int algo, int iterations, int64_t ten_low, int64_t ten_high)
{
    if (algo != QAPB_ALGO_2OPT && algo != QAPB_ALGO_TABU) return fail(QAPB_ERR_INVALID, "unknown algorithm " + std::to_string(algo));
    if (iterations < 1) return fail(QAPB_ERR_INVALID, "iterations must be >= 1, got " + std::to_string(iterations));
    if (algo == QAPB_ALGO_TABU && !(1 <= ten_low && ten_low <= ten_high))
        return fail(QAPB_ERR_INVALID, "invalid tenure interval [" + std::to_string(ten_low) + ", " + std::to_string(ten_high) + "]");
    if (algo == QAPB_ALGO_TABU && (double)iterations + (double)ten_high >= 2147483647.0)
        return fail(QAPB_ERR_UNSUPPORTED, "iterations + tenure must fit int32");
    return QAPB_OK;
}

extern "C" int qapb_multistart_seeds(qapb_handle *h, int algo, const uint64_t *seeds, int count, int iterations,
                                     int64_t ten_low, int64_t ten_high, int64_t *per_start_costs, int64_t *best_perms,
                                     void *stream)
{
    int rc = check_common(h, count);
    if (rc) return rc;
    rc = check_multistart_args(algo, iterations, ten_low, ten_high);
    if (rc) return rc;
    if (!seeds || !per_start_costs || !best_perms) return fail(QAPB_ERR_INVALID, "NULL buffer");
    // workspace head: cur perms [count,n], cur costs [count]
    const size_t perm_bytes = (size_t)count * h->n * sizeof(int64_t);
    const size_t head = perm_bytes + (size_t)count * sizeof(int64_t);
    rc = ensure_ws(h, plan_ws(h, count, head).total);
    if (rc) return rc;
    SearchParams P;
    base_params(h, P);
    P.mode = algo == QAPB_ALGO_TABU ? MODE_TABU : MODE_TWO_OPT;
    P.rng = 1;
    P.iterations = iterations;
    P.seeds = (const unsigned long long *)seeds;
    P.ten_lo = ten_low;
    P.ten_hi = ten_high;
    P.best = best_perms; P.best_cost = per_start_costs;
    P.cur = (int64_t *)h->ws; P.cur_cost = (int64_t *)((char *)h->ws + perm_bytes);
    return launch_search(h, P, count, head, (cudaStream_t)stream);
}

extern "C" int qapb_multistart_trace(qapb_handle *h, int algo, const uint64_t *seeds, int count, int iterations,
                                     int64_t ten_low, int64_t ten_high, int64_t *per_start_costs, int64_t *best_perms,
                                     int64_t *steps_done, int64_t *move_i, int64_t *move_j, int64_t *move_delta,
                                     void *stream)
{
    int rc = check_common(h, count);
    if (rc) return rc;
    rc = check_multistart_args(algo, iterations, ten_low, ten_high);
    if (rc) return rc;
    if (!seeds || !per_start_costs || !best_perms || !steps_done || !move_i || !move_j || !move_delta)
        return fail(QAPB_ERR_INVALID, "NULL buffer");
    const size_t perm_bytes = (size_t)count * h->n * sizeof(int64_t);
    const size_t head = perm_bytes + (size_t)count * sizeof(int64_t);
    rc = ensure_ws(h, plan_ws(h, count, head).total);
    if (rc) return rc;
    SearchParams P;
    base_params(h, P);
    P.mode = algo == QAPB_ALGO_TABU ? MODE_TABU : MODE_TWO_OPT;
    P.rng = 1;
    P.iterations = iterations;
    P.seeds = (const unsigned long long *)seeds;
    P.ten_lo = ten_low;
    P.ten_hi = ten_high;
    P.best = best_perms; P.best_cost = per_start_costs;
    P.cur = (int64_t *)h->ws; P.cur_cost = (int64_t *)((char *)h->ws + perm_bytes);
    P.steps = steps_done;
    P.tr_i = move_i; P.tr_j = move_j; P.tr_d = move_delta;  // selects the recording instantiation
    return launch_search(h, P, count, head, (cudaStream_t)stream);
}

extern "C" int qapb_plan_candidates(qapb_handle *h, int32_t *plans, int cap, int *count)
{
    if (!h || !count || (cap > 0 && !plans)) return fail(QAPB_ERR_INVALID, "NULL argument");
    *count = 0;
    if (h->storage != 3) return QAPB_OK;  // generic kernel: one configuration
    qapb_handle probe = *h;               // try each candidate on a copy (no device state is touched)
    for (const auto &c : hybrid_candidates(h)) {
        const unsigned target = (c[3] == 1 && c[1] <= 256) ? 113u * 1024u : 0u;
        if (!try_hybrid_plan(&probe, device_smem_cap(h->device), c[0], c[1], c[2], c[3], target)) continue;
        if (*count < cap)
            for (int q = 0; q < 4; ++q) plans[*count * 4 + q] = c[q];
        ++*count;
    }
    return QAPB_OK;
}

// Re-plan a handle (qapb_set_plan, and the batch-size switch of qapb_multistart).
static int apply_plan(qapb_handle *h, int reg_units, int unit_threads, int smem_units, int diag_in_smem)
{
    CU(cudaSetDevice(h->device));
    if (h->have_timing) CU(cudaEventSynchronize(h->ev1));  // no launch of the old plan in flight
    qapb_handle probe = *h;
    const unsigned target = (diag_in_smem == 1 && unit_threads <= 256) ? 113u * 1024u : 0u;
    if ((reg_units != 0 && reg_units != 1 && reg_units != 2) || unit_threads < 0 || unit_threads % 32 != 0 || smem_units < 0 ||
        !try_hybrid_plan(&probe, device_smem_cap(h->device), reg_units, unit_threads, smem_units, diag_in_smem, target))
        return fail(QAPB_ERR_INVALID, "plan {" + std::to_string(reg_units) + ", " + std::to_string(unit_threads) + ", " +
                                          std::to_string(smem_units) + ", " + std::to_string(diag_in_smem) + "} does not fit this instance");
    probe.ctas_per_sm = 0;  // re-queried by qapb_get_info
    *h = probe;
    std::vector<uint16_t> units(h->nunits);  // the unit order follows the plan
    fill_unit_table(h, units.data());
    CU(cudaMemcpy(h->dunit, units.data(), units.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    return QAPB_OK;
}

extern "C" int qapb_set_plan(qapb_handle *h, int reg_units, int unit_threads, int smem_units, int diag_in_smem)
{
    if (!h) return fail(QAPB_ERR_INVALID, "NULL handle");
    if (h->storage != 3) return fail(QAPB_ERR_UNSUPPORTED, "this instance runs in the generic kernel: no alternative plans");
    const int rc = apply_plan(h, reg_units, unit_threads, smem_units, diag_in_smem);
    if (rc == QAPB_OK) h->user_plan = 1;  // the caller's choice stands: no switching by batch size
    return rc;
}

extern "C" int qapb_last_total_steps(qapb_handle *h, int64_t *steps)
{
    if (!h || !steps) return fail(QAPB_ERR_INVALID, "NULL argument");
    if (h->steps_total_off == (size_t)-1 || !h->ws) return fail(QAPB_ERR_INVALID, "no multistart recorded");
    CU(cudaSetDevice(h->device));
    CU(cudaEventSynchronize(h->ev1));
    CU(cudaMemcpy(steps, (char *)h->ws + h->steps_total_off, sizeof(int64_t), cudaMemcpyDeviceToHost));
    return QAPB_OK;
}

extern "C" int qapb_last_kernel_ms(qapb_handle *h, float *ms)
{
    if (!h || !ms) return fail(QAPB_ERR_INVALID, "NULL argument");
    if (!h->have_timing) return fail(QAPB_ERR_INVALID, "no launch recorded");
    CU(cudaSetDevice(h->device));
    CU(cudaEventSynchronize(h->ev1));
    CU(cudaEventElapsedTime(ms, h->ev0, h->ev1));
    return QAPB_OK;
}

// ------------------------------------------------------------ host variants --
namespace {
struct DevBuf {  // scratch from the block cache; released after the (synchronous) read-back
    void *p = nullptr;
    size_t bytes = 0;
    int device = 0;
    ~DevBuf() { pool_free(device, p, bytes); }
    cudaError_t alloc(size_t want)
    {
        cudaGetDevice(&device);
        p = pool_alloc(device, want ? want : 1, &bytes);
        return p ? cudaSuccess : cudaErrorMemoryAllocation;
    }
    template <typename T> T *as() { return (T *)p; }
};
}  // namespace
#define H2D(dst, src, bytes) CU(cudaMemcpy((dst), (src), (bytes), cudaMemcpyHostToDevice))
#define D2H(dst, src, bytes) CU(cudaMemcpy((dst), (src), (bytes), cudaMemcpyDeviceToHost))

extern "C" int qapb_full_cost_host(qapb_handle *h, const int64_t *perms, int batch, int64_t *costs)
{
    int rc = check_common(h, batch);
    if (rc) return rc;
    if (!perms || !costs) return fail(QAPB_ERR_INVALID, "NULL buffer");
    DevBuf dp, dc;
    const size_t pb = (size_t)batch * h->n * 8;
    CU(dp.alloc(pb)); CU(dc.alloc((size_t)batch * 8));
    H2D(dp.p, perms, pb);
    rc = qapb_full_cost(h, dp.as<int64_t>(), batch, dc.as<int64_t>(), nullptr);
    if (rc) return rc;
    D2H(costs, dc.p, (size_t)batch * 8);
    return QAPB_OK;
}

extern "C" int qapb_all_deltas_host(qapb_handle *h, const int64_t *perms, int batch, int64_t *deltas)
{
    int rc = check_common(h, batch);
    if (rc) return rc;
    if (!perms || !deltas) return fail(QAPB_ERR_INVALID, "NULL buffer");
    DevBuf dp, dd;
    const size_t pb = (size_t)batch * h->n * 8, ob = (size_t)batch * ((size_t)h->n * (h->n - 1) / 2) * 8;
    CU(dp.alloc(pb)); CU(dd.alloc(ob));
    H2D(dp.p, perms, pb);
    rc = qapb_all_deltas(h, dp.as<int64_t>(), batch, dd.as<int64_t>(), nullptr);
    if (rc) return rc;
    D2H(deltas, dd.p, ob);
    return QAPB_OK;
}

extern "C" int qapb_two_opt_host(qapb_handle *h, const int64_t *perms, int batch, int iterations, int64_t *best,
                                 int64_t *best_cost, int64_t *cur, int64_t *cur_cost, int64_t *move_i,
                                 int64_t *move_j, int64_t *move_delta)
{
    int rc = check_common(h, batch);
    if (rc) return rc;
    if (iterations < 1) return fail(QAPB_ERR_INVALID, "iterations must be >= 1, got " + std::to_string(iterations));
    if (!perms || !best || !best_cost || !cur || !cur_cost) return fail(QAPB_ERR_INVALID, "NULL buffer");
    const bool tr = move_i && move_j && move_delta;
    const size_t pb = (size_t)batch * h->n * 8, sb = (size_t)batch * 8, tb = (size_t)batch * iterations * 8;
    DevBuf dp, dbest, dbc, dcur, dcc, dmi, dmj, dmd;
    CU(dp.alloc(pb)); CU(dbest.alloc(pb)); CU(dbc.alloc(sb)); CU(dcur.alloc(pb)); CU(dcc.alloc(sb));
    if (tr) { CU(dmi.alloc(tb)); CU(dmj.alloc(tb)); CU(dmd.alloc(tb)); }
    H2D(dp.p, perms, pb);
    rc = qapb_two_opt(h, dp.as<int64_t>(), batch, iterations, dbest.as<int64_t>(), dbc.as<int64_t>(), dcur.as<int64_t>(),
                      dcc.as<int64_t>(), tr ? dmi.as<int64_t>() : nullptr, tr ? dmj.as<int64_t>() : nullptr,
                      tr ? dmd.as<int64_t>() : nullptr, nullptr);
    if (rc) return rc;
    D2H(best, dbest.p, pb); D2H(best_cost, dbc.p, sb); D2H(cur, dcur.p, pb); D2H(cur_cost, dcc.p, sb);
    if (tr) { D2H(move_i, dmi.p, tb); D2H(move_j, dmj.p, tb); D2H(move_delta, dmd.p, tb); }
    return QAPB_OK;
}

extern "C" int qapb_tabu_host(qapb_handle *h, const int64_t *perms, int batch, int iterations, const int64_t *tenures,
                              int64_t *best, int64_t *best_cost, int64_t *cur, int64_t *cur_cost, int64_t *cells,
                              int64_t *stopped_early, int64_t *steps_done, int64_t *trail_i, int64_t *trail_j,
                              int64_t *trail_delta, int64_t *trail_tabu)
{
    int rc = check_common(h, batch);
    if (rc) return rc;
    if (iterations < 1) return fail(QAPB_ERR_INVALID, "iterations must be >= 1, got " + std::to_string(iterations));
    if (!perms || !tenures || !best || !best_cost || !cur || !cur_cost) return fail(QAPB_ERR_INVALID, "NULL buffer");
    const bool tr = trail_i && trail_j && trail_delta && trail_tabu;
    const int n = h->n;
    // expiry iterations c + tenure are int32 on the device
    for (int b = 0; b < batch; ++b)
        for (int c = 1; c <= iterations; ++c) {
            const int64_t t = tenures[(size_t)b * iterations + (c - 1)];
            if (t > 2147483647LL - c || t < -2147483647LL)
                return fail(QAPB_ERR_UNSUPPORTED, "iteration + tenure must fit int32 (tenure " + std::to_string(t) + ")");
        }
    const size_t pb = (size_t)batch * n * 8, sb = (size_t)batch * 8, tb = (size_t)batch * iterations * 8;
    const size_t cb = (size_t)batch * n * n * 8;
    DevBuf dp, dten, dbest, dbc, dcur, dcc, dcells, dstop, dsteps, dti, dtj, dtd, dtt;
    CU(dp.alloc(pb)); CU(dten.alloc(tb)); CU(dbest.alloc(pb)); CU(dbc.alloc(sb)); CU(dcur.alloc(pb)); CU(dcc.alloc(sb));
    CU(dstop.alloc(sb)); CU(dsteps.alloc(sb));
    if (cells) CU(dcells.alloc(cb));
    if (tr) { CU(dti.alloc(tb)); CU(dtj.alloc(tb)); CU(dtd.alloc(tb)); CU(dtt.alloc(tb)); }
    H2D(dp.p, perms, pb);
    H2D(dten.p, tenures, tb);
    rc = qapb_tabu(h, dp.as<int64_t>(), batch, iterations, dten.as<int64_t>(), dbest.as<int64_t>(), dbc.as<int64_t>(),
                   dcur.as<int64_t>(), dcc.as<int64_t>(), cells ? dcells.as<int64_t>() : nullptr, dstop.as<int64_t>(),
                   dsteps.as<int64_t>(), tr ? dti.as<int64_t>() : nullptr, tr ? dtj.as<int64_t>() : nullptr,
                   tr ? dtd.as<int64_t>() : nullptr, tr ? dtt.as<int64_t>() : nullptr, nullptr);
    if (rc) return rc;
    D2H(best, dbest.p, pb); D2H(best_cost, dbc.p, sb); D2H(cur, dcur.p, pb); D2H(cur_cost, dcc.p, sb);
    if (cells) D2H(cells, dcells.p, cb);
    if (stopped_early) D2H(stopped_early, dstop.p, sb);
    if (steps_done) D2H(steps_done, dsteps.p, sb);
    if (tr) { D2H(trail_i, dti.p, tb); D2H(trail_j, dtj.p, tb); D2H(trail_delta, dtd.p, tb); D2H(trail_tabu, dtt.p, tb); }
    return QAPB_OK;
}

extern "C" int qapb_multistart_host(qapb_handle *h, int algo, uint64_t master_seed, uint64_t first_index, int count,
                                    int iterations, int64_t ten_low, int64_t ten_high, int64_t *per_start_costs,
                                    int64_t *best_key, int64_t *best_perm)
{
    int rc = check_common(h, count);
    if (rc) return rc;
    if (!per_start_costs || !best_key || !best_perm) return fail(QAPB_ERR_INVALID, "NULL buffer");
    // one device block [costs | key | perm], one read-back
    DevBuf out;
    const size_t words = (size_t)count + 2 + (size_t)h->n;
    CU(out.alloc(words * 8));
    int64_t *d = out.as<int64_t>();
    rc = qapb_multistart(h, algo, master_seed, first_index, count, iterations, ten_low, ten_high, d, d + count,
                         d + count + 2, nullptr);
    if (rc) return rc;
    std::vector<int64_t> host(words);
    D2H(host.data(), d, words * 8);
    memcpy(per_start_costs, host.data(), (size_t)count * 8);
    memcpy(best_key, host.data() + count, 16);
    memcpy(best_perm, host.data() + count + 2, (size_t)h->n * 8);
    return QAPB_OK;
}

extern "C" int qapb_multistart_seeds_host(qapb_handle *h, int algo, const uint64_t *seeds, int count, int iterations,
                                          int64_t ten_low, int64_t ten_high, int64_t *per_start_costs,
                                          int64_t *best_perms)
{
    int rc = check_common(h, count);
    if (rc) return rc;
    if (!seeds || !per_start_costs || !best_perms) return fail(QAPB_ERR_INVALID, "NULL buffer");
    const size_t cb = (size_t)count * 8, pb = (size_t)count * h->n * 8;
    DevBuf buf;  // [seeds | costs | perms]
    CU(buf.alloc(2 * cb + pb));
    char *d = buf.as<char>();
    H2D(d, seeds, cb);
    rc = qapb_multistart_seeds(h, algo, (const uint64_t *)d, count, iterations, ten_low, ten_high, (int64_t *)(d + cb),
                               (int64_t *)(d + 2 * cb), nullptr);
    if (rc) return rc;
    D2H(per_start_costs, d + cb, cb);
    D2H(best_perms, d + 2 * cb, pb);
    return QAPB_OK;
}

extern "C" int qapb_multistart_trace_host(qapb_handle *h, int algo, const uint64_t *seeds, int count, int iterations,
                                          int64_t ten_low, int64_t ten_high, int64_t *per_start_costs,
                                          int64_t *best_perms, int64_t *steps_done, int64_t *move_i, int64_t *move_j,
                                          int64_t *move_delta)
{
    int rc = check_common(h, count);
    if (rc) return rc;
    if (iterations < 1) return fail(QAPB_ERR_INVALID, "iterations must be >= 1, got " + std::to_string(iterations));
    if (!seeds || !per_start_costs || !best_perms || !steps_done || !move_i || !move_j || !move_delta)
        return fail(QAPB_ERR_INVALID, "NULL buffer");
    const size_t cb = (size_t)count * 8, pb = (size_t)count * h->n * 8, tb = (size_t)count * iterations * 8;
    DevBuf buf;  // [seeds | costs | steps | perms | move_i | move_j | move_delta]
    CU(buf.alloc(3 * cb + pb + 3 * tb));
    char *d = buf.as<char>();
    H2D(d, seeds, cb);
    CU(cudaMemsetAsync(d + 3 * cb + pb, 0, 3 * tb, nullptr));  // rows past steps_done read as zero
    rc = qapb_multistart_trace(h, algo, (const uint64_t *)d, count, iterations, ten_low, ten_high, (int64_t *)(d + cb),
                               (int64_t *)(d + 3 * cb), (int64_t *)(d + 2 * cb), (int64_t *)(d + 3 * cb + pb),
                               (int64_t *)(d + 3 * cb + pb + tb), (int64_t *)(d + 3 * cb + pb + 2 * tb), nullptr);
    if (rc) return rc;
    D2H(per_start_costs, d + cb, cb);
    D2H(steps_done, d + 2 * cb, cb);
    D2H(best_perms, d + 3 * cb, pb);
    D2H(move_i, d + 3 * cb + pb, tb);
    D2H(move_j, d + 3 * cb + pb + tb, tb);
    D2H(move_delta, d + 3 * cb + pb + 2 * tb, tb);
    return QAPB_OK;
}

extern "C" int qapb_probe_smem_peak(int device, double *bytes_per_sec)
{
    if (!bytes_per_sec) return fail(QAPB_ERR_INVALID, "bad argument");
    CU(cudaSetDevice(device));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    DevBuf sink;
    CU(sink.alloc(4));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    const int iters = 4000, threads = 1024, blocks = prop.multiProcessorCount * 2;
    qap_smem_probe_kernel<<<blocks, threads>>>(100, sink.as<int>());
    CU(cudaDeviceSynchronize());
    CU(cudaEventRecord(e0));
    qap_smem_probe_kernel<<<blocks, threads>>>(iters, sink.as<int>());
    CU(cudaEventRecord(e1));
    CU(cudaEventSynchronize(e1));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *bytes_per_sec = (double)iters * 8.0 * 16.0 * threads * blocks / (ms * 1e-3);
    return QAPB_OK;
}

extern "C" int qapb_probe_int_peak(int device, int kind, double *ops_per_sec)
{
    if (!ops_per_sec || kind < 0 || kind > 4) return fail(QAPB_ERR_INVALID, "bad argument");
    CU(cudaSetDevice(device));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    DevBuf sink;
    CU(sink.alloc(4));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    const int iters = 20000, threads = 1024, blocks = prop.multiProcessorCount * 2;
    auto launch = [&](int it) {
        if (kind == 0) qap_int_probe_kernel<0><<<blocks, threads>>>(it, sink.as<int>(), 3);
        else if (kind == 1) qap_int_probe_kernel<1><<<blocks, threads>>>(it, sink.as<int>(), 3);
        else if (kind == 2) qap_int_probe_kernel<2><<<blocks, threads>>>(it, sink.as<int>(), 3);
        else if (kind == 3) qap_int_probe_kernel<3><<<blocks, threads>>>(it, sink.as<int>(), 3);
        else qap_int_probe_kernel<4><<<blocks, threads>>>(it, sink.as<int>(), 3);
    };
    launch(200);
    CU(cudaDeviceSynchronize());
    CU(cudaEventRecord(e0));
    launch(iters);
    CU(cudaEventRecord(e1));
    CU(cudaEventSynchronize(e1));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double per_thread = (double)iters * 8.0 * (kind >= 2 ? 8.0 : 4.0);  // kinds 3, 4: four min + four xor
    *ops_per_sec = per_thread * threads * blocks / (ms * 1e-3);
    return QAPB_OK;
}
