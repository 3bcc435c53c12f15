// search_kernel.cuh -- device code of the QAP swap-delta hot path for sm_100a.
//
// One CTA owns one search (one start).  The per-search state is the *placement
// matrix* M and the vector h:
//
//   S[a][b] = sum_k ( D0[a][k]*F0[p_b][p_k] + D0[k][a]*F0[p_k][p_b] )     (cost of unit p_b at location a)
//   M[i][j] = S[i][j] + D0[i][j]*(F0[p_i][p_j] + F0[p_j][p_i]) + dd[i]*fd[p_j]     (i != j)
//   h[i]    = S[i][i] + dd[i]*fd[p_i]
//
// (F0/D0 = flow/distance with zeroed diagonals, fd/dd = their diagonals), for which
//
//   delta(i,j) = M[i][j] + M[j][i] - h[i] - h[j]
//
// reproduces the reference's O(n) exchange delta (_kernels.pyx:27-41) exactly,
// including the direct and diagonal terms, in integer arithmetic.  After a swap
// of locations r < s every entry of M outside rows/columns r,s receives the
// rank-2 correction  M[i][j] -= a[i]*b[j] + c[i]*e[j]  (a,c: column/row
// differences of D0; b,e: column/row differences of F0 gathered through p), and
// the 4n entries on rows/columns r,s have closed-form O(1) updates, so one
// iteration costs O(n^2) instead of the reference's O(n^3) re-evaluation
// (_kernels.pyx:159-161) while producing the same integers.
//
// M is tiled in 4x4 blocks; a *unit* is the block pair {(I,J),(J,I)}, I<J (or one
// diagonal block).  A thread owns whole units, so both M[i][j] and M[j][i] of a
// pair are thread-local and the update, the delta, the tabu/aspiration test
// (_kernels.pyx:162) and the running argmin are fused into one pass with
// 128-bit, bank-conflict-free shared-memory accesses ("spill layout":
// element (row w, thread t) of unit slot k lives at ((k*8+w)*T + t)*16 bytes).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qapb {

enum { MODE_TWO_OPT = 1, MODE_TABU = 2 };
enum { TENURE_CHUNK = 256 };  // tenure draws precomputed per refill

// ---- shared-memory layout, shared by host (size) and device (offsets) ------
struct SmemLayout {
    unsigned offM, offT, offA, offC, offB, offE, offH, offP, offU, offRedD, offRedK, offJ, offMisc, offTen;
    unsigned total;
};

__host__ __device__ inline unsigned align16(unsigned x) { return (x + 15u) & ~15u; }

__host__ __device__ inline SmemLayout make_layout(int npad, int nunits, int T, int upt,
                                                  int acc_bytes, int storage)
{
    SmemLayout L;
    unsigned o = 0;
    L.offM = o;
    if (storage == 0) o += (unsigned)upt * 8u * (unsigned)T * 4u * (unsigned)acc_bytes;
    o = align16(o);
    L.offT = o;
    if (storage <= 1) o += (unsigned)upt * (unsigned)T * 8u;  // per unit: 16-bit tabu mask word + earliest expiry
    o = align16(o);
    L.offA = o; o += 4u * npad;
    L.offC = o; o += 4u * npad;
    L.offB = o; o += 4u * npad;
    L.offE = o; o += 4u * npad;
    L.offH = o; o += (unsigned)acc_bytes * npad;
    o = align16(o);
    L.offP = o; o += 4u * npad;
    L.offJ = o; o += 4u * npad;
    L.offU = o; o += align16(2u * nunits);
    L.offRedD = o; o += 32u * 8u + 16u;
    L.offRedK = o; o += 32u * 4u;
    L.offMisc = o; o += 64u;
    L.offTen = o; o += 4u * TENURE_CHUNK;
    L.total = align16(o);
    return L;
}

struct HybLayout {  // search_hybrid.cuh
    unsigned offM, offTB, offMX, offA, offC, offB, offE, offH, offColR, offColS, offTR, offTS, offXR, offXS;
    unsigned offP, offJ, offRedD, offRedK, offMisc, offTen, offExp, offD16, offF16, offDT16, offFT16, offDG, total;
};

struct SearchParams {
    int n, nb, npad, nunits, noff, upt;
    int mode;        // MODE_*
    int rng;         // 1: derive start permutation + tenures on the device (multistart)
    int iterations;
    int symmetric;   // which matrices are symmetric: 0 none, 1 both, 2 distance only, 3 flow only
    int force_seq_rng;  // test hook: take the sequential (rejection-exact) RNG path
    int one, sixteen;   // runtime constants 1 and 16: multiplying by them keeps adds/shifts on the FMA (IMAD) pipe
    const int32_t *F, *FT, *D, *DT;  // [npad*npad], zero diagonal, zero padded
    const int32_t *fd, *dd;          // [npad] diagonals
    const uint16_t *unit_ij;         // [nunits]  I | J<<8
    const int64_t *perms;            // [B,n]            (rng == 0)
    const int64_t *tenures;          // [B,iterations]   (tabu, rng == 0)
    unsigned long long master_seed, first_index;
    const unsigned long long *seeds;  // [B] explicit per-start SplitMix64 states (rng == 1) or null
    long long ten_lo, ten_hi;
    int64_t *best, *best_cost, *cur, *cur_cost;
    int64_t *cells;                  // [B,n,n] or null
    int64_t *stopped, *steps;        // [B] or null
    int64_t *tr_i, *tr_j, *tr_d, *tr_tabu;  // [B,iterations] or null
    void *gM;                        // global placement matrices (storage 1)
    void *gT;                        // tabu expiry per (unit, slot), int32 (generic kernel; hybrid when not in smem)
    unsigned long long gM_stride, gT_stride;  // elements per start
    long long *dbg;                  // optional phase-cycle counters (development), else null
    SmemLayout lay;                  // generic kernel: offsets live in the constant bank
    HybLayout hlay;                  // hybrid kernel
    const int32_t *perm32;           // [B,npad] start permutations (qap_start_kernel)
    const unsigned long long *start_state;  // [B] SplitMix64 state after the shuffle
    const void *initM, *initH;       // [B,npad,npad], [B,npad] from qap_build_m_kernel (int32 or int64 state)
    unsigned inv_t;                  // generic: ceil(2^32 / threads), for uid / T without a division
    int toff, us, exp_in_smem;       // hybrid plan: off-diagonal threads, shared-memory units per thread
    int staged;                      // hybrid: int16 copies of D, F (and transposes) staged in shared memory
    int dsm;                         // hybrid: diagonal blocks in shared memory, owned by the last nb threads
    int batch;                       // searches of this launch (search_warp.cuh packs several into a CTA)
};

// ---- accumulator traits -----------------------------------------------------
template <typename acc_t> struct Acc;
template <> struct Acc<int32_t> {
    static __device__ __forceinline__ int32_t maxv() { return 0x7fffffff; }
    static __device__ __forceinline__ int32_t bighalf() { return 1 << 29; }
    static __device__ __forceinline__ int32_t clamp_thr(long long v)
    {
        return v < -2147483647LL ? (int32_t)0x80000000 : (int32_t)v;  // v <= 0 always
    }
};
template <> struct Acc<int64_t> {
    static __device__ __forceinline__ int64_t maxv() { return 0x7fffffffffffffffLL; }
    static __device__ __forceinline__ int64_t bighalf() { return 1LL << 61; }
    static __device__ __forceinline__ int64_t clamp_thr(long long v) { return v; }
};

// Row of four accumulators in the spill layout.
__device__ __forceinline__ void ld_row(const int32_t *base, int row, int T, int t, int32_t (&v)[4])
{
    int4 q = reinterpret_cast<const int4 *>(base)[row * T + t];
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
}
__device__ __forceinline__ void st_row(int32_t *base, int row, int T, int t, const int32_t (&v)[4])
{
    reinterpret_cast<int4 *>(base)[row * T + t] = make_int4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void ld_row(const int64_t *base, int row, int T, int t, int64_t (&v)[4])
{
    const longlong2 *b2 = reinterpret_cast<const longlong2 *>(base);
    longlong2 q0 = b2[(row * 2) * T + t], q1 = b2[(row * 2 + 1) * T + t];
    v[0] = q0.x; v[1] = q0.y; v[2] = q1.x; v[3] = q1.y;
}
__device__ __forceinline__ void st_row(int64_t *base, int row, int T, int t, const int64_t (&v)[4])
{
    longlong2 *b2 = reinterpret_cast<longlong2 *>(base);
    b2[(row * 2) * T + t] = make_longlong2(v[0], v[1]);
    b2[(row * 2 + 1) * T + t] = make_longlong2(v[2], v[3]);
}
__device__ __forceinline__ int32_t *elem_ptr(int32_t *base, int row, int T, int t, int lane4)
{
    return base + ((size_t)(row * T + t) * 4 + lane4);
}
__device__ __forceinline__ int64_t *elem_ptr(int64_t *base, int row, int T, int t, int lane4)
{
    return base + ((size_t)((row * 2 + (lane4 >> 1)) * T + t) * 2 + (lane4 & 1));
}

__device__ __forceinline__ void ld_vec4(const int32_t *arr, int blk, int32_t (&v)[4])
{
    int4 q = reinterpret_cast<const int4 *>(arr)[blk];
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
}
__device__ __forceinline__ void ld_h4(const int32_t *arr, int blk, int32_t (&v)[4]) { ld_vec4(arr, blk, v); }
__device__ __forceinline__ void ld_h4(const int64_t *arr, int blk, int64_t (&v)[4])
{
    const longlong2 *b2 = reinterpret_cast<const longlong2 *>(arr);
    longlong2 q0 = b2[blk * 2], q1 = b2[blk * 2 + 1];
    v[0] = q0.x; v[1] = q0.y; v[2] = q1.x; v[3] = q1.y;
}

// ---- SplitMix64 on the device (rng.py:12-20,35-47,62-70) ---------------------
#define QAPB_GAMMA 0x9E3779B97F4A7C15ULL
__device__ __forceinline__ unsigned long long mix64(unsigned long long z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// randbelow with the exact rejection rule: accept r iff r <= 2^64-1 - (2^64 mod bound).
__device__ inline unsigned long long randbelow_seq(unsigned long long &state, unsigned long long bound)
{
    unsigned long long rem = (0ULL - bound) % bound;
    unsigned long long last_ok = ~0ULL - rem;
    for (;;) {
        state += QAPB_GAMMA;
        unsigned long long r = mix64(state);
        if (r <= last_ok) return r % bound;
    }
}


// Tenure stream (tabu.py:184-186), TENURE_CHUNK draws at a time: draw k of a chunk is
// mix64(state + (k+1)*GAMMA), computed by thread k; if any draw would be rejected by
// randbelow (probability ~ span/2^64) thread 0 replays the chunk with the exact
// sequential rule.  Every thread keeps the stream state, so no 64-bit division sits on
// the per-iteration critical path.  Must be called by all threads of the CTA.
__device__ inline void fill_tenure_chunk(unsigned long long &state, long long lo, long long hi, int force_seq,
                                         int32_t *sTen, long long *sMisc, int tid, int T)
{
    const unsigned long long span = (unsigned long long)(hi - lo + 1);
    const unsigned long long last_ok = ~0ULL - (0ULL - span) % span;
    int reject = force_seq;
    for (int k = tid; k < TENURE_CHUNK; k += T) {
        const unsigned long long r = mix64(state + QAPB_GAMMA * ((unsigned long long)k + 1ULL));
        if (r > last_ok) reject = 1;
        sTen[k] = (int32_t)(lo + (long long)(r % span));
    }
    reject = __syncthreads_or(reject);
    if (reject) {
        if (tid == 0) {
            unsigned long long st = state;
            for (int k = 0; k < TENURE_CHUNK; ++k) sTen[k] = (int32_t)(lo + (long long)randbelow_seq(st, span));
            sMisc[3] = (long long)st;
        }
        __syncthreads();
        state = (unsigned long long)sMisc[3];
    } else {
        state += QAPB_GAMMA * (unsigned long long)TENURE_CHUNK;
    }
}

// ---- warp / block reductions ------------------------------------------------
// Lexicographic minimum of (value, key) over a warp; all lanes get the result.
__device__ __forceinline__ void warp_argmin(int32_t &d, unsigned &key)
{
    int32_t m = __reduce_min_sync(0xffffffffu, d);
    unsigned k = __reduce_min_sync(0xffffffffu, d == m ? key : 0xffffffffu);
    d = m;
    key = k;
}
__device__ __forceinline__ void warp_argmin(int64_t &d, unsigned &key)
{
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        int64_t od = __shfl_xor_sync(0xffffffffu, d, off);
        unsigned ok = __shfl_xor_sync(0xffffffffu, key, off);
        if (od < d || (od == d && ok < key)) {
            d = od;
            key = ok;
        }
    }
}

__device__ __forceinline__ long long block_sum_i64(long long v, long long *scratch /* >= 33 */, int tid, int T)
{
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if ((tid & 31) == 0) scratch[tid >> 5] = v;
    __syncthreads();
    if (tid < 32) {
        long long s = tid < (T >> 5) ? scratch[tid] : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (tid == 0) scratch[32] = s;
    }
    __syncthreads();
    return scratch[32];
}

__device__ __forceinline__ unsigned pair_key(int i, int j, int flag)
{
    return ((unsigned)i << 17) | ((unsigned)j << 1) | (unsigned)flag;
}

// Locate element M[x][y] (x != y) in the spill layout: returns row index
// (k*8 + w) and owning thread / lane.
struct ElemLoc { int row, t, lane4; };
__device__ __forceinline__ ElemLoc locate(int x, int y, int nb, int noff, int T, unsigned inv_t)
{
    int X = x >> 2, Y = y >> 2, uid, w, l;
    if (X < Y) {
        uid = X * nb - ((X * (X + 1)) >> 1) + (Y - X - 1);
        w = x & 3; l = y & 3;
    } else if (X > Y) {
        uid = Y * nb - ((Y * (Y + 1)) >> 1) + (X - Y - 1);
        w = 4 + (y & 3); l = x & 3;  // the lower block is stored transposed (row u holds L[0..3][u])
    } else {
        uid = noff + X;
        w = x & 3; l = y & 3;
    }
    int k = (int)__umulhi((unsigned)uid, inv_t);  // uid / T by the host's ceil(2^32 / T): exact for uid * T < 2^32
    ElemLoc e;
    e.t = uid - k * T;
    e.row = k * 8 + w;
    e.lane4 = l;
    return e;
}

// -----------------------------------------------------------------------------
// The generic search kernel: any n <= 1020, int32 or int64 state.  STORAGE 0 keeps M in
// shared memory, STORAGE 1 in an L2-resident workspace, STORAGE 2 (n > ~700) also keeps the
// per-unit tabu masks there.  Start permutation, stream state,
// M and h come from qap_start_kernel / qap_build_m_kernel (build_kernels.cuh).  M is
// streamed through registers one row pair at a time (row u of the upper block with row u of
// the transposed lower block), so eight accumulators are live per thread.  The tabu
// triangle is a 16-bit mask per unit (pairs that are tabu now) plus the unit's earliest
// expiry in shared memory; the expiry iterations themselves live in an L2-resident array
// that is touched only when a pair is set or expires.
// -----------------------------------------------------------------------------
__device__ __forceinline__ void expire_unit_bits(unsigned &tb, int32_t &mexp, int c, const int32_t *xp16)
{
    // one 128-bit load per block row that has a bit set: the rows are independent, so their L2 latencies
    // overlap (a loop over single bits pays one latency per bit)
    int32_t nm = 0x7fffffff;
    unsigned keep = tb;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        if ((tb >> (4 * u)) & 15u) {
            const int4 e4 = reinterpret_cast<const int4 *>(xp16)[u];
            const int32_t e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const unsigned bit = 1u << (4 * u + v);
                if (tb & bit) {
                    if (e[v] <= c) keep &= ~bit;
                    else if (e[v] != 0x7fffffff) nm = min(nm, e[v]);
                }
            }
        }
    }
    tb = keep;
    mexp = nm;
}

template <typename acc_t, int STORAGE, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) qap_search_kernel(const SearchParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, W = T >> 5;
    const int b = blockIdx.x;
    const int n = P.n, nb = P.nb, npad = P.npad, noff = P.noff, nunits = P.nunits, upt = P.upt;
    const SmemLayout &lay = P.lay;

    acc_t *M = STORAGE == 0 ? reinterpret_cast<acc_t *>(smem_raw + lay.offM)
                            : reinterpret_cast<acc_t *>(P.gM) + (size_t)b * P.gM_stride;
    int32_t *xp = reinterpret_cast<int32_t *>(P.gT) + (size_t)b * P.gT_stride;  // [nunits*16] (+ masks, STORAGE 2)
    unsigned *sTB = STORAGE <= 1 ? reinterpret_cast<unsigned *>(smem_raw + lay.offT)  // [upt*T] tabu-now masks
                                 : reinterpret_cast<unsigned *>(xp + (size_t)nunits * 16);
    int32_t *sMX = reinterpret_cast<int32_t *>(sTB + (size_t)upt * T);  // [upt*T] earliest expiry
    int32_t *sA = reinterpret_cast<int32_t *>(smem_raw + lay.offA);
    int32_t *sC = reinterpret_cast<int32_t *>(smem_raw + lay.offC);
    int32_t *sB = reinterpret_cast<int32_t *>(smem_raw + lay.offB);
    int32_t *sE = reinterpret_cast<int32_t *>(smem_raw + lay.offE);
    acc_t *sH = reinterpret_cast<acc_t *>(smem_raw + lay.offH);
    int32_t *sP = reinterpret_cast<int32_t *>(smem_raw + lay.offP);
    uint16_t *sU = reinterpret_cast<uint16_t *>(smem_raw + lay.offU);
    long long *sRed64 = reinterpret_cast<long long *>(smem_raw + lay.offRedD);  // 33 x 8 B
    acc_t *sRedD = reinterpret_cast<acc_t *>(smem_raw + lay.offRedD);
    unsigned *sRedK = reinterpret_cast<unsigned *>(smem_raw + lay.offRedK);
    long long *sMisc = reinterpret_cast<long long *>(smem_raw + lay.offMisc);
    int32_t *sTen = reinterpret_cast<int32_t *>(smem_raw + lay.offTen);

    const int32_t *__restrict__ F = P.F;
    const int32_t *__restrict__ FT = P.FT;
    const int32_t *__restrict__ D = P.D;
    const int32_t *__restrict__ DT = P.DT;
    const bool sym = P.symmetric != 0;  // single-product rank-2 update: at least one symmetric matrix
    const acc_t MAXV = Acc<acc_t>::maxv();
    const int32_t MAXE = 0x7fffffff;

    // ---------------------------------------------------------------- setup
    const acc_t *__restrict__ Hinit = reinterpret_cast<const acc_t *>(P.initH) + (size_t)b * npad;
    const acc_t *__restrict__ Minit = reinterpret_cast<const acc_t *>(P.initM) + (size_t)b * npad * npad;
    for (int u = tid; u < nunits; u += T) sU[u] = P.unit_ij[u];
    for (int i = tid; i < npad; i += T) {
        sA[i] = 0; sC[i] = 0; sB[i] = 0; sE[i] = 0;
        sH[i] = Hinit[i];
        sP[i] = P.perm32[(size_t)b * npad + i];
    }
    unsigned long long rng_state = P.rng ? P.start_state[b] : 0ULL;  // stream state after the shuffle
    if (P.cells) {
        int64_t *cz = P.cells + (size_t)b * n * n;
        for (int i = tid; i < n * n; i += T) cz[i] = 0;
    }
    __syncthreads();

    // full cost (_kernels.pyx:18-24), int64, including the diagonal products.
    long long cost;
    {
        long long part = 0;
        for (int idx = tid; idx < n * n; idx += T) {
            int i = idx / n, j = idx - i * n;
            int pi = sP[i], pj = sP[j];
            part += (i == j) ? (long long)P.fd[pi] * P.dd[i]
                             : (long long)F[pi * npad + pj] * D[i * npad + j];
        }
        cost = block_sum_i64(part, sRed64, tid, T);
        __syncthreads();
    }

    // units into the spill layout (lower block transposed); tabu masks: pads and non-pairs are
    // permanently set with expiry MAXE
    for (int k = 0; k < upt; ++k) {
        const int uid = tid + k * T;
        if (uid >= nunits) { sTB[k * T + tid] = 0xffffu; sMX[k * T + tid] = MAXE; continue; }
        const int I = sU[uid] & 0xff, J = sU[uid] >> 8;
        unsigned dead = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            acc_t Ur[4], Lt[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                Ur[v] = Minit[(size_t)(4 * I + u) * npad + 4 * J + v];
                Lt[v] = Minit[(size_t)(4 * J + v) * npad + 4 * I + u];
                if (4 * I + u >= n || 4 * J + v >= n || (I == J && u >= v)) dead |= 1u << (u * 4 + v);
            }
            st_row(M, k * 8 + u, T, tid, Ur);
            st_row(M, k * 8 + 4 + u, T, tid, Lt);
        }
        sTB[k * T + tid] = dead;
        sMX[k * T + tid] = MAXE;
#pragma unroll
        for (int q = 0; q < 16; ++q) xp[(size_t)uid * 16 + q] = ((dead >> q) & 1u) ? MAXE : 0;
    }
    __syncthreads();

    // ------------------------------------------------------------ iterations
    long long best_cost = cost;
    acc_t thr = 0;  // best_cost - cost, clamped; aspiration <=> d < thr  (_kernels.pyx:162)
    const bool tabu = P.mode == MODE_TABU;
    const int iters = P.iterations;
    int steps_done = 0, stopped = 0;
    int64_t *best_out = P.best + (size_t)b * n;
    for (int i = tid; i < n; i += T) best_out[i] = sP[i];

    for (int c = 1; c <= iters; ++c) {
        long long ten = 0;
        if (tabu) {
            if (!P.rng) {
                ten = P.tenures[(size_t)b * iters + (c - 1)];  // consumed after the pass
            } else if (((c - 1) & (TENURE_CHUNK - 1)) == 0) {
                fill_tenure_chunk(rng_state, P.ten_lo, P.ten_hi, P.force_seq_rng, sTen, sMisc, tid, T);
            }
        }

        // ---- fused pass: rank-2 update, delta, admissibility, running argmin
        acc_t bd = MAXV;
        unsigned bkey = 0xffffffffu;
        for (int k = 0; k < upt; ++k) {
            const int uid = tid + k * T;
            if (uid >= nunits) break;
            const int I = sU[uid] & 0xff, J = sU[uid] >> 8;
            unsigned tbk = sTB[k * T + tid];
            if (c >= sMX[k * T + tid]) {  // some pair of this unit stops being tabu now
                int32_t mx;
                expire_unit_bits(tbk, mx, c, xp + (size_t)uid * 16);
                sTB[k * T + tid] = tbk;
                sMX[k * T + tid] = mx;
            }
            acc_t m = MAXV;
            int slot = 0;
            if (I != J) {
                int32_t aJ[4], bJ[4], cJ[4], eJ[4];
                ld_vec4(sA, J, aJ); ld_vec4(sB, J, bJ);
                if (!sym) { ld_vec4(sC, J, cJ); ld_vec4(sE, J, eJ); }
                acc_t hJ[4];
                ld_h4(sH, J, hJ);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc_t Ur[4], Lr[4];
                    ld_row(M, k * 8 + u, T, tid, Ur);
                    ld_row(M, k * 8 + 4 + u, T, tid, Lr);
                    if (c > 1) {
                        const int32_t aIu = sA[4 * I + u], bIu = sB[4 * I + u];
                        if (sym) {  // one product: the published a, b are pre-combined (and a, c negated; see the prep phase)
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                Ur[v] += (acc_t)aIu * (acc_t)bJ[v];
                                Lr[v] += (acc_t)aJ[v] * (acc_t)bIu;
                            }
                        } else {
                            const int32_t cIu = sC[4 * I + u], eIu = sE[4 * I + u];
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                Ur[v] += (acc_t)aIu * (acc_t)bJ[v] + (acc_t)cIu * (acc_t)eJ[v];
                                Lr[v] += (acc_t)aJ[v] * (acc_t)bIu + (acc_t)cJ[v] * (acc_t)eIu;
                            }
                        }
                        st_row(M, k * 8 + u, T, tid, Ur);
                        st_row(M, k * 8 + 4 + u, T, tid, Lr);
                    }
                    const acc_t hIu = sH[4 * I + u];
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const acc_t d = Ur[v] + Lr[v] - hIu - hJ[v];
                        const bool tb = (tbk >> (u * 4 + v)) & 1u;
                        if ((!tb || d < thr) && d < m) { m = d; slot = u * 4 + v; }
                    }
                }
            } else {
                acc_t U[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) ld_row(M, k * 8 + u, T, tid, U[u]);
                if (c > 1) {
                    int32_t aI[4], bI[4], cI[4], eI[4];
                    ld_vec4(sA, I, aI); ld_vec4(sB, I, bI); ld_vec4(sC, I, cI); ld_vec4(sE, I, eI);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            if (u != v)
                                U[u][v] += sym ? (acc_t)aI[u] * (acc_t)bI[v]
                                               : (acc_t)aI[u] * (acc_t)bI[v] + (acc_t)cI[u] * (acc_t)eI[v];
#pragma unroll
                    for (int u = 0; u < 4; ++u) st_row(M, k * 8 + u, T, tid, U[u]);
                }
                acc_t hI[4];
                ld_h4(sH, I, hI);
#pragma unroll
                for (int u = 0; u < 3; ++u)
#pragma unroll
                    for (int v = u + 1; v < 4; ++v) {
                        const acc_t d = U[u][v] + U[v][u] - hI[u] - hI[v];
                        const bool tb = (tbk >> (u * 4 + v)) & 1u;
                        if ((!tb || d < thr) && d < m) { m = d; slot = u * 4 + v; }
                    }
            }
            if (m != MAXV && m <= bd) {
                const unsigned key = pair_key(4 * I + (slot >> 2), 4 * J + (slot & 3), (tbk >> slot) & 1u);
                if (m < bd || key < bkey) { bd = m; bkey = key; }
            }
        }
        warp_argmin(bd, bkey);
        if (lane == 0) { sRedD[warp] = bd; sRedK[warp] = bkey; }
        __syncthreads();  // ---------------------------------------------- sync #1
        bd = lane < W ? sRedD[lane] : MAXV;
        bkey = lane < W ? sRedK[lane] : 0xffffffffu;
        warp_argmin(bd, bkey);
        if (bd == MAXV) {  // no admissible move: premature stop (_kernels.pyx:168-170)
            stopped = 1;
            break;
        }
        const int r = (int)(bkey >> 17), s = (int)((bkey >> 1) & 0xffffu);
        const int was_tabu = (int)(bkey & 1u);
        cost += (long long)bd;
        const bool improved = cost < best_cost;
        if (improved) best_cost = cost;
        thr = Acc<acc_t>::clamp_thr(best_cost - cost);
        if (tabu && P.rng) ten = sTen[(c - 1) & (TENURE_CHUNK - 1)];
        steps_done = c;

        if (tid == 0) {
            if (P.tr_i) {
                const size_t o = (size_t)b * iters + (c - 1);
                P.tr_i[o] = r; P.tr_j[o] = s; P.tr_d[o] = (int64_t)bd;
                if (P.tr_tabu) P.tr_tabu[o] = was_tabu;
            }
        }

        // ---- prep: difference vectors (old permutation), h, rows/columns r,s
        {
            const int pr = sP[r], ps = sP[s];
            const int32_t Drs = D[r * npad + s], Dsr = D[s * npad + r];
            const int32_t Fpspr = F[ps * npad + pr], Fprps = F[pr * npad + ps];
            for (int i = tid; i < n; i += T) {
                const int pi = sP[i];
                const int32_t Dsi = D[s * npad + i], Dri = D[r * npad + i];
                const int32_t Dis = DT[s * npad + i], Dir = DT[r * npad + i];
                const int32_t Fpips = FT[ps * npad + pi], Fpipr = FT[pr * npad + pi];
                const int32_t Fpspi = F[ps * npad + pi], Fprpi = F[pr * npad + pi];
                int32_t a = Dis - Dir, cc = Dsi - Dri, bb = Fpips - Fpipr, e = Fpspi - Fprpi;
                if (improved) best_out[i] = (i == r) ? ps : (i == s) ? pr : pi;
                if (i == r) {
                    // corners and h[r], h[s]
                    ElemLoc lrs = locate(r, s, nb, noff, T, P.inv_t), lsr = locate(s, r, nb, noff, T, P.inv_t);
                    acc_t *prs = elem_ptr(M, lrs.row, T, lrs.t, lrs.lane4);
                    acc_t *psr = elem_ptr(M, lsr.row, T, lsr.t, lsr.lane4);
                    const acc_t mrs = *prs, msr = *psr, hr = sH[r], hs = sH[s];
                    *prs = hr + (acc_t)(Drs - Dsr) * (acc_t)Fpspr;
                    *psr = hs + (acc_t)(Dsr - Drs) * (acc_t)Fprps;
                    sH[r] = mrs + (acc_t)(Dsr - Drs) * (acc_t)Fprps;
                    sH[s] = msr + (acc_t)(Drs - Dsr) * (acc_t)Fpspr;
                    a = 0; cc = 0; bb = 0; e = 0;
                } else if (i == s) {
                    if (tabu) {  // cells[bi][bj] = c + t; cells[bj][bi] += 1  (_kernels.pyx:176-178)
                        const int R = r >> 2, S = s >> 2;
                        const int uid = (R < S) ? R * nb - ((R * (R + 1)) >> 1) + (S - R - 1) : noff + R;
                        const int kq = (int)__umulhi((unsigned)uid, P.inv_t), tq = uid - kq * T;
                        const int q = (r & 3) * 4 + (s & 3);
                        const int32_t new_exp = (int32_t)(c + ten);
                        sTB[kq * T + tq] |= 1u << q;
                        sMX[kq * T + tq] = min(sMX[kq * T + tq], new_exp);
                        xp[(size_t)uid * 16 + q] = new_exp;
                        if (P.cells) {
                            int64_t *cz = P.cells + (size_t)b * n * n;
                            cz[(size_t)r * n + s] = (int64_t)c + ten;
                            atomicAdd(reinterpret_cast<unsigned long long *>(cz + (size_t)s * n + r), 1ULL);  // (a reduction without return: the load-add-store would wait for L2)
                        }
                    }
                    a = 0; cc = 0; bb = 0; e = 0;
                } else {
                    ElemLoc lri = locate(r, i, nb, noff, T, P.inv_t), lsi = locate(s, i, nb, noff, T, P.inv_t);
                    ElemLoc lir = locate(i, r, nb, noff, T, P.inv_t), lis = locate(i, s, nb, noff, T, P.inv_t);
                    acc_t *pri = elem_ptr(M, lri.row, T, lri.t, lri.lane4);
                    acc_t *psi = elem_ptr(M, lsi.row, T, lsi.t, lsi.lane4);
                    acc_t *pir = elem_ptr(M, lir.row, T, lir.t, lir.lane4);
                    acc_t *pis = elem_ptr(M, lis.row, T, lis.t, lis.lane4);
                    const acc_t mri = *pri, msi = *psi, mir = *pir, mis = *pis;
                    const acc_t be = (acc_t)bb + (acc_t)e;
                    const acc_t fs_ps = (acc_t)Fpips + (acc_t)Fpspi;  // Fs[p_i][p_s]
                    const acc_t fs_pr = (acc_t)Fpipr + (acc_t)Fprpi;  // Fs[p_i][p_r]
                    *pri = mri - (acc_t)Drs * (acc_t)bb - (acc_t)Dsr * (acc_t)e + (acc_t)Dri * be;
                    *psi = msi + (acc_t)Dsr * (acc_t)bb + (acc_t)Drs * (acc_t)e - (acc_t)Dsi * be;
                    *pir = mis + (acc_t)a * ((acc_t)Fpspr - fs_ps) + (acc_t)cc * (acc_t)Fprps;
                    *pis = mir + (acc_t)a * (fs_pr - (acc_t)Fprps) - (acc_t)cc * (acc_t)Fpspr;
                    sH[i] -= (acc_t)a * (acc_t)bb + (acc_t)cc * (acc_t)e;
                }
                // single-product forms: both symmetric a == c, b == e -> (2a) b; D = D^T only a == c -> a (b + e);
                // F = F^T only b == e -> (a + c) b
                // a and c are stored NEGATED, so the update is a multiply-add (one IMAD.WIDE per product with
                // int64 state instead of a product and a 64-bit subtraction)
                sA[i] = -(P.symmetric == 1 ? 2 * a : P.symmetric == 3 ? a + cc : a);
                sB[i] = P.symmetric == 2 ? bb + e : bb;
                sC[i] = -cc; sE[i] = e;
            }
        }
        __syncthreads();  // ---------------------------------------------- sync #2
        if (tid == 0) { const int32_t t = sP[r]; sP[r] = sP[s]; sP[s] = t; }
    }
    __syncthreads();

    for (int i = tid; i < n; i += T) P.cur[(size_t)b * n + i] = sP[i];
    if (tid == 0) {
        P.best_cost[b] = best_cost;
        P.cur_cost[b] = cost;
        if (P.stopped) P.stopped[b] = stopped;
        if (P.steps) P.steps[b] = steps_done;
    }
}

// ---- kernels.full_cost, batched (one CTA per permutation) -------------------
__global__ void qap_full_cost_kernel(int n, int npad, const int32_t *__restrict__ F,
                                     const int32_t *__restrict__ D, const int32_t *__restrict__ fd,
                                     const int32_t *__restrict__ dd, const int64_t *__restrict__ perms,
                                     int64_t *__restrict__ costs)
{
    __shared__ long long scratch[33];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int32_t *sP = reinterpret_cast<int32_t *>(smem_raw);
    const int tid = threadIdx.x, T = blockDim.x, b = blockIdx.x;
    for (int i = tid; i < n; i += T) sP[i] = (int32_t)perms[(size_t)b * n + i];
    __syncthreads();
    long long part = 0;
    for (int idx = tid; idx < n * n; idx += T) {
        int i = idx / n, j = idx - i * n;
        int pi = sP[i], pj = sP[j];
        part += (i == j) ? (long long)fd[pi] * dd[i] : (long long)F[pi * npad + pj] * D[i * npad + j];
    }
    long long total = block_sum_i64(part, scratch, tid, T);
    if (tid == 0) costs[b] = total;
}

// ---- multistart reduce: min (cost, index), ties -> lowest index (multistart.py:156)
__global__ void qap_pick_best_kernel(int count, int n, unsigned long long first_index,
                                     const int64_t *__restrict__ costs,
                                     const int64_t *__restrict__ best_perms /* [count,n] */,
                                     int64_t *__restrict__ best_key, int64_t *__restrict__ best_perm,
                                     const int64_t *__restrict__ steps = nullptr, int64_t *__restrict__ total_steps = nullptr)
{
    __shared__ long long sc[32];
    __shared__ long long ssum[33];
    if (total_steps) {  // sum of steps_done over the starts: evals = sum * n(n-1)/2 even when starts stop early
        long long part = 0;
        for (int k = threadIdx.x; k < count; k += blockDim.x) part += steps[k];
        part = block_sum_i64(part, ssum, threadIdx.x, blockDim.x);
        if (threadIdx.x == 0) *total_steps = part;
    }
    __shared__ int si[32];
    __shared__ int winner;
    const int tid = threadIdx.x, T = blockDim.x;
    long long bc = 0x7fffffffffffffffLL;
    int bi = 0x7fffffff;
    for (int k = tid; k < count; k += T) {
        long long c = costs[k];
        if (c < bc || (c == bc && k < bi)) { bc = c; bi = k; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        long long oc = __shfl_xor_sync(0xffffffffu, bc, off);
        int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (oc < bc || (oc == bc && oi < bi)) { bc = oc; bi = oi; }
    }
    if ((tid & 31) == 0) { sc[tid >> 5] = bc; si[tid >> 5] = bi; }
    __syncthreads();
    if (tid < 32) {
        bc = tid < (T >> 5) ? sc[tid] : 0x7fffffffffffffffLL;
        bi = tid < (T >> 5) ? si[tid] : 0x7fffffff;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            long long oc = __shfl_xor_sync(0xffffffffu, bc, off);
            int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (oc < bc || (oc == bc && oi < bi)) { bc = oc; bi = oi; }
        }
        if (tid == 0) {
            winner = bi;
            best_key[0] = bc;
            best_key[1] = (int64_t)(first_index + (unsigned long long)bi);
        }
    }
    __syncthreads();
    for (int i = tid; i < n; i += T) best_perm[i] = best_perms[(size_t)winner * n + i];
}

// ---- shared-memory bandwidth probe: conflict-free 128-bit loads, eight independent chains per thread ----
__global__ void __launch_bounds__(1024) qap_smem_probe_kernel(int iters, int *sink)
{
    __shared__ int4 buf[1024 * 2];
    for (int k = threadIdx.x; k < 2048; k += blockDim.x) buf[k] = make_int4(k, k + 1, k + 2, k + 3);
    __syncthreads();
    int4 acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = make_int4(0, 0, 0, 0);
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int4 v = buf[(idx + 32 * q) & 2047];
            acc[q].x += v.x; acc[q].y ^= v.y; acc[q].z += v.z; acc[q].w ^= v.w;
        }
        idx = (idx + 256) & 2047;
    }
    int t = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t ^= acc[q].x ^ acc[q].y ^ acc[q].z ^ acc[q].w;
    if (t == 0x12345678) *sink = 1;
}

// ---- integer-pipe peak probe -----------------------------------------------
template <int KIND>
__global__ void qap_int_probe_kernel(int iters, int *sink, int seed)
{
    int x0 = threadIdx.x + seed, x1 = x0 * 3 + 1, x2 = x0 * 5 + 2, x3 = x0 * 7 + 3;
    int y0 = x0 ^ 11, y1 = x1 ^ 13, y2 = x2 ^ 17, y3 = x3 ^ 19;
    const int m = seed | 1, a = seed + 7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (KIND == 0 || KIND == 2) { x0 = x0 * m + a; x1 = x1 * m + a; x2 = x2 * m + a; x3 = x3 * m + a; }
            if (KIND == 3) {  // DPX add-then-min (VIADDMNMX), four independent chains
                y0 = __viaddmin_s32(x0, a, y0); y1 = __viaddmin_s32(x1, a, y1);
                y2 = __viaddmin_s32(x2, a, y2); y3 = __viaddmin_s32(x3, a, y3);
                x0 ^= y1; x1 ^= y2; x2 ^= y3; x3 ^= y0;
            }
            if (KIND == 4) {  // plain min (VIMNMX)
                y0 = min(x0, y0); y1 = min(x1, y1); y2 = min(x2, y2); y3 = min(x3, y3);
                x0 ^= y1; x1 ^= y2; x2 ^= y3; x3 ^= y0;
            }
            if (KIND == 1 || KIND == 2) {
                y0 = (y0 + a) + y1;
                y1 = (y1 + a) + y2;
                y2 = (y2 + a) + y3;
                y3 = (y3 + a) + y0;
            }
        }
    }
    if ((x0 ^ x1 ^ x2 ^ x3 ^ y0 ^ y1 ^ y2 ^ y3) == 0x12345678) *sink = 1;
}

}  // namespace qapb
