// search_warp.cuh -- one WARP per search, n <= 32 (nug12, tai30a: BASELINE configs[0] and configs[1]).
//
// The hybrid kernel (search_hybrid.cuh) spreads a search over a CTA and pays two block barriers, a
// two-level argmin and register-indexed fix-up regions per iteration; at n <= 32 a whole search is 28
// off-diagonal units, so that machinery is all that is left of the iteration.  Here a search is one warp
// and nothing but warp-synchronous code:
//   * lane l is LOCATION l for the publish phase (p[l], h[l] live in its registers), the owner of one
//     off-diagonal UNIT (block pair {(I,J),(J,I)}, 16 pairs; the unit whose chunk slot is l) for the pass, and
//     the owner of the diagonal-block pairs l and l + 32 (of 6 per diagonal block), one scalar pair at a
//     time -- every lane runs the same instruction stream, there is no diagonal warp or diagonal path to
//     diverge into;
//   * the units live in the warp's slice of shared memory and stream through registers once per pass
//     (conflict-free 128-bit loads and stores of the owner lane); the 4n entries on rows/columns r,s of a move
//     are fixed in place there: the lane of location i patches M[i][r], M[r][i], M[i][s], M[s][i] -- four
//     loads, four stores, addresses from a table shared by the CTA -- no column dump, no fix-up vectors, no
//     register-indexed switch, and no divergent region on the serial path behind the argmin;
//   * the argmin is two `redux.sync`; the two barriers of an iteration are `__syncwarp()`;
//   * the start permutation, the tenure stream (32 draws at a time, one per lane, exact sequential replay on
//     a rejected draw; the tenure of an iteration comes out of its lane by shuffle) and the initial
//     placement matrix are produced in this kernel: a small-n multistart is two launches (search, pick);
//   * searches share nothing but the address table, so a CTA holds 1-4 warps; at n <= 16 a search is a
//     half-warp (G = 16) and a warp runs two.
// Same integers as every other plan: the formulas of the publish phase are the ones of search_hybrid.cuh.
// int32 state with packed selection keys only (|delta| < 2^27, host-proven); other instances of this size
// keep the hybrid plans.
#pragma once
#include "search_hybrid.cuh"

namespace qapb {

// Layout of one search's slice of shared memory, in 32-bit words; G = lanes per search (32, or 16 for n <= 16:
// two searches per warp).  Unit (I,J) sits in chunk slot ((I + J) & 7) + 8 * rank (rank among the units with the
// same residue) -- the lane with that index owns it -- and element v of row w is stored at position (v + w) & 3 of
// its 16-byte chunk: the lanes of the fix-ups, which walk a column or a row of M (all block rows X against one
// block R), then hit 32 different banks, 4 ((X + R) & 7) + ((xu + ru) & 3), while the owner's own accesses stay
// conflict-free 128-bit ones.
template <int G> struct WkLay {
    static constexpr int RSW = G * 4;                // row stride of the unit layout
    static constexpr int M = 0;                      // 8 rows (0-3: upper block, 4-7: lower block transposed) x G units x 4
    static constexpr int DG = 8 * RSW;               // diagonal-block pairs: [round q][x | y][lane]
    static constexpr int XP = DG + 4 * G;            // G units x 16: tabu expiry per (unit, slot)
    static constexpr int A = XP + 16 * G;            // difference vectors of the last move (negated a, c)
    static constexpr int B = A + G;
    static constexpr int C = B + G;
    static constexpr int E = C + G;
    static constexpr int HI = E + G;                 // packed-key forms of h (search_hybrid.cuh)
    static constexpr int HJ = HI + G;
    static constexpr int P = HJ + G;                 // permutation (setup only)
    static constexpr int TOTAL = P + G;              // words per search
    static constexpr int TAB = G * G + 32;           // words shared by the CTA: address table, then slot / unit maps (64 + 64 bytes)
};
__host__ __device__ inline unsigned wk_smem_bytes(int G, int warps)
{
    const int total = G == 32 ? WkLay<32>::TOTAL : WkLay<16>::TOTAL;
    return 4u * (unsigned)(G * G + 32 + warps * (32 / G) * total);
}

// chunk slot of unit (I,J), I < J < nb
__host__ __device__ inline int wk_unit_slot(int I, int J, int nb)
{
    const int k = (I + J) & 7;
    int rank = 0;
    for (int a = 0; a < nb; ++a)
        for (int b2 = a + 1; b2 < nb; ++b2) {
            if (a == I && b2 == J) return k + 8 * rank;
            if (((a + b2) & 7) == k) ++rank;
        }
    return 0;
}

// Word offsets (in a search's slice) of M[x][y] and M[y][x], x != y.  One off-diagonal unit holds both entries,
// four rows apart; a pair inside a diagonal block lives in the slot of the lane that owns it.
template <int G>
__device__ __forceinline__ unsigned wk_pair_words(int x, int y, const unsigned char *slot_of)
{
    typedef WkLay<G> LY;
    const int X = x >> 2, xu = x & 3, Y = y >> 2, yu = y & 3;
    int w_xy, w_yx;
    if (X == Y) {
        const int lo = min(xu, yu), hi = max(xu, yu);
        const int pp = lo == 0 ? hi - 1 : lo == 1 ? hi + 1 : 5;   // (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)
        const int idx = 6 * X + pp, q = idx / G, l = idx - q * G;
        const int wx = LY::DG + q * 2 * G + l;                     // M[lo][hi]; M[hi][lo] is G words on
        w_xy = xu < yu ? wx : wx + G;
        w_yx = xu < yu ? wx + G : wx;
    } else {
        const bool up = X < Y;
        const int I = up ? X : Y, J = up ? Y : X;
        const int uid = slot_of[I * 8 + J];
        // X < Y: M[x][y] = U[xu][yu] (row xu, column yu), M[y][x] = L[yu][xu] (row 4 + xu, column yu)
        // X > Y: M[y][x] = U[yu][xu] (row yu, column xu), M[x][y] = L[xu][yu] (row 4 + yu, column xu)
        const int row = up ? xu : yu;
        const int wU = row * LY::RSW + uid * 4 + ((xu + yu) & 3);
        w_xy = up ? wU : wU + 4 * LY::RSW;
        w_yx = up ? wU + 4 * LY::RSW : wU;
    }
    return (unsigned)w_xy | ((unsigned)w_yx << 16);
}

// Predicated shared-memory accesses as single instructions: small `if` bodies on the serial path compile to
// divergent regions, and waiting for their reconvergence (stall "branch resolving" at the BSYNC) was 7 % of an
// iteration with the flush of the touched units alone.
__device__ __forceinline__ int32_t lds32_if(bool p, const int32_t *ptr, int32_t otherwise)
{
    int32_t v = otherwise;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.s32 %0, [%1];\n\t}"
                 : "+r"(v) : "r"((unsigned)__cvta_generic_to_shared(ptr)), "r"((unsigned)p) : "memory");
    return v;
}
__device__ __forceinline__ void stg64_if(bool p, int64_t *ptr, int64_t v)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.s64 [%0], %1;\n\t}" :: "l"(ptr), "l"(v), "r"((unsigned)p) : "memory");
}
__device__ __forceinline__ void redg64_inc_if(bool p, int64_t *ptr)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q red.global.add.u64 [%0], 1;\n\t}" :: "l"(ptr), "r"((unsigned)p) : "memory");
}
__device__ __forceinline__ void sts32_if(bool p, int32_t *ptr, int32_t v)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.s32 [%0], %1;\n\t}"
                 :: "r"((unsigned)__cvta_generic_to_shared(ptr)), "r"(v), "r"((unsigned)p) : "memory");
}

// G tenures (tabu.py:184-186), one per lane: draw k of the chunk is mix64(state + (k+1)*GAMMA); a draw that
// randbelow would reject (probability ~ span / 2^64) makes every lane replay the chunk with the exact rule.
template <int G>
__device__ __forceinline__ int32_t warp_tenure_chunk(unsigned gmask, unsigned long long &state, unsigned long long span,
                                                     unsigned long long last_ok, long long lo, int force_seq, int gl)
{
    const unsigned long long r = mix64(state + QAPB_GAMMA * ((unsigned long long)gl + 1ULL));
    int32_t t = 0;
    if (__any_sync(gmask, (r > last_ok) || force_seq)) {
        unsigned long long st = state;
        for (int k = 0; k < G; ++k) {
            const int32_t v = (int32_t)(lo + (long long)randbelow_seq(st, span));
            if (k == gl) t = v;
        }
        state = st;
    } else {
        t = (int32_t)(lo + (long long)(r % span));
        state += QAPB_GAMMA * (unsigned long long)G;
    }
    return t;
}

// SYMM: 1 = both matrices symmetric (one product per entry), 0 = the general two-product update.
// NOTABU: 2opt instantiation (no tabu state at all).  REC: trail / cells / caller-provided tenures.
// G: lanes per search.
template <int SYMM, bool NOTABU, bool REC, int G>
#ifndef QAPB_WARP_MINB
#define QAPB_WARP_MINB 1
#endif
__global__ void __launch_bounds__(256, QAPB_WARP_MINB) qap_search_warp_kernel(const SearchParams P)
{
    typedef WkLay<G> LY;
    constexpr bool FULLSYM = SYMM == 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, gl = lane & (G - 1);
    // Every warp collective names the FULL warp (a run-time sub-warp mask makes the compiler guard each shuffle with
    // MATCH / VOTE convergence checks); with G = 16 the two searches of a warp therefore run in lockstep, shuffles
    // and votes segmented by their width argument.
    constexpr unsigned gmask = 0xffffffffu;
    const int n = P.n, nb = P.nb, npad = P.npad, noff = P.noff;

    // shared by the searches of the CTA: chunk slot of every unit and its inverse, then the address table:
    // entry [y][x] = words of M[x][y] and M[y][x]
    unsigned *sTab = reinterpret_cast<unsigned *>(smem_raw);
    unsigned char *sSlot = reinterpret_cast<unsigned char *>(sTab + G * G);  // [I * 8 + J] -> slot
    unsigned char *sUnit = sSlot + 64;                                        // [slot] -> I | J << 4, 0xff = none
    for (int t = threadIdx.x; t < 64; t += blockDim.x) {
        const int a = t >> 3, b2 = t & 7;
        sUnit[t] = 0xff;
        sSlot[t] = (a < b2 && b2 < nb) ? (unsigned char)wk_unit_slot(a, b2, nb) : 0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 64; t += blockDim.x) {
        const int a = t >> 3, b2 = t & 7;
        if (a < b2 && b2 < nb) sUnit[sSlot[t]] = (unsigned char)(a | (b2 << 4));
    }
    for (int e = threadIdx.x; e < G * G; e += blockDim.x) {
        const int y = e / G, x = e - y * G;
        sTab[e] = (x != y && x < npad && y < npad) ? wk_pair_words<G>(x, y, sSlot) : 0u;
    }
    __syncthreads();

    // Two searches per warp (G = 16): both halves must stay in step until the warp is done.  A half without a search
    // of its own (odd batch) runs a clone of the last one and writes nothing, and a search that runs out of
    // admissible moves goes on INERT: it keeps executing the iteration on a dummy move (0, 1) -- every address stays
    // valid, its matrix is garbage from then on -- while its results (costs, permutations, step count) are frozen.
    constexpr bool HALF = G == 16;
    const int b_raw = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 / G) + lane / G;
    if (b_raw - lane / G >= P.batch) return;  // whole warps only
    const bool ghost = b_raw >= P.batch;
    const int b = ghost ? P.batch - 1 : b_raw;
    int32_t *sW = reinterpret_cast<int32_t *>(smem_raw) + LY::TAB + ((threadIdx.x >> 5) * (32 / G) + lane / G) * LY::TOTAL;
    int32_t *sM = sW + LY::M;
    int32_t *sDG = sW + LY::DG;
    int32_t *xp = sW + LY::XP;
    int32_t *sP = sW + LY::P;
    Vecs V;
    V.A = sW + LY::A; V.B = sW + LY::B; V.C = sW + LY::C; V.E = sW + LY::E; V.HI = sW + LY::HI; V.HJ = sW + LY::HJ;
    V.H = V.ColR = V.ColS = V.TR = V.TS = V.XR = V.XS = nullptr;

    const int32_t *__restrict__ F = P.F;
    const int32_t *__restrict__ FT = P.FT;
    const int32_t *__restrict__ D = P.D;
    const int32_t *__restrict__ DT = P.DT;
    const int32_t MAXV = 0x7fffffff;
    const int32_t PADV = 1 << 25;
    const int one = P.one, sixteen = P.sixteen;
    const bool tabu = !NOTABU && P.mode == MODE_TABU;
    const int iters = P.iterations;

    // ---------------------------------------------------------------- setup
    const bool loc = gl < n;          // this lane is a location
    const int xu = gl & 3;
    // ---- start permutation and stream state (rng.py:62-70, core.py:81-87; what qap_start_kernel does for the
    // CTA-wide kernels): the n - 1 shuffle draws one per lane, the swaps through shuffles; a draw that randbelow
    // would reject makes every lane replay the exact sequential rule
    int my_p = 0;
    unsigned long long rstate = 0ULL;
    if (P.rng) {
        const unsigned long long seed =
            P.seeds ? P.seeds[b] : mix64(P.master_seed + QAPB_GAMMA * (P.first_index + (unsigned long long)b + 1ULL));
        int reject = P.force_seq_rng;
        unsigned jv = 0;  // lane k: the draw for position i = n - 1 - k
        if (gl < n - 1) {
            const unsigned long long bound = (unsigned long long)(n - gl);
            const unsigned long long r = mix64(seed + QAPB_GAMMA * ((unsigned long long)gl + 1ULL));
            if (r > ~0ULL - (0ULL - bound) % bound) reject = 1;
            jv = (unsigned)(r % bound);
        }
        reject = __any_sync(gmask, reject);
        my_p = loc ? gl : 0;
        unsigned long long st = seed;
        for (int i = n - 1; i >= 1; --i) {
            const int j = reject ? (int)randbelow_seq(st, (unsigned long long)i + 1ULL) : (int)__shfl_sync(gmask, jv, n - 1 - i, G);
            const int vi = __shfl_sync(gmask, my_p, i, G), vj = __shfl_sync(gmask, my_p, j, G);
            my_p = gl == i ? vj : gl == j ? vi : my_p;
        }
        rstate = reject ? st : seed + QAPB_GAMMA * (unsigned long long)(n - 1);
    } else {
        my_p = loc ? (int)P.perms[(size_t)b * n + gl] : 0;
    }
    V.A[gl] = 0; V.B[gl] = 0; V.C[gl] = 0; V.E[gl] = 0;
    sP[gl] = my_p;
    if (REC && P.cells && !ghost) {
        int64_t *cz = P.cells + (size_t)b * n * n;
        for (int i = gl; i < n * n; i += G) cz[i] = 0;
    }

    // off-diagonal unit of this lane: the one whose chunk slot (wk_unit_slot) is the lane index
    const bool own = sUnit[gl] != 0xff;
    const int I = own ? (sUnit[gl] & 15) : 0, J = own ? (sUnit[gl] >> 4) : 1;
    // diagonal-block pairs gl and gl + G (pair pp of block Bk: (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)), state in
    // this lane's slots sDG[q*2G + gl] = M[i][j], sDG[q*2G + G + gl] = M[j][i]
    int di[2], dj[2];
    bool dalive[2];
    int32_t dexp[2] = {0, 0};  // expiry iteration of the pair (cells[i][j]); 0 = never tabu
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int idx = gl + G * q;
        const int Bk = idx / 6, pp = idx - 6 * Bk;
        const int u = pp < 3 ? 0 : pp < 5 ? 1 : 2;
        const int v = pp < 3 ? pp + 1 : pp < 5 ? pp - 1 : 3;
        di[q] = 4 * Bk + u; dj[q] = 4 * Bk + v;
        dalive[q] = idx < 6 * nb && dj[q] < n;
        if (!dalive[q]) { di[q] = 0; dj[q] = 1; }
    }

    // ---- the placement matrix of the start (what qap_build_m_whole_kernel does for the CTA-wide kernels):
    //   S[a][b] = sum_k D0[a][k] F0[p_b][p_k] + D0[k][a] F0[p_k][p_b]
    //   M[i][j] = S[i][j] + D0[i][j] (F0[p_i][p_j] + F0[p_j][p_i]) + dd[i] fd[p_j],   h[i] = S[i][i] + dd[i] fd[p_i]
    // with the gathered flow matrix staged in the (still unused) unit slots: first Gm[k][j] = F0[p_j][p_k] for the
    // first sum, then its transpose for the second (both matrices symmetric: twice the first sum).
    unsigned tb = 0xffffu, deadm = 0xffffu;  // pairs that are tabu now (pad slots permanently set: deadm)
    int32_t mexp = MAXV;                     // earliest expiry among the clearable bits
    int4 *myM = reinterpret_cast<int4 *>(sM) + gl;   // row w of this lane's unit: myM[w * G], rotated by w
    // The unit streams from its shared-memory slot through these registers once per pass.  (Keeping it in registers
    // and moving only the ~13 units that touch block R or S of a move saves nothing: a predicated 128-bit access of
    // 13 scattered lanes costs 3.4 of the 4 wavefronts of a full-warp one, and as `if` bodies the flush and the
    // reload are divergent regions on the serial path.)
    int32_t U[4][4], L[4][4];
    int32_t h = 0;
    {
        int32_t *sG = sM;  // G x G words
        int32_t dx[2] = {0, 0}, dy[2] = {0, 0};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) { U[u][v] = 0; L[u][v] = 0; }
        __syncwarp(gmask);
#pragma unroll 1
        for (int phase = 0; phase < (FULLSYM ? 1 : 2); ++phase) {
            // phase 0: buffer[k][j] = F0[p_j][p_k], left factor D0[a][k] (rows of D^T); phase 1: the transposes
            const int32_t *__restrict__ lhs = phase == 0 ? DT : D;
            if (phase == 1) __syncwarp(gmask);
            for (int k = 0; k < G; ++k) {
                int32_t g = 0;
                if (loc && k < n) g = phase == 0 ? F[my_p * npad + sP[k]] : F[sP[k] * npad + my_p];
                sG[k * G + gl] = g;
            }
            __syncwarp(gmask);
            for (int k = 0; k < n; ++k) {
                int32_t aI[4], aJ[4], gI[4], gJ[4];
                ld_vec4(lhs + k * npad, I, aI); ld_vec4(lhs + k * npad, J, aJ);
                ld_vec4(sG + k * G, I, gI); ld_vec4(sG + k * G, J, gJ);
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        U[u][v] += aI[u] * gJ[v];
                        L[v][u] += aJ[v] * gI[u];
                    }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int32_t li = lhs[k * npad + di[q]], lj = lhs[k * npad + dj[q]];
                    dx[q] += li * sG[k * G + dj[q]];
                    dy[q] += lj * sG[k * G + di[q]];
                }
                h += lhs[k * npad + (loc ? gl : 0)] * sG[k * G + gl];
            }
        }
        // direct and diagonal terms (the buffer holds F0[p_k][p_j] at [k][j], or its transpose: the sum of
        // the two orientations is the same), pads
        const int32_t two = FULLSYM ? 2 : 1;
        unsigned dead = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int i = 4 * I + u, j = 4 * J + v;
                if (i >= n || j >= n || !own) {
                    dead |= 1u << (u * 4 + v);
                    U[u][v] = PADV; L[v][u] = PADV;
                } else {
                    const int32_t fs = sG[i * G + j] + sG[j * G + i];
                    U[u][v] = two * U[u][v] + D[i * npad + j] * fs + P.dd[i] * P.fd[sP[j]];
                    L[v][u] = two * L[v][u] + D[j * npad + i] * fs + P.dd[j] * P.fd[sP[i]];
                }
            }
        tb = dead;
        deadm = dead;
#pragma unroll
        for (int q = 0; q < 16; ++q) xp[gl * 16 + q] = ((dead >> q) & 1u) ? MAXV : 0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            int32_t x = PADV, y = PADV;
            if (dalive[q]) {
                const int i = di[q], j = dj[q];
                const int32_t fs = sG[i * G + j] + sG[j * G + i];
                x = two * dx[q] + D[i * npad + j] * fs + P.dd[i] * P.fd[sP[j]];
                y = two * dy[q] + D[j * npad + i] * fs + P.dd[j] * P.fd[sP[i]];
            }
            sDG[q * 2 * G + gl] = x;
            sDG[q * 2 * G + G + gl] = y;
        }
        h = loc ? two * h + P.dd[gl] * P.fd[my_p] : 0;
    }
    V.HI[gl] = 4 * xu - 16 * h;
    V.HJ[gl] = xu - 16 * h;
    __syncwarp(gmask);  // (the staged flow matrix has been read: its region now takes the unit slots)
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // position k of a chunk holds element (k - u) & 3 of its row
        myM[u * G] = make_int4(U[u][(0 - u) & 3], U[u][(1 - u) & 3], U[u][(2 - u) & 3], U[u][(3 - u) & 3]);
        myM[(4 + u) * G] = make_int4(L[(0 - u) & 3][u], L[(1 - u) & 3][u], L[(2 - u) & 3][u], L[(3 - u) & 3][u]);
    }
    __syncwarp(gmask);

    long long cost;  // _kernels.pyx:18-24, int64, including the diagonal products
    {
        long long part = 0;
        if (loc) {
            for (int j = 0; j < n; ++j) {
                const int pj = sP[j];
                part += (j == gl) ? (long long)P.fd[my_p] * P.dd[gl] : (long long)F[my_p * npad + pj] * D[gl * npad + j];
            }
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) part += __shfl_xor_sync(gmask, part, off, G);
        cost = part;
    }
    long long best_cost = cost;
    int32_t thr = 0;  // best_cost - cost, clamped; aspiration <=> delta < thr  (_kernels.pyx:162)
    int best_p = my_p;
    int steps_done = 0, stopped = 0;
    const unsigned long long span = (unsigned long long)(P.ten_hi - P.ten_lo + 1);
    const unsigned long long last_ok = (tabu && P.rng) ? ~0ULL - (0ULL - span) % span : 0ULL;
    int32_t my_ten = 0;
    // entry of moved location y: table word y * G + gl.  (A 32-bit shared-window address kept in a register: from
    // the pointer the compiler re-derives the window base with S2UR SR_CgaCtaId in every iteration.)
    unsigned tab_sa = (unsigned)__cvta_generic_to_shared(sTab + gl);
    asm volatile("" : "+r"(tab_sa));

    bool inert = false;  // (G = 16) stopped early: takes part in the warp-wide reductions only
    for (int c = 1; c <= iters; ++c) {
        int32_t my_d = MAXV;
        unsigned my_key = 0xffffffffu;
        int my_which = 0, my_slot = 0;  // 0: the off-diagonal unit, 1 / 2: diagonal pair q = 0 / 1
        if (tabu && ((c - 1) & (G - 1)) == 0) {
            if (P.rng) my_ten = warp_tenure_chunk<G>(gmask, rstate, span, last_ok, P.ten_lo, P.force_seq_rng, gl);
            else if (REC) my_ten = (c - 1 + gl < iters) ? (int32_t)P.tenures[(size_t)b * iters + (c - 1 + gl)] : 0;
        }
        // ---------------- pass: rank-2 update of the previous move (the difference vectors are zero at its
        // two locations and before the first move), delta, admissibility, first minimum
        {
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // position k of a chunk holds element (k - u) & 3 of its row
                const int4 a = myM[u * G];
                const int4 l = myM[(4 + u) * G];
                const int32_t av[4] = {a.x, a.y, a.z, a.w}, lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
                for (int v = 0; v < 4; ++v) { U[u][v] = av[(v + u) & 3]; L[v][u] = lv[(v + u) & 3]; }
            }
            int32_t aI[4], bI[4], aJ[4], bJ[4];
            ld_vec4(V.A, I, aI); ld_vec4(V.B, I, bI); ld_vec4(V.A, J, aJ); ld_vec4(V.B, J, bJ);
            if (FULLSYM) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        U[u][v] += aI[u] * bJ[v];
                        L[v][u] += aJ[v] * bI[u];
                    }
            } else {
                int32_t cI[4], eI[4], cJ[4], eJ[4];
                ld_vec4(V.C, I, cI); ld_vec4(V.E, I, eI); ld_vec4(V.C, J, cJ); ld_vec4(V.E, J, eJ);
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        U[u][v] += aI[u] * bJ[v] + cI[u] * eJ[v];
                        L[v][u] += aJ[v] * bI[u] + cJ[v] * eI[u];
                    }
            }
            // back to the slot (the lanes of the fix-ups read the entries on rows / columns r,s of the coming move
            // there): stored here, the unit is off the serial path behind the argmin
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // position k of a chunk holds element (k - u) & 3 of its row
                myM[u * G] = make_int4(U[u][(0 - u) & 3], U[u][(1 - u) & 3], U[u][(2 - u) & 3], U[u][(3 - u) & 3]);
                myM[(4 + u) * G] = make_int4(L[(0 - u) & 3][u], L[(1 - u) & 3][u], L[(2 - u) & 3][u], L[(3 - u) & 3][u]);
            }
            int32_t dk;
            int sk;
            // (2opt: pad pairs carry 2^25 in both entries, so their keys lose against every real pair)
            unit_select<true, NOTABU>(U, L, NOTABU ? 0u : tb, I, J, thr, V, one, sixteen, dk, sk);
            my_d = dk;
            my_key = pair_key(4 * I + (sk >> 2), 4 * J + (sk & 3), 0);
            my_slot = sk;
            if (dk == MAXV || !own) { my_d = MAXV; my_key = 0xffffffffu; }
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            int32_t x = sDG[q * 2 * G + gl], y = sDG[q * 2 * G + G + gl];
            const int32_t ai = V.A[di[q]], bj = V.B[dj[q]], aj = V.A[dj[q]], bi = V.B[di[q]];
            x += ai * bj;
            y += aj * bi;
            if (!FULLSYM) {
                const int32_t ci = V.C[di[q]], ej = V.E[dj[q]], cj = V.C[dj[q]], ei = V.E[di[q]];
                x += ci * ej;
                y += cj * ei;
            }
            const int32_t hi = __shfl_sync(gmask, h, di[q], G), hj = __shfl_sync(gmask, h, dj[q], G);
            sDG[q * 2 * G + gl] = x;
            sDG[q * 2 * G + G + gl] = y;
            const int32_t d = x + y - hi - hj;
            const bool adm = dalive[q] & (NOTABU | (dexp[q] <= c) | (d < thr));
            const unsigned key = pair_key(di[q], dj[q], 0);
            const bool take = adm & ((d < my_d) | ((d == my_d) & (key < my_key)));  // (no short-circuit branches)
            my_d = take ? d : my_d;
            my_key = take ? key : my_key;
            my_which = take ? 1 + q : my_which;
        }
        // lexicographic minimum of (delta, key) over the search's lanes
        int32_t bd;
        unsigned bkey;
        if (HALF) {
            const bool up = lane >= 16;
            __syncwarp();
            const int32_t d0 = __reduce_min_sync(0xffffffffu, up ? MAXV : my_d);
            const int32_t d1 = __reduce_min_sync(0xffffffffu, up ? my_d : MAXV);
            bd = up ? d1 : d0;
            const unsigned kk = my_d == bd ? my_key : 0xffffffffu;
            const unsigned k0 = __reduce_min_sync(0xffffffffu, up ? 0xffffffffu : kk);
            const unsigned k1 = __reduce_min_sync(0xffffffffu, up ? kk : 0xffffffffu);
            bkey = up ? k1 : k0;
        } else {
            bd = __reduce_min_sync(gmask, my_d);
            bkey = __reduce_min_sync(gmask, my_d == bd ? my_key : 0xffffffffu);
        }
        if (bd == MAXV && !inert) {  // no admissible move: premature stop (_kernels.pyx:168-170)
            stopped = 1;
            if (!HALF) break;
            inert = true;
        }
        const bool live = !(HALF && inert);
        const int r = live ? (int)(bkey >> 17) : 0, s = live ? (int)((bkey >> 1) & 0xffffu) : 1;
        if (live) cost += (long long)bd;
        const bool improved = live && cost < best_cost;
        if (improved) best_cost = cost;
        if (live) {
            thr = Acc<int32_t>::clamp_thr(best_cost - cost);
            steps_done = c;
        }
        const bool is_winner = live && my_key == bkey;
        const int pr = __shfl_sync(gmask, my_p, r, G), ps = __shfl_sync(gmask, my_p, s, G);
        const int32_t ten = tabu ? __shfl_sync(gmask, my_ten, (c - 1) & (G - 1), G) : 0;
        __syncwarp(gmask);  // -------------------------------------------- sync #1: every unit is in its slot

        // ---------------- publish: difference vectors of the move (old permutation), h', and the entries on
        // rows / columns r,s of M fixed in place by the lane of their location
        const int i = loc ? gl : 0;
        const int pi = loc ? my_p : 0;
        const bool mid = loc && (gl != r) && (gl != s);
        unsigned tr, ts;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tr) : "r"(tab_sa + (unsigned)r * (G * 4)));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ts) : "r"(tab_sa + (unsigned)s * (G * 4)));
        int32_t *p_ir = sW + (tr & 0xffffu), *p_ri = sW + (tr >> 16);
        int32_t *p_is = sW + (ts & 0xffffu), *p_si = sW + (ts >> 16);
        int32_t m_ir = 0, m_ri = 0, m_is = 0, m_si = 0;
        if (loc && gl != r) m_ir = *p_ir;   // (lane s: M[s][r])
        if (loc && gl != s) m_is = *p_is;   // (lane r: M[r][s])
        if (mid) { m_ri = *p_ri; m_si = *p_si; }
        int32_t kr = 0, ks = 0;  // corner terms, zero when both matrices are symmetric
        if (FULLSYM) {
            const int32_t Drs = D[r * npad + s], Fpspr = F[ps * npad + pr];
            const int32_t Dsi = D[s * npad + i], Dri = D[r * npad + i];
            const int32_t Fpspi = F[ps * npad + pi], Fprpi = F[pr * npad + pi];
            const int32_t a = mid ? Dsi - Dri : 0, bb = mid ? Fpspi - Fprpi : 0;
            const int32_t a2 = 2 * a, b2 = 2 * bb;
            V.A[gl] = -a2;
            V.B[gl] = bb;
            if (mid) {
                h -= a2 * bb;
                *p_ir = m_is + a2 * (Fpspr - Fpspi);        // M'[i][r] = M[i][s] + tR[i]
                *p_is = m_ir + a2 * (Fprpi - Fpspr);        // M'[i][s] = M[i][r] + tS[i]
                *p_ri = m_ri + b2 * (Dri - Drs);            // M'[r][i] = M[r][i] + xR[i]
                *p_si = m_si + b2 * (Drs - Dsi);            // M'[s][i] = M[s][i] + xS[i]
            }
        } else {
            const int32_t Drs = D[r * npad + s], Dsr = D[s * npad + r];
            const int32_t Fpspr = F[ps * npad + pr], Fprps = F[pr * npad + ps];
            const int32_t Dsi = D[s * npad + i], Dri = D[r * npad + i];
            const int32_t Dis = DT[s * npad + i], Dir = DT[r * npad + i];
            const int32_t Fpips = FT[ps * npad + pi], Fpipr = FT[pr * npad + pi];
            const int32_t Fpspi = F[ps * npad + pi], Fprpi = F[pr * npad + pi];
            const int32_t a = mid ? Dis - Dir : 0, cc = mid ? Dsi - Dri : 0;
            const int32_t bb = mid ? Fpips - Fpipr : 0, e = mid ? Fpspi - Fprpi : 0;
            const int32_t be = bb + e;
            V.A[gl] = -a;
            V.B[gl] = bb;
            V.C[gl] = -cc;
            V.E[gl] = e;
            kr = (Drs - Dsr) * Fpspr;
            ks = (Dsr - Drs) * Fprps;
            if (mid) {
                h -= a * bb + cc * e;
                *p_ir = m_is + a * (Fpspr - (Fpips + Fpspi)) + cc * Fprps;
                *p_is = m_ir + a * ((Fpipr + Fprpi) - Fprps) - cc * Fpspr;
                *p_ri = m_ri - Drs * bb - Dsr * e + Dri * be;
                *p_si = m_si + Dsr * bb + Drs * e - Dsi * be;
            }
        }
        // corners: M'[r][s] = h[r] + kr, h'[r] = M[r][s] + ks;  M'[s][r] = h[s] + ks, h'[s] = M[s][r] + kr
        if (loc && gl == r) { *p_is = h + kr; h = m_is + ks; }
        if (loc && gl == s) { *p_ir = h + ks; h = m_ir + kr; }
        V.HI[gl] = 4 * xu - 16 * h;
        V.HJ[gl] = xu - 16 * h;
        if (live) my_p = (gl == r) ? ps : (gl == s) ? pr : my_p;
        if (improved) best_p = my_p;

        // ---- the lane owning the winning pair: tabu memory (branch-free: a divergent region costs its reconvergence),
        // trail
        {
            const int32_t new_exp = (int32_t)(c + ten);
            const bool wu = is_winner && my_which == 0;   // the pair is in this lane's off-diagonal unit
            unsigned was = wu ? (tb >> my_slot) & 1u : 0u;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const bool wq = is_winner && my_which == 1 + q;
                was = (wq && dexp[q] > c) ? 1u : was;
                dexp[q] = (wq && tabu) ? new_exp : dexp[q];
            }
            const bool wt = wu && tabu;
            tb |= wt ? 1u << my_slot : 0u;
            mexp = wt ? min(mexp, new_exp) : mexp;
            sts32_if(wt, xp + gl * 16 + my_slot, new_exp);
            if (REC && P.tr_i && !ghost) {  // trail row (_kernels.pyx:182-187); was_tabu = cells[bi][bj] > c (:171)
                const size_t o = (size_t)b * iters + (c - 1);
                stg64_if(is_winner, P.tr_i + o, r);
                stg64_if(is_winner, P.tr_j + o, s);
                stg64_if(is_winner, P.tr_d + o, (int64_t)bd);
                if (P.tr_tabu) stg64_if(is_winner, P.tr_tabu + o, (int64_t)was);
            }
            if (REC && tabu && P.cells && !ghost) {  // cells[r][s] = c + t, cells[s][r] += 1 (_kernels.pyx:176-178)
                int64_t *cz = P.cells + (size_t)b * n * n;
                stg64_if(is_winner, cz + (size_t)r * n + s, (int64_t)c + ten);
                redg64_inc_if(is_winner, cz + (size_t)s * n + r);  // (a reduction without return: the load-add-store would wait for L2)
            }
        }
        // ---- tabu bits that expire at the next iteration are cleared here
        if (!NOTABU) {
            const bool due = own && c + 1 >= mexp;
            const unsigned live = tb & ~deadm;
            const bool one = (live & (live - 1u)) == 0u;  // one tabu pair in this unit (the usual case): one predicated load
            const int32_t e = lds32_if(due && one, xp + gl * 16 + (__ffs(live | 0x10000u) - 1), MAXV);
            const bool clr = due && one && e <= c + 1;
            tb = clr ? tb & ~live : tb;
            mexp = (due && one) ? (clr ? MAXV : e) : mexp;
            if (due && !one) expire_bits(tb, mexp, c + 1, xp + gl * 16);
        }
        __syncwarp(gmask);  // -------------------------------------------- sync #2
    }

    if (ghost) return;
    if (loc) {
        P.best[(size_t)b * n + gl] = best_p;
        P.cur[(size_t)b * n + gl] = my_p;
    }
    if (gl == 0) {
        P.best_cost[b] = best_cost;
        P.cur_cost[b] = cost;
        if (P.stopped) P.stopped[b] = stopped;
        if (P.steps) P.steps[b] = steps_done;
    }
}

}  // namespace qapb
