// search_hybrid.cuh -- the flagship search kernel (int32 state, n <= 256).
//
// Same algorithm and the same integers as qap_search_kernel (search_kernel.cuh).  The
// placement matrix M is split between the two on-chip memories of the SM:
//   * every off-diagonal thread keeps UR units (block pairs {(I,J),(J,I)}, 32 registers each)
//     in REGISTERS for the whole run, and
//   * a further US units per thread in SHARED MEMORY in a spill layout (row w of slot k of
//     thread t at ((k*8+w)*Toff + t)*16 bytes: every access is a conflict-free 128-bit
//     LDS/STS) that are streamed through registers once per iteration.
// The nb diagonal 4x4 blocks live in registers of the last DW warps (n <= 128) or, for the plans
// with shared-memory units, in shared memory with the last nb threads (DSM), so that every warp
// carries off-diagonal units.  The tabu triangle is a 16-bit mask per unit (pairs that are tabu
// now); expiry iterations live in an array that is only touched when a pair is set or expires
// (shared memory when it fits, else L2).  The split is chosen per instance on the host (qapb.cu,
// plan_hybrid): n = 100 runs two searches per SM with one register unit per thread (352 threads),
// n = 160 two searches per SM with 2 register + 2 shared-memory units per thread (256 threads),
// n = 256 one search per SM on 512 threads with 1024 units in registers and 992 in 124 KB of
// shared memory -- neither memory alone can hold the 256 KB of state of an n = 256 search.
//
// After move (r,s) the 4n entries on rows/columns r,s do not follow the rank-2 rule.  They
// are fixed at the start of the next pass from six n-vectors published between the two
// barriers of an iteration:
//   colR[i] = M[i][r], colS[i] = M[i][s]     dumped by the threads that own those columns
//   tR[i], tS[i]                             additive terms of  M'[i][r] = colS[i] + tR[i],
//                                                               M'[i][s] = colR[i] + tS[i]
//   xR[i], xS[i]                             additive terms of  M'[r][i] = M[r][i] + xR[i], ...
// with the corner values M'[r][s], M'[s][r] folded into tS[r], tR[s] (colR[r] = colS[s] = 0)
// and h[r], h[s] written by the thread that owns the winning pair.  r & 3 and s & 3 are
// uniform across the CTA, so register indices are selected with uniform switches.
#pragma once
#include "search_kernel.cuh"

namespace qapb {

// Shared-memory layout.  The n-vectors and the small reduction / tenure buffers sit at offsets that
// depend only on the size class NPADMAX (128 or 256), so the kernel addresses them with immediates
// (HYB_* below) instead of recomputing bases from the constant bank in every phase; the big,
// rarely-addressed regions (expiries, staged matrices, shared-memory units) follow at runtime offsets.
#define HYB_VEC(k, NPM) ((k) * 4 * (NPM))               /* A,C,B,E,H,ColR,ColS,TR,TS,XR,XS,P,HI,HJ: k = 0..13 */
#define HYB_REDD(NPM) (14 * 4 * (NPM))
#define HYB_REDK(NPM) (HYB_REDD(NPM) + 32 * 8 + 16)
#define HYB_MISC(NPM) (HYB_REDK(NPM) + 32 * 4)
#define HYB_TEN(NPM) (HYB_MISC(NPM) + 64)
#define HYB_FIXED_END(NPM) (HYB_TEN(NPM) + 4 * TENURE_CHUNK)

__host__ __device__ inline HybLayout make_hyb_layout(int npad, int nb, int toff, int us, int exp_in_smem,
                                                     int staged = 0, int symmetric = 1, int dsm = 0, int onewarp = 0)
{
    HybLayout L;
    const unsigned npm = onewarp ? 32u : npad <= 128 ? 128u : 256u;
    L.offA = HYB_VEC(0, npm); L.offC = HYB_VEC(1, npm); L.offB = HYB_VEC(2, npm); L.offE = HYB_VEC(3, npm);
    L.offH = HYB_VEC(4, npm); L.offColR = HYB_VEC(5, npm); L.offColS = HYB_VEC(6, npm); L.offTR = HYB_VEC(7, npm);
    L.offTS = HYB_VEC(8, npm); L.offXR = HYB_VEC(9, npm); L.offXS = HYB_VEC(10, npm); L.offP = HYB_VEC(11, npm);
    L.offJ = HYB_VEC(12, npm);
    L.offRedD = HYB_REDD(npm); L.offRedK = HYB_REDK(npm); L.offMisc = HYB_MISC(npm); L.offTen = HYB_TEN(npm);
    unsigned o = align16(HYB_FIXED_END(npm));
    L.offExp = o;
    if (exp_in_smem) o += 64u * (unsigned)(nb * (nb - 1) / 2 + nb);  // tabu expiry per (unit, slot)
    o = align16(o);
    L.offM = o; o += (unsigned)us * 8u * (unsigned)toff * 16u;
    L.offTB = o; o += align16(4u * (unsigned)us * (unsigned)toff);
    L.offMX = o; o += align16(4u * (unsigned)us * (unsigned)toff);
    L.offDG = o;   // diagonal blocks in shared memory (DSM plans): 16 words + mask + earliest expiry each
    if (dsm) o += 64u * (unsigned)nb + align16(8u * (unsigned)nb);
    const unsigned m16 = staged ? align16(2u * (unsigned)npad * (unsigned)npad) : 0u;
    L.offD16 = o; o += m16;
    L.offF16 = o; o += m16;
    L.offDT16 = o; o += symmetric ? 0u : m16;
    L.offFT16 = o; o += symmetric ? 0u : m16;
    L.total = align16(o);
    return L;
}

struct Vecs {
    int32_t *A, *C, *B, *E, *H, *ColR, *ColS, *TR, *TS, *XR, *XS;
    int32_t *HI, *HJ;  // packed-key forms of h: HI[i] = -16 h[i] + 4 (i & 3), HJ[i] = -16 h[i] + (i & 3)
};

__device__ __forceinline__ void st_vec4(int32_t *arr, int blk, int32_t a, int32_t b, int32_t c, int32_t d)
{
    reinterpret_cast<int4 *>(arr)[blk] = make_int4(a, b, c, d);
}

// One unit from the row-major M of qap_build_m_kernel; dead = mask of pad pairs.  Pad entries are
// set to `padv`: large enough that a pad pair never aspirates, small enough that its packed key
// 16 delta + slot stays below 2^31 (2^25 with packed keys, where |M|, |h| < 2^25 is host-proven).
__device__ __forceinline__ void load_unit(const int32_t *__restrict__ Mi, int npad, int n, int I, int J,
                                          int32_t (&U)[4][4], int32_t (&L)[4][4], unsigned &dead, int32_t padv)
{
    dead = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int4 a = *reinterpret_cast<const int4 *>(Mi + (size_t)(4 * I + u) * npad + 4 * J);
        const int4 c = *reinterpret_cast<const int4 *>(Mi + (size_t)(4 * J + u) * npad + 4 * I);
        U[u][0] = a.x; U[u][1] = a.y; U[u][2] = a.z; U[u][3] = a.w;
        L[u][0] = c.x; L[u][1] = c.y; L[u][2] = c.z; L[u][3] = c.w;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (4 * I + u >= n || 4 * J + v >= n) {
                dead |= 1u << (u * 4 + v);
                if (I != J || u != v) { U[u][v] = padv; L[v][u] = padv; }
            }
}

#define QAPB_SWITCH4(idx, BODY)            \
    switch (idx) {                         \
        case 0: { constexpr int q = 0; BODY } break; \
        case 1: { constexpr int q = 1; BODY } break; \
        case 2: { constexpr int q = 2; BODY } break; \
        default: { constexpr int q = 3; BODY } break; \
    }

// ---- one off-diagonal unit: rank-2 update, then rows / columns r,s of the previous move --------
template <bool SYM>
__device__ __forceinline__ void unit_update(int32_t (&U)[4][4], int32_t (&L)[4][4], int Ik, int Jk, int R, int S,
                                            int ru, int su, const Vecs &V)
{
    int32_t aI[4], bI[4], aJ[4], bJ[4];
    ld_vec4(V.A, Ik, aI); ld_vec4(V.B, Ik, bI); ld_vec4(V.A, Jk, aJ); ld_vec4(V.B, Jk, bJ);
    // V.A and V.C hold the NEGATED difference vectors, so the update is a plain multiply-add
    if (SYM) {  // a is pre-doubled: a == c, b == e
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                U[u][v] += aI[u] * bJ[v];
                L[v][u] += aJ[v] * bI[u];
            }
    } else {
        int32_t cI[4], eI[4], cJ[4], eJ[4];
        ld_vec4(V.C, Ik, cI); ld_vec4(V.E, Ik, eI); ld_vec4(V.C, Jk, cJ); ld_vec4(V.E, Jk, eJ);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                U[u][v] += aI[u] * bJ[v] + cI[u] * eJ[v];
                L[v][u] += aJ[v] * bI[u] + cJ[v] * eI[u];
            }
    }
    // Rows / columns r and s.  Block row I == R holds row r in U and column r in L; block column
    // J == R holds row r in L and column r in U (I == R and J == R exclude each other).  r & 3 is
    // uniform, so the register index is chosen by a uniform switch *outside* the per-thread test:
    // one divergent region per moved location instead of two.
    {
        const bool hI = Ik == R, hJ = Jk == R;
        if (hI | hJ) {
            const int o = hI ? Jk : Ik;
            const int fI = hI ? 1 : 0, fJ = hJ ? 1 : 0;  // row increments as IMADs (FMA pipe), not SEL + IADD
            int32_t x[4], cs[4], t[4];
            ld_vec4(V.XR, o, x); ld_vec4(V.ColS, o, cs); ld_vec4(V.TR, o, t);
            QAPB_SWITCH4(ru, {
_Pragma("unroll")
                for (int w = 0; w < 4; ++w) {
                    const int32_t nv = cs[w] + t[w];
                    U[q][w] += x[w] * fI;
                    L[w][q] = hI ? nv : L[w][q];
                    L[q][w] += x[w] * fJ;
                    U[w][q] = hJ ? nv : U[w][q];
                }
            })
        }
    }
    {
        const bool hI = Ik == S, hJ = Jk == S;
        if (hI | hJ) {
            const int o = hI ? Jk : Ik;
            const int fI = hI ? 1 : 0, fJ = hJ ? 1 : 0;
            int32_t x[4], cr[4], t[4];
            ld_vec4(V.XS, o, x); ld_vec4(V.ColR, o, cr); ld_vec4(V.TS, o, t);
            QAPB_SWITCH4(su, {
_Pragma("unroll")
                for (int w = 0; w < 4; ++w) {
                    const int32_t nv = cr[w] + t[w];
                    U[q][w] += x[w] * fI;
                    L[w][q] = hI ? nv : L[w][q];
                    L[q][w] += x[w] * fJ;
                    U[w][q] = hJ ? nv : U[w][q];
                }
            })
        }
    }
}

// ---- delta, admissibility (_kernels.pyx:162), first minimum of one off-diagonal unit -----------
// The ALU pipe (IADD3 / ISETP / IMNMX, half rate) is the busiest pipe of the pass, so the first
// add of each delta and the (delta, slot) packing are multiplications by the runtime constants
// 1 and 16: they issue as IMAD on the FMA pipe.  PACKED: |delta| < 2^27 (host-proven), key =
// delta*16 + slot orders by (delta, slot), so the running first-minimum is one predicated
// IMNMX per pair in four independent chains.
// km = min(km, kd) if the pair is admissible: its tabu bit is clear, or kd < thr16 (aspiration).
// Written in PTX so that it is LOP3 (bit -> predicate) + ISETP.LT.OR + a predicated VIMNMX.
template <int BIT>
__device__ __forceinline__ void admissible_min(int32_t &km, int32_t kd, unsigned tbk, int32_t thr16)
{
    asm("{\n\t"
        ".reg .pred p, q;\n\t"
        ".reg .b32 t;\n\t"
        "and.b32 t, %2, %3;\n\t"
        "setp.eq.u32 q, t, 0;\n\t"
        "setp.lt.or.s32 p, %1, %4, q;\n\t"
        "@p min.s32 %0, %0, %1;\n\t"
        "}"
        : "+r"(km)
        : "r"(kd), "r"(tbk), "n"(1u << BIT), "r"(thr16));
}

// ---- WIDE: unsigned 32-bit state, 64-bit deltas --------------------------------------------------
// Instances whose proven bound on |M| and |h| exceeds 2^31 but not 2^32, with non-negative entries (the
// tai*b shapes: 2.25e9 at n = 150), keep M and h as UNSIGNED 32-bit values -- every one of them is a
// non-negative cost, and all updates are exact modulo 2^32 -- in the same registers / shared memory as the
// int32 plans, so two searches still share an SM.  Only the delta of a pair, M[i][j] + M[j][i] - h[i] - h[j],
// which needs 34 bits, the aspiration threshold and the argmin are 64-bit.
template <bool WIDE> struct DeltaT { typedef int32_t type; };
template <> struct DeltaT<true> { typedef int64_t type; };
template <typename DT> __device__ __forceinline__ DT delta_max();
template <> __device__ __forceinline__ int32_t delta_max<int32_t>() { return 0x7fffffff; }
template <> __device__ __forceinline__ int64_t delta_max<int64_t>() { return 0x7fffffffffffffffLL; }
__device__ __forceinline__ int64_t wide_delta(int32_t u, int32_t l, int32_t hi, int32_t hj)
{
    return (int64_t)(uint32_t)u + (int64_t)(uint32_t)l - (int64_t)(uint32_t)hi - (int64_t)(uint32_t)hj;
}

// CH running first-minima (a 64-bit value and a slot each): one per block row where the registers allow it (one
// register unit per thread: tai150b 484 -> 502 G evals/s), one per pair of rows in the two-register-unit plans
template <int CH>
__device__ __forceinline__ void unit_select_wide(const int32_t (&U)[4][4], const int32_t (&L)[4][4], unsigned tbk, int Ik,
                                                 int Jk, int64_t thr, const Vecs &V, int64_t &dbest, int &sbest)
{
    static_assert(CH == 2 || CH == 4, "two or four chains");
    int32_t hI[4], hJ[4];
    ld_vec4(V.H, Ik, hI);
    ld_vec4(V.H, Jk, hJ);
    int64_t rd[4] = {delta_max<int64_t>(), delta_max<int64_t>(), delta_max<int64_t>(), delta_max<int64_t>()};
    int rs[4] = {0, 4, 8, 12};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int ch = CH == 4 ? u : (u >> 1) * 2;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t d = wide_delta(U[u][v], L[v][u], hI[u], hJ[v]);
            const bool adm = !(tbk & (1u << (u * 4 + v))) || (d < thr);
            if (adm && d < rd[ch]) { rd[ch] = d; rs[ch] = u * 4 + v; }
        }
    }
    if (CH == 4) {
        if (rd[1] < rd[0]) { rd[0] = rd[1]; rs[0] = rs[1]; }
        if (rd[3] < rd[2]) { rd[2] = rd[3]; rs[2] = rs[3]; }
    }
    if (rd[2] < rd[0]) { rd[0] = rd[2]; rs[0] = rs[2]; }
    dbest = rd[0];
    sbest = rs[0];
}

__device__ __forceinline__ void diag_select_wide(const int32_t (&U)[4][4], unsigned tbk, int Ik, int64_t thr, const Vecs &V,
                                                 int64_t &dbest, int &sbest)
{
    int32_t hI[4];
    ld_vec4(V.H, Ik, hI);
    dbest = delta_max<int64_t>();
    sbest = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = u + 1; v < 4; ++v) {
            const int64_t d = wide_delta(U[u][v], U[v][u], hI[u], hI[v]);
            const bool adm = !(tbk & (1u << (u * 4 + v))) || (d < thr);
            if (adm && d < dbest) { dbest = d; sbest = u * 4 + v; }
        }
}

template <bool PACKED, bool NOTABU>
__device__ __forceinline__ void unit_select(const int32_t (&U)[4][4], const int32_t (&L)[4][4], unsigned tbk, int Ik,
                                            int Jk, int32_t thr, const Vecs &V, int one, int sixteen,
                                            int32_t &dbest, int &sbest)
{
    const int32_t MAXV = 0x7fffffff;
    if (PACKED) {
        // Both pipes of an SMSP issue one warp instruction every two cycles, and the ALU pipe (IADD3 /
        // LOP3 / ISETP / VIMNMX / SEL) is the busy one in this pass.  The key of a pair,
        //   kd = 16 delta + slot = (16 U + HI[u]) + (16 L + HJ[v]),   HI = -16 h + 4u,  HJ = -16 h + v,
        // is therefore three IMADs (FMA pipe; the last one multiplies by the runtime constant 1), and
        // admissibility + running minimum are exactly three ALU instructions: LOP3 (tabu bit ->
        // predicate), ISETP.LT.OR (aspiration: kd < 16 thr <=> delta < thr), predicated VIMNMX.
        int32_t hi[4], hj[4];
        ld_vec4(V.HI, Ik, hi);
        ld_vec4(V.HJ, Jk, hj);
        const int32_t thr16 = max(thr, -(1 << 27)) * 16;  // |delta| < 2^27 (host-proven)
        int32_t km[4] = {MAXV, MAXV, MAXV, MAXV};
        if (NOTABU && tbk == 0) {
            // 2opt instantiation, no pad slot in this unit: the running minimum alone, one ALU instruction
            // per pair.  (Compiled out of the tabu kernels: there most warps would hold both kinds of
            // units and execute both paths, and the extra code costs them 2-8 %.)
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int32_t t1 = U[u][v] * sixteen + hi[u];
                    const int32_t t2 = L[v][u] * sixteen + hj[v];
                    km[u] = min(km[u], t1 * one + t2);
                }
            const int32_t m0 = min(min(km[0], km[1]), min(km[2], km[3]));
            dbest = m0 >> 4;
            sbest = m0 & 15;
            return;
        }
#define QAPB_PAIR(u, v)                                                             \
    {                                                                               \
        const int32_t t1 = U[u][v] * sixteen + hi[u];                               \
        const int32_t t2 = L[v][u] * sixteen + hj[v];                               \
        admissible_min<(u) * 4 + (v)>(km[u], t1 * one + t2, tbk, thr16);            \
    }
        QAPB_PAIR(0, 0) QAPB_PAIR(0, 1) QAPB_PAIR(0, 2) QAPB_PAIR(0, 3)
        QAPB_PAIR(1, 0) QAPB_PAIR(1, 1) QAPB_PAIR(1, 2) QAPB_PAIR(1, 3)
        QAPB_PAIR(2, 0) QAPB_PAIR(2, 1) QAPB_PAIR(2, 2) QAPB_PAIR(2, 3)
        QAPB_PAIR(3, 0) QAPB_PAIR(3, 1) QAPB_PAIR(3, 2) QAPB_PAIR(3, 3)
#undef QAPB_PAIR
        const int32_t m = min(min(km[0], km[1]), min(km[2], km[3]));
        dbest = (m == MAXV) ? MAXV : (m >> 4);
        sbest = m & 15;
    } else {
        int32_t hI[4], hJ[4];
        ld_vec4(V.H, Ik, hI);
        ld_vec4(V.H, Jk, hJ);
        int32_t rd[4];
        int rs[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            rd[u] = MAXV;
            rs[u] = u * 4;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int32_t d = (U[u][v] * one + L[v][u]) - hI[u] - hJ[v];
                const bool adm = !(tbk & (1u << (u * 4 + v))) || (d < thr);
                if (adm && d < rd[u]) { rd[u] = d; rs[u] = u * 4 + v; }
            }
        }
        if (rd[1] < rd[0]) { rd[0] = rd[1]; rs[0] = rs[1]; }
        if (rd[3] < rd[2]) { rd[2] = rd[3]; rs[2] = rs[3]; }
        if (rd[2] < rd[0]) { rd[0] = rd[2]; rs[0] = rs[2]; }
        dbest = rd[0];
        sbest = rs[0];
    }
}

// ---- diagonal block: update + fix-ups.  Per moved location: the column assignment, then the row increment
// (x[.] is zero at r and s, so the two locations do not disturb each other's corner values) -- two divergent
// regions per iteration instead of four: the pass of the diagonal warp is as long as an off-diagonal one.
template <bool SYM>
__device__ __forceinline__ void diag_update(int32_t (&U)[4][4], int Ik, int R, int S, int ru, int su, const Vecs &V)
{
    int32_t aI[4], bI[4];
    ld_vec4(V.A, Ik, aI); ld_vec4(V.B, Ik, bI);
    if (SYM) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (u != v) U[u][v] += aI[u] * bI[v];
    } else {
        int32_t cI[4], eI[4];
        ld_vec4(V.C, Ik, cI); ld_vec4(V.E, Ik, eI);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (u != v) U[u][v] += aI[u] * bI[v] + cI[u] * eI[v];
    }
    if (Ik == R) {
        int32_t cs[4], t[4], x[4];
        ld_vec4(V.ColS, Ik, cs); ld_vec4(V.TR, Ik, t); ld_vec4(V.XR, Ik, x);
        QAPB_SWITCH4(ru, {
_Pragma("unroll")
            for (int u = 0; u < 4; ++u) if (u != q) U[u][q] = cs[u] + t[u];
_Pragma("unroll")
            for (int v = 0; v < 4; ++v) if (v != q) U[q][v] += x[v];
        })
    }
    if (Ik == S) {
        int32_t cr[4], t[4], x[4];
        ld_vec4(V.ColR, Ik, cr); ld_vec4(V.TS, Ik, t); ld_vec4(V.XS, Ik, x);
        QAPB_SWITCH4(su, {
_Pragma("unroll")
            for (int u = 0; u < 4; ++u) if (u != q) U[u][q] = cr[u] + t[u];
_Pragma("unroll")
            for (int v = 0; v < 4; ++v) if (v != q) U[q][v] += x[v];
        })
    }
}

// The six pairs of a diagonal block.  PACKED: the keys of the off-diagonal units (16 delta + slot) in three
// independent chains of admissible_min; else plain deltas in one compare-and-select chain.
template <bool PACKED>
__device__ __forceinline__ void diag_select(const int32_t (&U)[4][4], unsigned tbk, int Ik, int32_t thr, const Vecs &V,
                                            int32_t &dbest, int &sbest)
{
    const int32_t MAXV = 0x7fffffff;
    if (PACKED) {
        int32_t hi[4], hj[4];
        ld_vec4(V.HI, Ik, hi);
        ld_vec4(V.HJ, Ik, hj);
        const int32_t thr16 = max(thr, -(1 << 27)) * 16;
        int32_t km[3] = {MAXV, MAXV, MAXV};
#define QAPB_DPAIR(u, v, ch) admissible_min<(u) * 4 + (v)>(km[ch], (U[u][v] + U[v][u]) * 16 + (hi[u] + hj[v]), tbk, thr16);
        QAPB_DPAIR(0, 1, 0) QAPB_DPAIR(0, 2, 1) QAPB_DPAIR(0, 3, 2)
        QAPB_DPAIR(1, 2, 0) QAPB_DPAIR(1, 3, 1) QAPB_DPAIR(2, 3, 2)
#undef QAPB_DPAIR
        const int32_t m = min(min(km[0], km[1]), km[2]);
        dbest = (m == MAXV) ? MAXV : (m >> 4);
        sbest = m & 15;
    } else {
        int32_t hI[4];
        ld_vec4(V.H, Ik, hI);
        dbest = MAXV;
        sbest = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = u + 1; v < 4; ++v) {
                const int32_t d = U[u][v] + U[v][u] - hI[u] - hI[v];
                const bool adm = !(tbk & (1u << (u * 4 + v))) || (d < thr);
                if (adm && d < dbest) { dbest = d; sbest = u * 4 + v; }
            }
    }
}

// ---- tabu bits of a unit: clear the ones whose expiry has been reached ------------------------
__device__ __forceinline__ void expire_bits(unsigned &tb, int32_t &mexp, int c, const int32_t *xp16)
{
    // one 128-bit load per block row that has a bit set (a loop over single bits serialises one
    // load latency per bit -- it was the straggler of the publish phase)
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

// SYMM: 0 = both matrices asymmetric (two products per entry in the rank-2 update), 1 = both symmetric,
// 2 = exactly one symmetric: the update is still ONE product per entry (D = D^T => a == c, so
// a_i b_j + c_i e_j = a_i (b_j + e_j); F = F^T => b == e), the publish phase uses the general formulas
// and stores the combined vector (P.symmetric: 2 = distance symmetric, 3 = flow symmetric).
// REC: the run may record a trail / the tabu memory `cells` (the single-run entries); the multi-start
// entries never do, and their instantiations leave that code out of the winner's serial chain.
// DD: no dedicated diagonal warps -- the nb diagonal blocks ride, two per thread (one in U, one in L:
// the register footprint of one off-diagonal unit), in the threads that follow the last off-diagonal
// unit.  n = 100: 300 + 13 threads = 10 warps instead of 11, which at 64 registers is what lets THREE
// searches share an SM.
// OW (n <= 32 with DD): the whole search is ONE warp -- 28 off-diagonal units and four lanes with two diagonal
// blocks each at n = 29..32 -- so the two block barriers of an iteration become warp barriers, the warp
// argmin is already the result, and 32 independent searches share an SM (size class 32 of the shared-memory
// layout: 5.6 KB per search).
template <int SYMM, bool PACKED, int UR, bool SMEMU, bool STG, int MAXREG, bool DSM = false, bool NOTABU = false,
          bool REC = true, bool DD = false, bool OW = false, bool WIDE = false, bool NP256 = false>
__global__ void __maxnreg__(MAXREG) qap_search_hybrid_kernel(const SearchParams P)
{
    static_assert(!OW || (DD && !STG), "one-warp searches: paired diagonal blocks, no staged matrices");
    static_assert(!WIDE || !PACKED, "64-bit deltas have no packed keys");
    typedef typename DeltaT<WIDE>::type delta_t;   // type of a delta, of the aspiration threshold and of the argmin value
    const delta_t MAXD = delta_max<delta_t>();
    static_assert(!DD || (UR == 1 && !SMEMU && !DSM), "paired diagonal blocks: one register unit per thread");
    constexpr bool SYM = SYMM != 0;       // single-product pass
    constexpr bool FULLSYM = SYMM == 1;   // symmetric closed forms in the publish phase, no transposes
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, W = T >> 5;
    const int b = blockIdx.x;
    const int n = P.n, nb = P.nb, npad = P.npad, noff = P.noff;
    const int Toff = P.toff;              // off-diagonal threads
    const int US = SMEMU ? P.us : 0;      // shared-memory units per thread (compiled out when none)
    const HybLayout &lay = P.hlay;
    int32_t *sM = reinterpret_cast<int32_t *>(smem_raw + lay.offM);
    unsigned *sTB = reinterpret_cast<unsigned *>(smem_raw + lay.offTB);
    int32_t *sMX = reinterpret_cast<int32_t *>(smem_raw + lay.offMX);
    constexpr int NPM = OW ? 32 : (SMEMU || NP256) ? 256 : 128;  // size class of the plan (host: make_hyb_layout: n > 128 <=> shared-memory units or NP256)
    Vecs V;
    V.A = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(0, NPM));
    V.C = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(1, NPM));
    V.B = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(2, NPM));
    V.E = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(3, NPM));
    V.H = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(4, NPM));
    V.ColR = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(5, NPM));
    V.ColS = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(6, NPM));
    V.TR = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(7, NPM));
    V.TS = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(8, NPM));
    V.XR = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(9, NPM));
    V.XS = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(10, NPM));
    int32_t *sP = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(11, NPM));
    V.HI = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(12, NPM));
    V.HJ = reinterpret_cast<int32_t *>(smem_raw + HYB_VEC(13, NPM));
    long long *sRed64 = reinterpret_cast<long long *>(smem_raw + HYB_REDD(NPM));
    int32_t *sRedD = reinterpret_cast<int32_t *>(smem_raw + HYB_REDD(NPM));
    unsigned *sRedK = reinterpret_cast<unsigned *>(smem_raw + HYB_REDK(NPM));
    long long *sMisc = reinterpret_cast<long long *>(smem_raw + HYB_MISC(NPM));
    int32_t *sTen = reinterpret_cast<int32_t *>(smem_raw + HYB_TEN(NPM));
    // expiry iteration per (unit, slot): shared memory when it fits, else the L2-resident workspace
    // (register-only plans always keep it in shared memory, so the pointer stays in the shared window)
    int32_t *xp = (!SMEMU || P.exp_in_smem) ? reinterpret_cast<int32_t *>(smem_raw + lay.offExp)
                                            : reinterpret_cast<int32_t *>(P.gT) + (size_t)b * P.gT_stride;

    const int32_t *__restrict__ F = P.F;
    const int32_t *__restrict__ FT = P.FT;
    const int32_t *__restrict__ D = P.D;
    const int32_t *__restrict__ DT = P.DT;
    const int32_t MAXV = 0x7fffffff;
    const int one = P.one, sixteen = P.sixteen;
    // pad entries: never the minimum, never aspirated (WIDE: 2^32 - 1 as an unsigned value, so that the delta
    // of a pad pair, 2 (2^32 - 1) - h[i] - h[j], stays positive: the host admits bounds up to 4.0e9 only)
    const int32_t PADV = WIDE ? (int32_t)0xFFFFFFFFu : PACKED ? (1 << 25) : (1 << 29);
    // STG: int16 copies of D, F (and their transposes when asymmetric) in shared memory, so the
    // publish phase between the barriers never waits on an L1/L2 miss
    const int16_t *sD16 = reinterpret_cast<const int16_t *>(smem_raw + lay.offD16);
    const int16_t *sF16 = reinterpret_cast<const int16_t *>(smem_raw + lay.offF16);
    const int16_t *sDT16 = FULLSYM ? sD16 : reinterpret_cast<const int16_t *>(smem_raw + lay.offDT16);
    const int16_t *sFT16 = FULLSYM ? sF16 : reinterpret_cast<const int16_t *>(smem_raw + lay.offFT16);
    auto ldD = [&](int a, int c2) -> int32_t { return STG ? (int32_t)sD16[a * npad + c2] : D[a * npad + c2]; };
    auto ldF = [&](int a, int c2) -> int32_t { return STG ? (int32_t)sF16[a * npad + c2] : F[a * npad + c2]; };
    auto ldDT = [&](int a, int c2) -> int32_t { return STG ? (int32_t)sDT16[a * npad + c2] : DT[a * npad + c2]; };
    auto ldFT = [&](int a, int c2) -> int32_t { return STG ? (int32_t)sFT16[a * npad + c2] : FT[a * npad + c2]; };
    if (STG) {
        int16_t *wD = reinterpret_cast<int16_t *>(smem_raw + lay.offD16);
        int16_t *wF = reinterpret_cast<int16_t *>(smem_raw + lay.offF16);
        for (int e = tid; e < npad * npad; e += T) { wD[e] = (int16_t)D[e]; wF[e] = (int16_t)F[e]; }
        if (!FULLSYM) {
            int16_t *wDT = reinterpret_cast<int16_t *>(smem_raw + lay.offDT16);
            int16_t *wFT = reinterpret_cast<int16_t *>(smem_raw + lay.offFT16);
            for (int e = tid; e < npad * npad; e += T) { wDT[e] = (int16_t)DT[e]; wFT[e] = (int16_t)FT[e]; }
        }
    }

    // ---------------------------------------------------------------- setup
    // start permutation, stream state, M and h come from qap_start_kernel / qap_build_m_kernel
    for (int i = tid; i < npad; i += T) {
        V.A[i] = 0; V.C[i] = 0; V.B[i] = 0; V.E[i] = 0;
        V.ColR[i] = 0; V.ColS[i] = 0; V.TR[i] = 0; V.TS[i] = 0; V.XR[i] = 0; V.XS[i] = 0;
        const int32_t h0 = reinterpret_cast<const int32_t *>(P.initH)[(size_t)b * npad + i];
        V.H[i] = h0;
        V.HI[i] = 4 * (i & 3) - 16 * h0;
        V.HJ[i] = (i & 3) - 16 * h0;
        sP[i] = P.perm32[(size_t)b * npad + i];
    }
    if (tid == 0) sMisc[4] = P.rng ? (long long)P.start_state[b] : 0LL;  // SplitMix64 state after the shuffle
    if (P.cells) {
        int64_t *cz = P.cells + (size_t)b * n * n;
        for (int i = tid; i < n * n; i += T) cz[i] = 0;
    }
    __syncthreads();

    long long cost;  // _kernels.pyx:18-24, int64, including the diagonal products
    {
        long long part = 0;
        for (int idx = tid; idx < n * n; idx += T) {
            int i = idx / n, j = idx - i * n;
            int pi = sP[i], pj = sP[j];
            part += (i == j) ? (long long)P.fd[pi] * P.dd[i] : (long long)ldF(pi, pj) * ldD(i, j);
        }
        cost = block_sum_i64(part, sRed64, tid, T);
        __syncthreads();
    }
    int my_pi = tid < n ? sP[tid] : 0;  // unit at location tid, kept in a register (T >= n by plan)
    const int32_t *__restrict__ Minit = reinterpret_cast<const int32_t *>(P.initM) + (size_t)b * npad * npad;

    // ---- unit ownership.  tb = mask of pairs that are tabu now (pads / non-pairs permanently
    // set, expiry MAXV), mexp = earliest expiry among the clearable bits.
    const bool offt = tid < Toff;
    // diagonal blocks: one per thread of the last warps in registers, or (DSM) in shared memory, owned by
    // the last nb threads of the CTA in addition to their off-diagonal units
    const bool diag = !DSM && !DD && tid >= Toff && (tid - Toff) < nb;
    // DD: thread noff + q carries diagonal blocks 2q (in U) and 2q + 1 (in L; absent when 2q + 1 == nb)
    // (I[0], J[0] = the two blocks, J[0] = -1 for an absent one; own[0] tells a carrier from an idle thread)
    const bool ddiag = DD && tid >= noff;
    const bool dsm_owner = DSM && tid >= T - nb;
    const int dsmI = T - 1 - tid;  // diagonal block of a DSM owner
    int32_t *sDG = reinterpret_cast<int32_t *>(smem_raw + lay.offDG);              // [nb][16]
    unsigned *sDGtb = reinterpret_cast<unsigned *>(smem_raw + lay.offDG) + 16 * nb;  // [nb]
    int32_t *sDGmx = reinterpret_cast<int32_t *>(sDGtb + nb);                        // [nb]
    constexpr int WHICH_DIAG = 1000;
    int I[UR], J[UR], uidv[UR];
    bool own[UR];
    int32_t U[UR][4][4], L[UR][4][4];
    unsigned tb[UR];
    int32_t mexp[UR];
#pragma unroll
    for (int k = 0; k < UR; ++k) {
        const int uid = tid + k * Toff;
        own[k] = offt && (uid < noff);
        I[k] = 0; J[k] = 0; uidv[k] = 0; tb[k] = 0xffffu; mexp[k] = MAXV;
        if (own[k]) { I[k] = P.unit_ij[uid] & 0xff; J[k] = P.unit_ij[uid] >> 8; uidv[k] = uid; }
        if (k == 0 && diag) { I[0] = tid - Toff; J[0] = I[0]; uidv[0] = noff + I[0]; own[0] = true; }
        if (DD && k == 0 && ddiag && 2 * (tid - noff) < nb) {
            int32_t tmp[4][4];
            unsigned deadA, deadB = 0xffffu;
            const int ddA = 2 * (tid - noff), ddB = ddA + 1 < nb ? ddA + 1 : -1;
            I[0] = ddA; J[0] = ddB; uidv[0] = noff + ddA; own[0] = true;
            load_unit(Minit, npad, n, ddA, ddA, U[0], tmp, deadA, PADV);
            deadA |= 0xF731u;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) L[0][u][v] = 0;
            if (ddB >= 0) {
                load_unit(Minit, npad, n, ddB, ddB, L[0], tmp, deadB, PADV);
                deadB |= 0xF731u;
            }
            tb[0] = deadA | (deadB << 16);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                xp[(noff + ddA) * 16 + q] = ((deadA >> q) & 1u) ? MAXV : 0;
                if (ddB >= 0) xp[(noff + ddB) * 16 + q] = ((deadB >> q) & 1u) ? MAXV : 0;
            }
        } else if (own[k]) {
            unsigned dead;
            load_unit(Minit, npad, n, I[k], J[k], U[k], L[k], dead, PADV);
            if (diag) dead |= 0xF731u;  // slots with u >= v are not pairs of a diagonal block
            tb[k] = dead;
#pragma unroll
            for (int q = 0; q < 16; ++q) xp[uidv[k] * 16 + q] = ((dead >> q) & 1u) ? MAXV : 0;
        }
    }
    if (dsm_owner) {
        int32_t Ud[4][4], Ld[4][4];
        unsigned dead;
        load_unit(Minit, npad, n, dsmI, dsmI, Ud, Ld, dead, PADV);
        dead |= 0xF731u;  // slots with u >= v are not pairs of a diagonal block
#pragma unroll
        for (int u = 0; u < 4; ++u) st_vec4(sDG + 16 * dsmI, u, Ud[u][0], Ud[u][1], Ud[u][2], Ud[u][3]);
        sDGtb[dsmI] = dead;
        sDGmx[dsmI] = MAXV;
#pragma unroll
        for (int q = 0; q < 16; ++q) xp[(noff + dsmI) * 16 + q] = ((dead >> q) & 1u) ? MAXV : 0;
    }
    if (SMEMU && offt) {
        for (int k2 = 0; k2 < US; ++k2) {
            const int uid = UR * Toff + k2 * Toff + tid;
            if (uid < noff) {
                int32_t Us[4][4], Ls[4][4];
                unsigned dead;
                const int Ik = P.unit_ij[uid] & 0xff, Jk = P.unit_ij[uid] >> 8;
                load_unit(Minit, npad, n, Ik, Jk, Us, Ls, dead, PADV);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    st_row(sM, k2 * 8 + u, Toff, tid, Us[u]);
                    st_row(sM, k2 * 8 + 4 + u, Toff, tid, Ls[u]);
                }
                sTB[k2 * Toff + tid] = dead;
                sMX[k2 * Toff + tid] = MAXV;
#pragma unroll
                for (int q = 0; q < 16; ++q) xp[uid * 16 + q] = ((dead >> q) & 1u) ? MAXV : 0;
            }
        }
    }
    __syncthreads();

    // ------------------------------------------------------------ iterations
    long long best_cost = cost;
    delta_t thr = 0;  // best_cost - cost, clamped; aspiration <=> delta < thr  (_kernels.pyx:162)
    const bool tabu = P.mode == MODE_TABU;
    const int iters = P.iterations;
    int steps_done = 0, stopped = 0;
    int64_t *best_out = P.best + (size_t)b * n;
    for (int i = tid; i < n; i += T) best_out[i] = sP[i];
    int R = -1, S = -1, ru = 0, su = 0;  // previous move (block and in-block indices)

    long long tacc[6] = {0, 0, 0, 0, 0, 0};
    // phase-cycle counters of CTA 0 (scripts/phase_time.py): compiled in only with -DQAPB_PHASE_TIMING,
    // the clock reads and their predicates cost ~3 % of the loop otherwise
#ifdef QAPB_PHASE_TIMING
    const bool timing = P.dbg != nullptr && b == 0 && (tid == 0 || tid == 128 || tid == Toff);
#else
    constexpr bool timing = false;
#endif
    for (int c = 1; c <= iters; ++c) {
        long long tA = 0, tB = 0, tC = 0, tD = 0, tE = 0, tF = 0;
        if (timing) tA = clock64();
        if (tabu && P.rng && ((c - 1) & (TENURE_CHUNK - 1)) == 0) {
            // the stream state lives in shared memory between refills (two registers less in the loop)
            unsigned long long st = (unsigned long long)sMisc[4];
            fill_tenure_chunk(st, P.ten_lo, P.ten_hi, P.force_seq_rng, sTen, sMisc, tid, T);
            if (tid == 0) sMisc[4] = (long long)st;
        }
        if (REC && tabu && !P.rng && ((c - 1) & (TENURE_CHUNK - 1)) == 0) {
            // caller-provided tenures: stage the next chunk, so that the owner of the winning pair reads
            // shared memory instead of waiting for L2 on the serial path (visible after barrier 1;
            // c + tenure is taken modulo 2^32 either way)
            const int64_t *src = P.tenures + (size_t)b * iters + (c - 1);
            const int m = min((int)TENURE_CHUNK, iters - (c - 1));
            for (int k = tid; k < m; k += T) sTen[k] = (int32_t)src[k];
        }

        // ---------------- pass: update + select over this thread's units
        delta_t my_d = MAXD;
        unsigned my_key = 0xffffffffu;
        int my_which = 0, my_slot = 0;  // which: register unit k, or UR + k2 for a shared-memory unit
#pragma unroll
        for (int k = 0; k < UR; ++k) {
            if (!own[k]) continue;
            delta_t dk;
            int sk;
            if (DD && ddiag) {
                // two diagonal blocks: U = block I (tabu bits 0..15), L = block J (bits 16..31)
                if (R >= 0) diag_update<SYM>(U[k], I[k], R, S, ru, su, V);
                if constexpr (WIDE) diag_select_wide(U[k], tb[k] & 0xffffu, I[k], thr, V, dk, sk); else diag_select<PACKED>(U[k], tb[k] & 0xffffu, I[k], thr, V, dk, sk);
                if (dk != MAXD) {
                    my_d = dk; my_key = pair_key(4 * I[k] + (sk >> 2), 4 * I[k] + (sk & 3), 0); my_slot = sk;
                }
                if (J[k] >= 0) {
                    if (R >= 0) diag_update<SYM>(L[k], J[k], R, S, ru, su, V);
                    if constexpr (WIDE) diag_select_wide(L[k], tb[k] >> 16, J[k], thr, V, dk, sk); else diag_select<PACKED>(L[k], tb[k] >> 16, J[k], thr, V, dk, sk);
                    if (dk < my_d) {  // block J comes later in (i, j) order: strict
                        my_d = dk; my_key = pair_key(4 * J[k] + (sk >> 2), 4 * J[k] + (sk & 3), 0); my_slot = 16 + sk;
                    }
                }
                continue;
            }
            if (DD || I[k] != J[k]) {
                if (R >= 0) unit_update<SYM>(U[k], L[k], I[k], J[k], R, S, ru, su, V);
                if constexpr (WIDE) unit_select_wide<(UR == 1 && SMEMU) ? 4 : 2>(U[k], L[k], tb[k], I[k], J[k], thr, V, dk, sk); else unit_select<PACKED, NOTABU>(U[k], L[k], tb[k], I[k], J[k], thr, V, one, sixteen, dk, sk);
            } else {
                if (R >= 0) diag_update<SYM>(U[k], I[k], R, S, ru, su, V);
                if constexpr (WIDE) diag_select_wide(U[k], tb[k], I[k], thr, V, dk, sk); else diag_select<PACKED>(U[k], tb[k], I[k], thr, V, dk, sk);
            }
            if (dk != MAXD) {
                const unsigned key = pair_key(4 * I[k] + (sk >> 2), 4 * J[k] + (sk & 3), 0);
                if (dk < my_d || (dk == my_d && key < my_key)) { my_d = dk; my_key = key; my_which = k; my_slot = sk; }
            }
        }
        if (SMEMU && offt) {
#pragma unroll 1
            for (int k2 = 0; k2 < US; ++k2) {
                const int uid = UR * Toff + k2 * Toff + tid;
                if (uid >= noff) break;
                const int Ik = P.unit_ij[uid] & 0xff, Jk = P.unit_ij[uid] >> 8;
                int32_t Us[4][4], Ls[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    ld_row(sM, k2 * 8 + u, Toff, tid, Us[u]);
                    ld_row(sM, k2 * 8 + 4 + u, Toff, tid, Ls[u]);
                }
                if (R >= 0) {
                    unit_update<SYM>(Us, Ls, Ik, Jk, R, S, ru, su, V);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        st_row(sM, k2 * 8 + u, Toff, tid, Us[u]);
                        st_row(sM, k2 * 8 + 4 + u, Toff, tid, Ls[u]);
                    }
                }
                delta_t dk;
                int sk;
                if constexpr (WIDE) unit_select_wide<(UR == 1 && SMEMU) ? 4 : 2>(Us, Ls, sTB[k2 * Toff + tid], Ik, Jk, thr, V, dk, sk); else unit_select<PACKED, NOTABU>(Us, Ls, sTB[k2 * Toff + tid], Ik, Jk, thr, V, one, sixteen, dk, sk);
                if (dk != MAXD) {
                    const unsigned key = pair_key(4 * Ik + (sk >> 2), 4 * Jk + (sk & 3), 0);
                    if (dk < my_d || (dk == my_d && key < my_key)) { my_d = dk; my_key = key; my_which = UR + k2; my_slot = sk; }
                }
            }
        }
        if (dsm_owner) {
            int32_t Ud[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) ld_vec4(sDG + 16 * dsmI + 4 * u, 0, Ud[u]);
            if (R >= 0) {
                diag_update<SYM>(Ud, dsmI, R, S, ru, su, V);
#pragma unroll
                for (int u = 0; u < 4; ++u) st_vec4(sDG + 16 * dsmI, u, Ud[u][0], Ud[u][1], Ud[u][2], Ud[u][3]);
            }
            delta_t dk;
            int sk;
            if constexpr (WIDE) diag_select_wide(Ud, sDGtb[dsmI], dsmI, thr, V, dk, sk); else diag_select<PACKED>(Ud, sDGtb[dsmI], dsmI, thr, V, dk, sk);
            if (dk != MAXD) {
                const unsigned key = pair_key(4 * dsmI + (sk >> 2), 4 * dsmI + (sk & 3), 0);
                if (dk < my_d || (dk == my_d && key < my_key)) { my_d = dk; my_key = key; my_which = WHICH_DIAG; my_slot = sk; }
            }
        }

        if (timing) tB = clock64();
        delta_t bd = my_d;
        unsigned bkey = my_key;
        warp_argmin(bd, bkey);
        if (OW) {
            __syncwarp();  // ------------------------------------------------ sync #1 (one warp: the argmin is final)
        } else {
            delta_t *sRedT = reinterpret_cast<delta_t *>(sRedD);  // 32 x 8 bytes are reserved
            if (lane == 0) { sRedT[warp] = bd; sRedK[warp] = bkey; }
            __syncthreads();  // ------------------------------------------ sync #1
            bd = lane < W ? sRedT[lane] : MAXD;
            bkey = lane < W ? sRedK[lane] : 0xffffffffu;
            warp_argmin(bd, bkey);
        }
        if (bd == MAXD) {  // no admissible move: premature stop (_kernels.pyx:168-170)
            stopped = 1;
            break;
        }
        const int r = (int)(bkey >> 17), s = (int)((bkey >> 1) & 0xffffu);
        cost += (long long)bd;
        const bool improved = cost < best_cost;
        if (improved) best_cost = cost;
        thr = Acc<delta_t>::clamp_thr(best_cost - cost);
        steps_done = c;
        R = r >> 2; S = s >> 2; ru = r & 3; su = s & 3;
        // only the publish threads and the owner of the winning pair need the two units
        const bool is_winner = my_key == bkey;
        int pr = 0, ps = 0;
        if (tid < n || is_winner) { pr = sP[r]; ps = sP[s]; }
        if (timing) tC = clock64() + (pr & 0);

        // ---- owners of columns r and s publish them first (colR[r] = colS[s] = 0 by the diagonal lanes):
        // the owner of the winning pair then reads its corner values M[r][s] = colS[r], M[s][r] = colR[s]
        // back from shared memory instead of selecting registers by a run-time index
#pragma unroll
        for (int k = 0; k < UR; ++k) {
            if (!own[k]) continue;
            const int Ik = I[k], Jk = J[k];
            if (DD && ddiag) {
                const int ddA = Ik, ddB = Jk;
                if (ddA == R) {
                    QAPB_SWITCH4(ru, { st_vec4(V.ColR, ddA, q == 0 ? 0 : U[k][0][q], q == 1 ? 0 : U[k][1][q], q == 2 ? 0 : U[k][2][q], q == 3 ? 0 : U[k][3][q]); })
                }
                if (ddA == S) {
                    QAPB_SWITCH4(su, { st_vec4(V.ColS, ddA, q == 0 ? 0 : U[k][0][q], q == 1 ? 0 : U[k][1][q], q == 2 ? 0 : U[k][2][q], q == 3 ? 0 : U[k][3][q]); })
                }
                if (ddB == R) {
                    QAPB_SWITCH4(ru, { st_vec4(V.ColR, ddB, q == 0 ? 0 : L[k][0][q], q == 1 ? 0 : L[k][1][q], q == 2 ? 0 : L[k][2][q], q == 3 ? 0 : L[k][3][q]); })
                }
                if (ddB == S) {
                    QAPB_SWITCH4(su, { st_vec4(V.ColS, ddB, q == 0 ? 0 : L[k][0][q], q == 1 ? 0 : L[k][1][q], q == 2 ? 0 : L[k][2][q], q == 3 ? 0 : L[k][3][q]); })
                }
                continue;
            }
            if (DD || Ik != Jk) {
                // ONE uniform 16-way switch on (r & 3, s & 3) (a jump table: one indirect branch on the serial
                // path instead of two two-level trees), per-thread predicated 128-bit stores inside
#define QAPB_DUMP(a, b)                                                                                    \
    case (a) * 4 + (b):                                                                                    \
        if (Jk == R) st_vec4(V.ColR, Ik, U[k][0][a], U[k][1][a], U[k][2][a], U[k][3][a]);                  \
        if (Ik == R) st_vec4(V.ColR, Jk, L[k][0][a], L[k][1][a], L[k][2][a], L[k][3][a]);                  \
        if (Jk == S) st_vec4(V.ColS, Ik, U[k][0][b], U[k][1][b], U[k][2][b], U[k][3][b]);                  \
        if (Ik == S) st_vec4(V.ColS, Jk, L[k][0][b], L[k][1][b], L[k][2][b], L[k][3][b]);                  \
        break;
                switch (ru * 4 + su) {
                    QAPB_DUMP(0, 0) QAPB_DUMP(0, 1) QAPB_DUMP(0, 2) QAPB_DUMP(0, 3)
                    QAPB_DUMP(1, 0) QAPB_DUMP(1, 1) QAPB_DUMP(1, 2) QAPB_DUMP(1, 3)
                    QAPB_DUMP(2, 0) QAPB_DUMP(2, 1) QAPB_DUMP(2, 2) QAPB_DUMP(2, 3)
                    QAPB_DUMP(3, 0) QAPB_DUMP(3, 1) QAPB_DUMP(3, 2) QAPB_DUMP(3, 3)
                }
#undef QAPB_DUMP
            } else {
                if (Ik == R) {
                    QAPB_SWITCH4(ru, { st_vec4(V.ColR, Ik, q == 0 ? 0 : U[k][0][q], q == 1 ? 0 : U[k][1][q], q == 2 ? 0 : U[k][2][q], q == 3 ? 0 : U[k][3][q]); })
                }
                if (Ik == S) {
                    QAPB_SWITCH4(su, { st_vec4(V.ColS, Ik, q == 0 ? 0 : U[k][0][q], q == 1 ? 0 : U[k][1][q], q == 2 ? 0 : U[k][2][q], q == 3 ? 0 : U[k][3][q]); })
                }
            }
        }

        // ---------------- publish: difference vectors of the move (old permutation), additive
        // terms, h'[i] -- one location per thread
        if (tid < n) {
            const int i = tid;
            const int pi = my_pi;
            const bool mid = (i != r) && (i != s);
            if (improved) best_out[i] = (i == r) ? ps : (i == s) ? pr : pi;
            if (FULLSYM) {
                // D = D^T, F = F^T: a = c, b = e, and the closed forms collapse
                const int32_t Drs = ldD(r, s), Fpspr = ldF(ps, pr);
                const int32_t Dsi = ldD(s, i), Dri = ldD(r, i);
                const int32_t Fpspi = ldF(ps, pi), Fprpi = ldF(pr, pi);
                const int32_t a = mid ? Dsi - Dri : 0, bb = mid ? Fpspi - Fprpi : 0;
                const int32_t a2 = 2 * a, b2 = 2 * bb;
                V.A[i] = -a2;
                V.B[i] = bb;
                V.XR[i] = b2 * ((mid ? Dri : 0) - Drs);
                V.XS[i] = b2 * (Drs - (mid ? Dsi : 0));
                if (mid) {
                    const int32_t hn = V.H[i] - a2 * bb;
                    V.H[i] = hn;
                    if (PACKED) { V.HI[i] = 4 * (i & 3) - 16 * hn; V.HJ[i] = (i & 3) - 16 * hn; }
                    V.TR[i] = a2 * (Fpspr - Fpspi);
                    V.TS[i] = a2 * (Fprpi - Fpspr);
                } else if (i == r) {
                    V.TR[i] = 0;  // tS[r] is written by the owner of the pair
                } else {
                    V.TS[i] = 0;  // tR[s] is written by the owner of the pair
                }
            } else {
                const int32_t Drs = ldD(r, s), Dsr = ldD(s, r);
                const int32_t Fpspr = ldF(ps, pr), Fprps = ldF(pr, ps);
                const int32_t Dsi = ldD(s, i), Dri = ldD(r, i);
                const int32_t Dis = ldDT(s, i), Dir = ldDT(r, i);
                const int32_t Fpips = ldFT(ps, pi), Fpipr = ldFT(pr, pi);
                const int32_t Fpspi = ldF(ps, pi), Fprpi = ldF(pr, pi);
                const int32_t a = mid ? Dis - Dir : 0, cc = mid ? Dsi - Dri : 0;
                const int32_t bb = mid ? Fpips - Fpipr : 0, e = mid ? Fpspi - Fprpi : 0;
                const int32_t be = bb + e;
                if (SYMM == 2) {  // one symmetric matrix: combined vectors for the single-product update
                    V.A[i] = -(P.symmetric == 3 ? a + cc : a);
                    V.B[i] = P.symmetric == 2 ? bb + e : bb;
                } else {
                    V.A[i] = -a;
                    V.B[i] = bb;
                    V.C[i] = -cc;
                    V.E[i] = e;
                }
                V.XR[i] = -Drs * bb - Dsr * e + (mid ? Dri : 0) * be;
                V.XS[i] = Dsr * bb + Drs * e - (mid ? Dsi : 0) * be;
                if (mid) {
                    const int32_t hn = V.H[i] - (a * bb + cc * e);
                    V.H[i] = hn;
                    if (PACKED) { V.HI[i] = 4 * (i & 3) - 16 * hn; V.HJ[i] = (i & 3) - 16 * hn; }
                    V.TR[i] = a * (Fpspr - (Fpips + Fpspi)) + cc * Fprps;
                    V.TS[i] = a * ((Fpipr + Fprpi) - Fprps) - cc * Fpspr;
                } else if (i == r) {
                    V.TR[i] = 0;
                } else {
                    V.TS[i] = 0;
                }
            }
            my_pi = (i == r) ? ps : (i == s) ? pr : pi;
        }
        if (timing) tD = clock64();
        // ---- the thread owning the winning pair: corners, h[r], h[s], tabu memory, trail
        if (is_winner) {
            // corner terms (D[r][s] - D[s][r]) F[ps][pr] and (D[s][r] - D[r][s]) F[pr][ps]: zero when both
            // matrices are symmetric, so that case loads nothing here
            int32_t kr = 0, ks = 0;
            if (!FULLSYM) {
                const int32_t Drs = ldD(r, s), Dsr = ldD(s, r);
                const int32_t Fpspr = ldF(ps, pr), Fprps = ldF(pr, ps);
                kr = (Drs - Dsr) * Fpspr;
                ks = (Dsr - Drs) * Fprps;
            }
            // the tenure of this move (tabu.py:184-186): drawn on the device or provided by the caller
            const long long ten = !tabu ? 0 : ((P.rng || REC) ? (long long)sTen[(c - 1) & (TENURE_CHUNK - 1)]
                                                              : (long long)P.tenures[(size_t)b * iters + (c - 1)]);
            const int32_t new_exp = (int32_t)(c + ten);
            int32_t mrs = 0, msr = 0;
            unsigned was = 0;
            if (DSM && my_which == WHICH_DIAG) {
                mrs = sDG[16 * dsmI + ru * 4 + su];
                msr = sDG[16 * dsmI + su * 4 + ru];
                was = (sDGtb[dsmI] >> my_slot) & 1u;
                if (tabu) {
                    sDGtb[dsmI] |= 1u << my_slot;
                    sDGmx[dsmI] = min(sDGmx[dsmI], new_exp);
                    xp[(noff + dsmI) * 16 + my_slot] = new_exp;
                }
            } else if (!SMEMU || my_which < UR) {
#pragma unroll
                for (int k = 0; k < UR; ++k) {
                    if (k != my_which) continue;
                    mrs = V.ColS[r];  // this thread dumped both columns above: M[r][s], M[s][r]
                    msr = V.ColR[s];
                    was = (tb[k] >> my_slot) & 1u;
                    if (tabu) {
                        tb[k] |= 1u << my_slot;
                        mexp[k] = min(mexp[k], new_exp);
                        // (DD: slots 16..31 are the second diagonal block of this thread, the next row of xp)
                        xp[uidv[k] * 16 + my_slot] = new_exp;
                    }
                }
            } else {
                const int k2 = my_which - UR;
                mrs = sM[((size_t)((k2 * 8 + ru) * Toff + tid)) * 4 + su];      // U[ru][su]
                msr = sM[((size_t)((k2 * 8 + 4 + su) * Toff + tid)) * 4 + ru];  // L[su][ru]
                const unsigned old = sTB[k2 * Toff + tid];
                was = (old >> my_slot) & 1u;
                if (tabu) {
                    sTB[k2 * Toff + tid] = old | (1u << my_slot);
                    sMX[k2 * Toff + tid] = min(sMX[k2 * Toff + tid], new_exp);
                    xp[(UR * Toff + k2 * Toff + tid) * 16 + my_slot] = new_exp;
                }
            }
            const int32_t hr = V.H[r], hs = V.H[s];
            V.TS[r] = hr + kr;  // M'[r][s]
            V.TR[s] = hs + ks;  // M'[s][r]
            const int32_t hrn = mrs + ks, hsn = msr + kr;
            V.H[r] = hrn;
            V.H[s] = hsn;
            if (PACKED) {
                V.HI[r] = 4 * ru - 16 * hrn; V.HJ[r] = ru - 16 * hrn;
                V.HI[s] = 4 * su - 16 * hsn; V.HJ[s] = su - 16 * hsn;
            }
            if (REC && P.tr_i) {  // trail row (_kernels.pyx:182-187); was_tabu = cells[bi][bj] > c (:171)
                const size_t o = (size_t)b * iters + (c - 1);
                P.tr_i[o] = r; P.tr_j[o] = s; P.tr_d[o] = (int64_t)bd;
                if (P.tr_tabu) P.tr_tabu[o] = (int64_t)was;
            }
            if (REC && tabu && P.cells) {
                int64_t *cz = P.cells + (size_t)b * n * n;
                cz[(size_t)r * n + s] = (int64_t)c + ten;
                atomicAdd(reinterpret_cast<unsigned long long *>(cz + (size_t)s * n + r), 1ULL);  // (a reduction without return: the load-add-store would wait for L2)
            }
        }
        if (timing) tE = clock64();
        // ---- tabu bits that expire at the next iteration are cleared here; shared-memory units and
        // shared-memory diagonal blocks publish their parts of columns r and s
#pragma unroll
        for (int k = 0; k < UR; ++k)
            if (own[k] && c + 1 >= mexp[k]) {
                if (DD && ddiag) {
                    unsigned lo = tb[k] & 0xffffu, hi = tb[k] >> 16;
                    int32_t ma, mb;
                    expire_bits(lo, ma, c + 1, xp + uidv[k] * 16);
                    if (J[k] >= 0) expire_bits(hi, mb, c + 1, xp + (uidv[k] + 1) * 16);
                    else mb = MAXV;
                    tb[k] = lo | (hi << 16);
                    mexp[k] = min(ma, mb);
                } else {
                    expire_bits(tb[k], mexp[k], c + 1, xp + uidv[k] * 16);
                }
            }
        if (SMEMU && offt) {
#pragma unroll 1
            for (int k2 = 0; k2 < US; ++k2) {
                const int uid = UR * Toff + k2 * Toff + tid;
                if (uid >= noff) break;
                const int Ik = P.unit_ij[uid] & 0xff, Jk = P.unit_ij[uid] >> 8;
                // element (row w, lane l) of this unit: sM[((k2*8 + w)*Toff + tid)*4 + l]
                const int32_t *base = sM + ((size_t)(k2 * 8) * Toff + tid) * 4;
                const size_t rs4 = (size_t)Toff * 4;  // stride between rows
                if (Jk == R) st_vec4(V.ColR, Ik, base[0 * rs4 + ru], base[1 * rs4 + ru], base[2 * rs4 + ru], base[3 * rs4 + ru]);
                if (Ik == R) st_vec4(V.ColR, Jk, base[4 * rs4 + ru], base[5 * rs4 + ru], base[6 * rs4 + ru], base[7 * rs4 + ru]);
                if (Jk == S) st_vec4(V.ColS, Ik, base[0 * rs4 + su], base[1 * rs4 + su], base[2 * rs4 + su], base[3 * rs4 + su]);
                if (Ik == S) st_vec4(V.ColS, Jk, base[4 * rs4 + su], base[5 * rs4 + su], base[6 * rs4 + su], base[7 * rs4 + su]);
                int32_t mx = sMX[k2 * Toff + tid];
                if (c + 1 >= mx) {
                    unsigned tbv = sTB[k2 * Toff + tid];
                    expire_bits(tbv, mx, c + 1, xp + uid * 16);
                    sTB[k2 * Toff + tid] = tbv;
                    sMX[k2 * Toff + tid] = mx;
                }
            }
        }
        if (dsm_owner) {
            const int32_t *dg = sDG + 16 * dsmI;
            if (dsmI == R)
                st_vec4(V.ColR, dsmI, ru == 0 ? 0 : dg[0 + ru], ru == 1 ? 0 : dg[4 + ru], ru == 2 ? 0 : dg[8 + ru], ru == 3 ? 0 : dg[12 + ru]);
            if (dsmI == S)
                st_vec4(V.ColS, dsmI, su == 0 ? 0 : dg[0 + su], su == 1 ? 0 : dg[4 + su], su == 2 ? 0 : dg[8 + su], su == 3 ? 0 : dg[12 + su]);
            int32_t mx = sDGmx[dsmI];
            if (c + 1 >= mx) {
                unsigned tbv = sDGtb[dsmI];
                expire_bits(tbv, mx, c + 1, xp + (noff + dsmI) * 16);
                sDGtb[dsmI] = tbv;
                sDGmx[dsmI] = mx;
            }
        }
        if (timing) tF = clock64();
        if (OW) __syncwarp(); else __syncthreads();  // ------------------- sync #2
        if (tid == 0) { sP[r] = ps; sP[s] = pr; }
        if (timing) {
            const long long tG = clock64() + (sP[0] & 0);
            tacc[0] += tB - tA; tacc[1] += tC - tB; tacc[2] += tD - tC; tacc[3] += tE - tD; tacc[4] += tF - tE; tacc[5] += tG - tF;
        }
    }
    if (timing) {
        const int slot = tid == 0 ? 0 : (tid == 128 ? 1 : 2);
        for (int q = 0; q < 6; ++q) P.dbg[slot * 6 + q] = tacc[q];
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

}  // namespace qapb
