// search_reg.cuh -- register-resident variant of the search kernel (n <= 128, int32 state).
//
// Same algorithm and the same integers as qap_search_kernel (search_kernel.cuh), but the
// placement matrix M and the tabu triangle never leave the register file: thread t < noff
// owns off-diagonal unit t = block pair {(I,J),(J,I)} as 32 + 16 registers for the whole
// run, so the per-iteration pass is pure ALU work (rank-2 update, delta, admissibility,
// running argmin) fed by a handful of 128-bit shared-memory vector loads.  The last warp
// owns the nb diagonal 4x4 blocks, kept in shared memory.
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
// uniform across the CTA, so the register indices are selected with uniform switches.
#pragma once
#include "search_kernel.cuh"

namespace qapb {

__host__ __device__ inline RegLayout make_reg_layout(int npad, int nb)
{
    RegLayout L;
    unsigned o = 0;
    const unsigned v = 4u * (unsigned)npad;
    L.offA = o; o += v; L.offC = o; o += v; L.offB = o; o += v; L.offE = o; o += v; L.offH = o; o += v;
    L.offColR = o; o += v; L.offColS = o; o += v; L.offTR = o; o += v; L.offTS = o; o += v;
    L.offXR = o; o += v; L.offXS = o; o += v;
    L.offP = o; o += v; L.offJ = o; o += v;
    L.offDM = o; o += 64u * (unsigned)nb;
    L.offDT = o; o += 64u * (unsigned)nb;
    L.offRedD = o; o += 32u * 8u;
    L.offRedK = o; o += 32u * 4u;
    L.offMisc = o; o += 64u;
    L.offTen = o; o += 4u * TENURE_CHUNK;
    L.total = align16(o);
    return L;
}

__device__ __forceinline__ int32_t pick16(const int32_t (&A)[4][4], int slot)
{
    int32_t r = A[0][0];
#pragma unroll
    for (int q = 1; q < 16; ++q) r = (slot == q) ? A[q >> 2][q & 3] : r;
    return r;
}
__device__ __forceinline__ void put16(int32_t (&A)[4][4], int slot, int32_t val)
{
#pragma unroll
    for (int q = 0; q < 16; ++q) A[q >> 2][q & 3] = (slot == q) ? val : A[q >> 2][q & 3];
}
__device__ __forceinline__ void st_vec4(int32_t *arr, int blk, int32_t a, int32_t b, int32_t c, int32_t d)
{
    reinterpret_cast<int4 *>(arr)[blk] = make_int4(a, b, c, d);
}

// M entries of one unit from scratch (O(n) per entry): the full evaluator, also used by
// kernels.all_deltas.  U[u][v] = M[4I+u][4J+v], L[v][u] = M[4J+v][4I+u].
__device__ __forceinline__ void build_unit(const SearchParams &P, const int32_t *sP, int I, int J, bool sym,
                                           int32_t (&U)[4][4], int32_t (&L)[4][4], int32_t (&Ex)[4][4])
{
    const int n = P.n, npad = P.npad;
    const int32_t *__restrict__ F = P.F;
    const int32_t *__restrict__ FT = P.FT;
    const int32_t *__restrict__ D = P.D;
    const int32_t *__restrict__ DT = P.DT;
    int pI[4], pJ[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { pI[u] = sP[4 * I + u]; pJ[u] = sP[4 * J + u]; }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) { U[u][v] = 0; L[u][v] = 0; }
    for (int kk = 0; kk < n; ++kk) {
        const int pk = sP[kk];
        int32_t dI[4], dJ[4], fI[4], fJ[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            dI[u] = D[(4 * I + u) * npad + kk];
            dJ[u] = D[(4 * J + u) * npad + kk];
            fI[u] = F[pI[u] * npad + pk];
            fJ[u] = F[pJ[u] * npad + pk];
        }
        if (sym) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    U[u][v] += dI[u] * fJ[v];
                    L[v][u] += dJ[v] * fI[u];
                }
        } else {
            int32_t dtI[4], dtJ[4], ftI[4], ftJ[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                dtI[u] = DT[(4 * I + u) * npad + kk];
                dtJ[u] = DT[(4 * J + u) * npad + kk];
                ftI[u] = FT[pI[u] * npad + pk];
                ftJ[u] = FT[pJ[u] * npad + pk];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    U[u][v] += dI[u] * fJ[v] + dtI[u] * ftJ[v];
                    L[v][u] += dJ[v] * fI[u] + dtJ[v] * ftI[u];
                }
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int i = 4 * I + u, j = 4 * J + v;
            if (sym) { U[u][v] *= 2; L[v][u] *= 2; }
            const int32_t fs = F[pI[u] * npad + pJ[v]] + F[pJ[v] * npad + pI[u]];
            U[u][v] += D[i * npad + j] * fs + P.dd[i] * P.fd[pJ[v]];
            L[v][u] += D[j * npad + i] * fs + P.dd[j] * P.fd[pI[u]];
            const bool pad = (i >= n) || (j >= n);
            if (pad) { U[u][v] = 1 << 29; L[v][u] = 1 << 29; }
            if (i == j) { U[u][v] = 0; L[v][u] = 0; }
            Ex[u][v] = pad ? 0x7fffffff : 0;
        }
}

#define QAPB_SWITCH4(idx, BODY)            \
    switch (idx) {                         \
        case 0: { constexpr int q = 0; BODY } break; \
        case 1: { constexpr int q = 1; BODY } break; \
        case 2: { constexpr int q = 2; BODY } break; \
        default: { constexpr int q = 3; BODY } break; \
    }

// 16-way switch over slot = u*4+v; `qu`, `qv` are compile-time inside BODY.
#define QAPB_SWITCH16(uu, vv, BODY)                                        \
    QAPB_SWITCH4(uu, { constexpr int qu = q; switch (vv) {                 \
        case 0: { constexpr int qv = 0; BODY } break;                     \
        case 1: { constexpr int qv = 1; BODY } break;                     \
        case 2: { constexpr int qv = 2; BODY } break;                     \
        default: { constexpr int qv = 3; BODY } break; } })

template <bool SYM, bool PACKED, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) qap_search_reg_kernel(const SearchParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, W = T >> 5;
    const int b = blockIdx.x;
    const int n = P.n, nb = P.nb, npad = P.npad, noff = P.noff;
    const int Toff = T - 32;  // the last warp owns the diagonal blocks
    const RegLayout &lay = P.rlay;
    int32_t *sA = reinterpret_cast<int32_t *>(smem_raw + lay.offA);
    int32_t *sC = reinterpret_cast<int32_t *>(smem_raw + lay.offC);
    int32_t *sB = reinterpret_cast<int32_t *>(smem_raw + lay.offB);
    int32_t *sE = reinterpret_cast<int32_t *>(smem_raw + lay.offE);
    int32_t *sH = reinterpret_cast<int32_t *>(smem_raw + lay.offH);
    int32_t *sColR = reinterpret_cast<int32_t *>(smem_raw + lay.offColR);
    int32_t *sColS = reinterpret_cast<int32_t *>(smem_raw + lay.offColS);
    int32_t *sTR = reinterpret_cast<int32_t *>(smem_raw + lay.offTR);
    int32_t *sTS = reinterpret_cast<int32_t *>(smem_raw + lay.offTS);
    int32_t *sXR = reinterpret_cast<int32_t *>(smem_raw + lay.offXR);
    int32_t *sXS = reinterpret_cast<int32_t *>(smem_raw + lay.offXS);
    int32_t *sP = reinterpret_cast<int32_t *>(smem_raw + lay.offP);
    unsigned *sJ = reinterpret_cast<unsigned *>(smem_raw + lay.offJ);
    long long *sRed64 = reinterpret_cast<long long *>(smem_raw + lay.offRedD);
    int32_t *sRedD = reinterpret_cast<int32_t *>(smem_raw + lay.offRedD);
    unsigned *sRedK = reinterpret_cast<unsigned *>(smem_raw + lay.offRedK);
    long long *sMisc = reinterpret_cast<long long *>(smem_raw + lay.offMisc);
    int32_t *sTen = reinterpret_cast<int32_t *>(smem_raw + lay.offTen);

    const int32_t *__restrict__ F = P.F;
    const int32_t *__restrict__ FT = P.FT;
    const int32_t *__restrict__ D = P.D;
    const int32_t *__restrict__ DT = P.DT;
    const int32_t MAXV = 0x7fffffff;
    const int one = P.one, sixteen = P.sixteen;

    // ---------------------------------------------------------------- setup
    for (int i = tid; i < npad; i += T) {
        sA[i] = 0; sC[i] = 0; sB[i] = 0; sE[i] = 0; sH[i] = 0;
        sColR[i] = 0; sColS[i] = 0; sTR[i] = 0; sTS[i] = 0; sXR[i] = 0; sXS[i] = 0;
        sP[i] = (P.rng || i >= n) ? (i < n ? i : 0) : (int32_t)P.perms[(size_t)b * n + i];
    }
    unsigned long long rng_state = 0;
    if (P.rng) {
        const unsigned long long seed = mix64(P.master_seed + QAPB_GAMMA * (P.first_index + (unsigned long long)b + 1ULL));
        int reject = P.force_seq_rng;
        for (int k = tid; k < n - 1; k += T) {
            unsigned long long bound = (unsigned long long)(n - 1 - k) + 1ULL;
            unsigned long long r = mix64(seed + QAPB_GAMMA * ((unsigned long long)k + 1ULL));
            unsigned long long rem = (0ULL - bound) % bound;
            if (r > ~0ULL - rem) reject = 1;
            sJ[n - 1 - k] = (unsigned)(r % bound);
        }
        reject = __syncthreads_or(reject);
        if (tid == 0) {
            rng_state = seed;
            if (reject) {
                for (int i = n - 1; i >= 1; --i) {
                    unsigned j = (unsigned)randbelow_seq(rng_state, (unsigned long long)i + 1ULL);
                    int32_t t = sP[i]; sP[i] = sP[j]; sP[j] = t;
                }
            } else {
                for (int i = n - 1; i >= 1; --i) {
                    unsigned j = sJ[i];
                    int32_t t = sP[i]; sP[i] = sP[j]; sP[j] = t;
                }
                rng_state = seed + QAPB_GAMMA * (unsigned long long)(n - 1);
            }
            sMisc[2] = (long long)rng_state;
        }
    }
    if (P.cells) {
        int64_t *cz = P.cells + (size_t)b * n * n;
        for (int i = tid; i < n * n; i += T) cz[i] = 0;
    }
    __syncthreads();
    if (P.rng) rng_state = (unsigned long long)sMisc[2];

    long long cost;
    {
        long long part = 0;
        for (int idx = tid; idx < n * n; idx += T) {
            int i = idx / n, j = idx - i * n;
            int pi = sP[i], pj = sP[j];
            part += (i == j) ? (long long)P.fd[pi] * P.dd[i] : (long long)F[pi * npad + pj] * D[i * npad + j];
        }
        cost = block_sum_i64(part, sRed64, tid, T);
        __syncthreads();
    }
    for (int i = tid; i < n; i += T) {
        int pi = sP[i];
        int32_t acc = P.dd[i] * P.fd[pi];
        if (SYM) {
            for (int k = 0; k < n; ++k) acc += 2 * (D[i * npad + k] * F[pi * npad + sP[k]]);
        } else {
            for (int k = 0; k < n; ++k) {
                int pk = sP[k];
                acc += D[i * npad + k] * F[pi * npad + pk] + DT[i * npad + k] * FT[pi * npad + pk];
            }
        }
        sH[i] = acc;
    }

    // Unit ownership.  Off-diagonal thread: U = block (I,J), L = block (J,I), E = tabu expiry of
    // the 16 pairs.  Diagonal lane: I == J, U = the block itself (L unused), E valid for u < v.
    const bool offd = tid < noff;
    const bool diag = tid >= Toff && (tid - Toff) < nb;
    int I = 0, J = 0;
    if (offd) { I = P.unit_ij[tid] & 0xff; J = P.unit_ij[tid] >> 8; }
    if (diag) { I = tid - Toff; J = I; }
    int32_t U[4][4], L[4][4], E[4][4];
    if (offd || diag) {
        build_unit(P, sP, I, J, SYM, U, L, E);
        if (diag) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    if (u >= v) E[u][v] = 0x7fffffff;  // only pairs u < v exist in a diagonal block
        }
    }
    __syncthreads();

    // ------------------------------------------------------------ iterations
    long long best_cost = cost;
    int32_t thr = 0;
    const bool tabu = P.mode == MODE_TABU;
    const int iters = P.iterations;
    int steps_done = 0, stopped = 0;
    int64_t *best_out = P.best + (size_t)b * n;
    for (int i = tid; i < n; i += T) best_out[i] = sP[i];
    int R = -1, S = -1, ru = 0, su = 0;  // previous move (block and in-block indices)

    long long tacc[5] = {0, 0, 0, 0, 0};
    long long psub[3] = {0, 0, 0};
    const bool timing = P.dbg != nullptr && b == 0 && (tid == 0 || tid == 128 || tid == Toff);
    for (int c = 1; c <= iters; ++c) {
        long long tA = 0, tB = 0, tC = 0, tD = 0, tE = 0;
        if (timing) tA = clock64();
        long long ten = 0;
        if (tabu) {
            if (!P.rng) {
                ten = P.tenures[(size_t)b * iters + (c - 1)];
            } else if (((c - 1) & (TENURE_CHUNK - 1)) == 0) {
                fill_tenure_chunk(rng_state, P.ten_lo, P.ten_hi, P.force_seq_rng, sTen, sMisc, tid, T);
            }
        }

        int32_t my_d = MAXV;
        int my_slot = 0;
        long long q0 = 0, q1 = 0, q2 = 0;
        if (timing) q0 = clock64();
        if (offd) {
            if (R >= 0) {
                // ---- generic rank-2 update (a is pre-doubled for symmetric instances)
                int32_t aI[4], bI[4], aJ[4], bJ[4];
                ld_vec4(sA, I, aI); ld_vec4(sB, I, bI); ld_vec4(sA, J, aJ); ld_vec4(sB, J, bJ);
                if (SYM) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            U[u][v] -= aI[u] * bJ[v];
                            L[v][u] -= aJ[v] * bI[u];
                        }
                } else {
                    int32_t cI[4], eI[4], cJ[4], eJ[4];
                    ld_vec4(sC, I, cI); ld_vec4(sE, I, eI); ld_vec4(sC, J, cJ); ld_vec4(sE, J, eJ);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            U[u][v] -= aI[u] * bJ[v] + cI[u] * eJ[v];
                            L[v][u] -= aJ[v] * bI[u] + cJ[v] * eI[u];
                        }
                }
                if (timing) q1 = clock64();
                // ---- rows / columns r and s of the previous move
                if (I == R || J == R || I == S || J == S) {
                    if (I == R) {
                        int32_t x[4], cs[4], t[4];
                        ld_vec4(sXR, J, x); ld_vec4(sColS, J, cs); ld_vec4(sTR, J, t);
                        QAPB_SWITCH4(ru, {
_Pragma("unroll")
                            for (int v = 0; v < 4; ++v) { U[q][v] += x[v]; L[v][q] = cs[v] + t[v]; }
                        })
                    }
                    if (J == R) {
                        int32_t x[4], cs[4], t[4];
                        ld_vec4(sXR, I, x); ld_vec4(sColS, I, cs); ld_vec4(sTR, I, t);
                        QAPB_SWITCH4(ru, {
_Pragma("unroll")
                            for (int u = 0; u < 4; ++u) { L[q][u] += x[u]; U[u][q] = cs[u] + t[u]; }
                        })
                    }
                    if (I == S) {
                        int32_t x[4], cr[4], t[4];
                        ld_vec4(sXS, J, x); ld_vec4(sColR, J, cr); ld_vec4(sTS, J, t);
                        QAPB_SWITCH4(su, {
_Pragma("unroll")
                            for (int v = 0; v < 4; ++v) { U[q][v] += x[v]; L[v][q] = cr[v] + t[v]; }
                        })
                    }
                    if (J == S) {
                        int32_t x[4], cr[4], t[4];
                        ld_vec4(sXS, I, x); ld_vec4(sColR, I, cr); ld_vec4(sTS, I, t);
                        QAPB_SWITCH4(su, {
_Pragma("unroll")
                            for (int u = 0; u < 4; ++u) { L[q][u] += x[u]; U[u][q] = cr[u] + t[u]; }
                        })
                    }
                }
            }
            if (timing) q2 = clock64();
            // ---- delta, admissibility (_kernels.pyx:162), first minimum.  The ALU pipe (IADD3 /
            // ISETP / IMNMX, half rate) is the binding resource of this pass, so the first add of
            // each delta and the (delta, slot) packing are written as multiplications by the
            // runtime constants 1 and 16: they issue as IMAD on the otherwise idle FMA pipe.
            int32_t hI[4], hJ[4];
            ld_vec4(sH, I, hI);
            ld_vec4(sH, J, hJ);
            if (PACKED) {
                // |delta| < 2^27 (host-proven): key = delta*16 + slot orders by (delta, slot), so the
                // running first-minimum is one predicated IMNMX per pair; four independent chains.
                int32_t km[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    km[u] = MAXV;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int32_t d = (U[u][v] * one + L[v][u]) - hI[u] - hJ[v];
                        const bool adm = (E[u][v] <= c) || (d < thr);
                        const int32_t kd = (int32_t)((uint32_t)d * (uint32_t)sixteen + (uint32_t)(u * 4 + v));
                        if (adm) km[u] = min(km[u], kd);
                    }
                }
                const int32_t m = min(min(km[0], km[1]), min(km[2], km[3]));
                if (m != MAXV) { my_d = m >> 4; my_slot = m & 15; }
            } else {
                int32_t rd[4];
                int rs[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    rd[u] = MAXV;
                    rs[u] = u * 4;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int32_t d = (U[u][v] * one + L[v][u]) - hI[u] - hJ[v];
                        const bool adm = (E[u][v] <= c) || (d < thr);
                        if (adm && d < rd[u]) { rd[u] = d; rs[u] = u * 4 + v; }
                    }
                }
                if (rd[1] < rd[0]) { rd[0] = rd[1]; rs[0] = rs[1]; }
                if (rd[3] < rd[2]) { rd[2] = rd[3]; rs[2] = rs[3]; }
                if (rd[2] < rd[0]) { rd[0] = rd[2]; rs[0] = rs[2]; }
                my_d = rd[0];
                my_slot = rs[0];
            }
        } else if (diag) {
            if (R >= 0) {
                int32_t aI[4], bI[4];
                ld_vec4(sA, I, aI); ld_vec4(sB, I, bI);
                if (SYM) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            if (u != v) U[u][v] -= aI[u] * bI[v];
                } else {
                    int32_t cI[4], eI[4];
                    ld_vec4(sC, I, cI); ld_vec4(sE, I, eI);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            if (u != v) U[u][v] -= aI[u] * bI[v] + cI[u] * eI[v];
                }
                // rows / columns r and s inside this diagonal block: column assignments first,
                // then the row increments (x is 0 at the corner positions)
                if (I == R) {
                    int32_t cs[4], t[4];
                    ld_vec4(sColS, I, cs); ld_vec4(sTR, I, t);
                    QAPB_SWITCH4(ru, {
_Pragma("unroll")
                        for (int u = 0; u < 4; ++u) if (u != q) U[u][q] = cs[u] + t[u];
                    })
                }
                if (I == S) {
                    int32_t cr[4], t[4];
                    ld_vec4(sColR, I, cr); ld_vec4(sTS, I, t);
                    QAPB_SWITCH4(su, {
_Pragma("unroll")
                        for (int u = 0; u < 4; ++u) if (u != q) U[u][q] = cr[u] + t[u];
                    })
                }
                if (I == R) {
                    int32_t x[4];
                    ld_vec4(sXR, I, x);
                    QAPB_SWITCH4(ru, {
_Pragma("unroll")
                        for (int v = 0; v < 4; ++v) if (v != q) U[q][v] += x[v];
                    })
                }
                if (I == S) {
                    int32_t x[4];
                    ld_vec4(sXS, I, x);
                    QAPB_SWITCH4(su, {
_Pragma("unroll")
                        for (int v = 0; v < 4; ++v) if (v != q) U[q][v] += x[v];
                    })
                }
            }
            int32_t hI[4];
            ld_vec4(sH, I, hI);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = u + 1; v < 4; ++v) {
                    const int32_t d = U[u][v] + U[v][u] - hI[u] - hI[v];
                    const bool adm = (E[u][v] <= c) || (d < thr);
                    if (adm && d < my_d) { my_d = d; my_slot = u * 4 + v; }
                }
        }
        const unsigned my_key = (my_d != MAXV) ? pair_key(4 * I + (my_slot >> 2), 4 * J + (my_slot & 3), 0) : 0xffffffffu;

        if (timing) { tB = clock64(); psub[0] += q1 - q0; psub[1] += q2 - q1; psub[2] += tB - q2; }
        int32_t bd = my_d;
        unsigned bkey = my_key;
        warp_argmin(bd, bkey);
        if (lane == 0) { sRedD[warp] = bd; sRedK[warp] = bkey; }
        __syncthreads();  // ---------------------------------------------- sync #1
        if (timing) tC = clock64();
        bd = lane < W ? sRedD[lane] : MAXV;
        bkey = lane < W ? sRedK[lane] : 0xffffffffu;
        warp_argmin(bd, bkey);
        if (bd == MAXV) {
            stopped = 1;
            break;
        }
        const int r = (int)(bkey >> 17), s = (int)((bkey >> 1) & 0xffffu);
        cost += (long long)bd;
        const bool improved = cost < best_cost;
        if (improved) best_cost = cost;
        thr = Acc<int32_t>::clamp_thr(best_cost - cost);
        if (tabu && P.rng) ten = sTen[(c - 1) & (TENURE_CHUNK - 1)];
        steps_done = c;
        R = r >> 2; S = s >> 2; ru = r & 3; su = s & 3;
        const int pr = sP[r], ps = sP[s];
        if (timing) tD = clock64();

        // ---- difference vectors of the move (old permutation), additive terms, h: thread i < n
        if (tid < n) {
            const int i = tid;
            const int pi = sP[i];
            const bool mid = (i != r) && (i != s);
            if (improved) best_out[i] = (i == r) ? ps : (i == s) ? pr : pi;
            if (SYM) {
                // D = D^T, F = F^T: a = c, b = e, and the closed forms collapse
                const int32_t Drs = D[r * npad + s], Fpspr = F[ps * npad + pr];
                const int32_t Dsi = D[s * npad + i], Dri = D[r * npad + i];
                const int32_t Fpspi = F[ps * npad + pi], Fprpi = F[pr * npad + pi];
                const int32_t a = mid ? Dsi - Dri : 0, bb = mid ? Fpspi - Fprpi : 0;
                const int32_t a2 = 2 * a, b2 = 2 * bb;
                sA[i] = a2;
                sB[i] = bb;
                sXR[i] = b2 * ((mid ? Dri : 0) - Drs);
                sXS[i] = b2 * (Drs - (mid ? Dsi : 0));
                if (mid) {
                    sH[i] -= a2 * bb;
                    sTR[i] = a2 * (Fpspr - Fpspi);
                    sTS[i] = a2 * (Fprpi - Fpspr);
                } else if (i == r) {
                    sTR[i] = 0;  // tS[r] is written by the owner of the pair
                } else {
                    sTS[i] = 0;  // tR[s] is written by the owner of the pair
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
                sA[i] = a;
                sB[i] = bb;
                sC[i] = cc;
                sE[i] = e;
                sXR[i] = -Drs * bb - Dsr * e + (mid ? Dri : 0) * be;
                sXS[i] = Dsr * bb + Drs * e - (mid ? Dsi : 0) * be;
                if (mid) {
                    sH[i] -= a * bb + cc * e;
                    sTR[i] = a * (Fpspr - (Fpips + Fpspi)) + cc * Fprps;
                    sTS[i] = a * ((Fpipr + Fprpi) - Fprps) - cc * Fpspr;
                } else if (i == r) {
                    sTR[i] = 0;
                } else {
                    sTS[i] = 0;
                }
            }
        }
        // ---- the thread owning the winning pair: corners, h[r], h[s], tabu memory, trail
        if (my_key == bkey) {
            const int32_t Drs = D[r * npad + s], Dsr = D[s * npad + r];
            const int32_t Fpspr = F[ps * npad + pr], Fprps = F[pr * npad + ps];
            int32_t mrs = 0, msr = 0, old_exp = 0;
            const int32_t new_exp = (int32_t)(c + ten);
            if (offd) {
                QAPB_SWITCH16(ru, su, {
                    mrs = U[qu][qv]; msr = L[qv][qu]; old_exp = E[qu][qv];
                    if (tabu) E[qu][qv] = new_exp;
                })
            } else {
                QAPB_SWITCH16(ru, su, {
                    mrs = U[qu][qv]; msr = U[qv][qu]; old_exp = E[qu][qv];
                    if (tabu) E[qu][qv] = new_exp;
                })
            }
            const int32_t hr = sH[r], hs = sH[s];
            sTS[r] = hr + (Drs - Dsr) * Fpspr;  // M'[r][s]
            sTR[s] = hs + (Dsr - Drs) * Fprps;  // M'[s][r]
            sH[r] = mrs + (Dsr - Drs) * Fprps;
            sH[s] = msr + (Drs - Dsr) * Fpspr;
            if (P.tr_i) {  // trail row (_kernels.pyx:182-187); was_tabu = cells[bi][bj] > c (:171)
                const size_t o = (size_t)b * iters + (c - 1);
                P.tr_i[o] = r; P.tr_j[o] = s; P.tr_d[o] = (int64_t)bd;
                if (P.tr_tabu) P.tr_tabu[o] = old_exp > c ? 1 : 0;
            }
            if (tabu && P.cells) {
                int64_t *cz = P.cells + (size_t)b * n * n;
                cz[(size_t)r * n + s] = (int64_t)c + ten;
                cz[(size_t)s * n + r] += 1;
            }
        }
        // ---- owners of columns r and s publish them (colR[r] = colS[s] = 0 by the diagonal lanes)
        if (offd) {
            if (J == R) { QAPB_SWITCH4(ru, { st_vec4(sColR, I, U[0][q], U[1][q], U[2][q], U[3][q]); }) }
            if (I == R) { QAPB_SWITCH4(ru, { st_vec4(sColR, J, L[0][q], L[1][q], L[2][q], L[3][q]); }) }
            if (J == S) { QAPB_SWITCH4(su, { st_vec4(sColS, I, U[0][q], U[1][q], U[2][q], U[3][q]); }) }
            if (I == S) { QAPB_SWITCH4(su, { st_vec4(sColS, J, L[0][q], L[1][q], L[2][q], L[3][q]); }) }
        } else if (diag) {
            if (I == R) {
                QAPB_SWITCH4(ru, { st_vec4(sColR, I, q == 0 ? 0 : U[0][q], q == 1 ? 0 : U[1][q], q == 2 ? 0 : U[2][q], q == 3 ? 0 : U[3][q]); })
            }
            if (I == S) {
                QAPB_SWITCH4(su, { st_vec4(sColS, I, q == 0 ? 0 : U[0][q], q == 1 ? 0 : U[1][q], q == 2 ? 0 : U[2][q], q == 3 ? 0 : U[3][q]); })
            }
        }
        if (timing) tE = clock64();
        __syncthreads();  // ---------------------------------------------- sync #2
        if (timing) {
            const long long tF = clock64();
            tacc[0] += tB - tA; tacc[1] += tC - tB; tacc[2] += tD - tC; tacc[3] += tE - tD; tacc[4] += tF - tE;
        }
        if (tid == 0) { sP[r] = ps; sP[s] = pr; }
    }
    if (timing) {
        const int slot = tid == 0 ? 0 : (tid == 128 ? 1 : 2);
        for (int q = 0; q < 5; ++q) P.dbg[slot * 5 + q] = tacc[q];
        if (tid == 128) for (int q = 0; q < 3; ++q) P.dbg[10 + q] = psub[q];  // overwrites the diag slot's first entries
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
