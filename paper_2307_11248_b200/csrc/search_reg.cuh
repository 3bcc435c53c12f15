// search_reg.cuh -- register-resident variant of the search kernel (n <= 128, int32 state).
//
// Same algorithm and the same integers as qap_search_kernel (search_kernel.cuh), but the
// placement matrix M and the tabu triangle never leave the register file: thread t < noff
// owns one or two off-diagonal units (block pairs {(I,J),(J,I)}, 32 registers each) plus a
// 16-bit mask of their currently-tabu pairs for the whole run (expiry iterations live in a
// shared-memory array that is only touched when a pair is set or expires), so the per-iteration pass is pure ALU work (rank-2 update, delta, admissibility,
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
    L.offExp = o; o += 64u * (unsigned)(nb * (nb - 1) / 2 + nb);  // tabu expiry per (unit, slot)
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


// Upper bound (exclusive) on unit ids handled by off-diagonal threads: uid = t + k*Toff.
template <bool SYM, bool PACKED, int UPT, int MAXREG>
__global__ void __maxnreg__(MAXREG) qap_search_reg_kernel(const SearchParams P)
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
    int32_t *sExp = reinterpret_cast<int32_t *>(smem_raw + lay.offExp);  // [unit][16] expiry iteration

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

    // Unit ownership.  Off-diagonal thread t owns units t + k*Toff (k < UPT): U = block (I,J),
    // L = block (J,I).  Diagonal lane: one unit, I == J, U = the block itself (L unused), pairs u < v.
    // tb = mask of pairs that are tabu now (pads and non-pairs permanently set), mexp = earliest
    // expiry among the clearable bits.
    const bool diag = tid >= Toff && (tid - Toff) < nb;
    int I[UPT], J[UPT], uidv[UPT];
    bool own[UPT];
    int32_t U[UPT][4][4], L[UPT][4][4];
    unsigned tb[UPT];
    int32_t mexp[UPT];
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
        const int uid = tid + k * Toff;
        own[k] = (tid < Toff) && (uid < noff);
        I[k] = 0; J[k] = 0; uidv[k] = 0; tb[k] = 0xffffu; mexp[k] = MAXV;
        if (own[k]) { I[k] = P.unit_ij[uid] & 0xff; J[k] = P.unit_ij[uid] >> 8; uidv[k] = uid; }
        if (k == 0 && diag) { I[0] = tid - Toff; J[0] = I[0]; uidv[0] = noff + I[0]; own[0] = true; }
        if (own[k]) {
            int32_t Ex[4][4];
            build_unit(P, sP, I[k], J[k], SYM, U[k], L[k], Ex);
            unsigned m = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const bool dead = (Ex[u][v] != 0) || (diag && u >= v);  // pad pair or not a pair
                    if (dead) m |= 1u << (u * 4 + v);
                    sExp[uidv[k] * 16 + u * 4 + v] = dead ? MAXV : 0;
                }
            tb[k] = m;
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

    for (int c = 1; c <= iters; ++c) {
        long long ten = 0;
        if (tabu) {
            if (!P.rng) {
                ten = P.tenures[(size_t)b * iters + (c - 1)];
            } else if (((c - 1) & (TENURE_CHUNK - 1)) == 0) {
                fill_tenure_chunk(rng_state, P.ten_lo, P.ten_hi, P.force_seq_rng, sTen, sMisc, tid, T);
            }
        }

        int32_t my_d = MAXV;
        unsigned my_key = 0xffffffffu;
        int my_k = 0, my_slot = 0;
#pragma unroll
        for (int k = 0; k < UPT; ++k) {
            if (!own[k]) continue;
            const int Ik = I[k], Jk = J[k];
            // expire tabu bits (rare: only when the earliest expiry of this unit is reached)
            if (c >= mexp[k]) {
                unsigned bits = tb[k];
                int32_t nm = MAXV;
                while (bits) {
                    const int q = __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int32_t e = sExp[uidv[k] * 16 + q];
                    if (e <= c) tb[k] &= ~(1u << q);
                    else if (e != MAXV) nm = min(nm, e);
                }
                mexp[k] = nm;
            }
            int32_t kd_best = MAXV;  // PACKED: delta*16+slot; else plain delta
            int slot_best = 0;
            if (Ik != Jk) {
                if (R >= 0) {
                    // ---- generic rank-2 update (a is pre-doubled for symmetric instances)
                    int32_t aI[4], bI[4], aJ[4], bJ[4];
                    ld_vec4(sA, Ik, aI); ld_vec4(sB, Ik, bI); ld_vec4(sA, Jk, aJ); ld_vec4(sB, Jk, bJ);
                    if (SYM) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                U[k][u][v] -= aI[u] * bJ[v];
                                L[k][v][u] -= aJ[v] * bI[u];
                            }
                    } else {
                        int32_t cI[4], eI[4], cJ[4], eJ[4];
                        ld_vec4(sC, Ik, cI); ld_vec4(sE, Ik, eI); ld_vec4(sC, Jk, cJ); ld_vec4(sE, Jk, eJ);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                U[k][u][v] -= aI[u] * bJ[v] + cI[u] * eJ[v];
                                L[k][v][u] -= aJ[v] * bI[u] + cJ[v] * eI[u];
                            }
                    }
                    // ---- rows / columns r and s of the previous move
                    if (Ik == R || Jk == R || Ik == S || Jk == S) {
                        if (Ik == R) {
                            int32_t x[4], cs[4], t[4];
                            ld_vec4(sXR, Jk, x); ld_vec4(sColS, Jk, cs); ld_vec4(sTR, Jk, t);
                            QAPB_SWITCH4(ru, {
_Pragma("unroll")
                                for (int v = 0; v < 4; ++v) { U[k][q][v] += x[v]; L[k][v][q] = cs[v] + t[v]; }
                            })
                        }
                        if (Jk == R) {
                            int32_t x[4], cs[4], t[4];
                            ld_vec4(sXR, Ik, x); ld_vec4(sColS, Ik, cs); ld_vec4(sTR, Ik, t);
                            QAPB_SWITCH4(ru, {
_Pragma("unroll")
                                for (int u = 0; u < 4; ++u) { L[k][q][u] += x[u]; U[k][u][q] = cs[u] + t[u]; }
                            })
                        }
                        if (Ik == S) {
                            int32_t x[4], cr[4], t[4];
                            ld_vec4(sXS, Jk, x); ld_vec4(sColR, Jk, cr); ld_vec4(sTS, Jk, t);
                            QAPB_SWITCH4(su, {
_Pragma("unroll")
                                for (int v = 0; v < 4; ++v) { U[k][q][v] += x[v]; L[k][v][q] = cr[v] + t[v]; }
                            })
                        }
                        if (Jk == S) {
                            int32_t x[4], cr[4], t[4];
                            ld_vec4(sXS, Ik, x); ld_vec4(sColR, Ik, cr); ld_vec4(sTS, Ik, t);
                            QAPB_SWITCH4(su, {
_Pragma("unroll")
                                for (int u = 0; u < 4; ++u) { L[k][q][u] += x[u]; U[k][u][q] = cr[u] + t[u]; }
                            })
                        }
                    }
                }
                // ---- delta, admissibility (_kernels.pyx:162), first minimum.  The ALU pipe (IADD3 /
                // ISETP / IMNMX, half rate) is the busiest pipe of this pass, so the first add of each
                // delta and the (delta, slot) packing are multiplications by the runtime constants 1
                // and 16: they issue as IMAD on the FMA pipe.
                int32_t hI[4], hJ[4];
                ld_vec4(sH, Ik, hI);
                ld_vec4(sH, Jk, hJ);
                const unsigned tbk = tb[k];
                if (PACKED) {
                    int32_t km[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        km[u] = MAXV;
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const int32_t d = (U[k][u][v] * one + L[k][v][u]) - hI[u] - hJ[v];
                            const bool adm = !(tbk & (1u << (u * 4 + v))) || (d < thr);
                            const int32_t kd = (int32_t)((uint32_t)d * (uint32_t)sixteen + (uint32_t)(u * 4 + v));
                            if (adm) km[u] = min(km[u], kd);
                        }
                    }
                    kd_best = min(min(km[0], km[1]), min(km[2], km[3]));
                } else {
                    int32_t rd[4];
                    int rs[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        rd[u] = MAXV;
                        rs[u] = u * 4;
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const int32_t d = (U[k][u][v] * one + L[k][v][u]) - hI[u] - hJ[v];
                            const bool adm = !(tbk & (1u << (u * 4 + v))) || (d < thr);
                            if (adm && d < rd[u]) { rd[u] = d; rs[u] = u * 4 + v; }
                        }
                    }
                    if (rd[1] < rd[0]) { rd[0] = rd[1]; rs[0] = rs[1]; }
                    if (rd[3] < rd[2]) { rd[2] = rd[3]; rs[2] = rs[3]; }
                    if (rd[2] < rd[0]) { rd[0] = rd[2]; rs[0] = rs[2]; }
                    kd_best = rd[0];
                    slot_best = rs[0];
                }
            } else {
                // ---- diagonal block
                if (R >= 0) {
                    int32_t aI[4], bI[4];
                    ld_vec4(sA, Ik, aI); ld_vec4(sB, Ik, bI);
                    if (SYM) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                if (u != v) U[k][u][v] -= aI[u] * bI[v];
                    } else {
                        int32_t cI[4], eI[4];
                        ld_vec4(sC, Ik, cI); ld_vec4(sE, Ik, eI);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                if (u != v) U[k][u][v] -= aI[u] * bI[v] + cI[u] * eI[v];
                    }
                    // column assignments first, then the row increments (x is 0 at the corners)
                    if (Ik == R) {
                        int32_t cs[4], t[4];
                        ld_vec4(sColS, Ik, cs); ld_vec4(sTR, Ik, t);
                        QAPB_SWITCH4(ru, {
_Pragma("unroll")
                            for (int u = 0; u < 4; ++u) if (u != q) U[k][u][q] = cs[u] + t[u];
                        })
                    }
                    if (Ik == S) {
                        int32_t cr[4], t[4];
                        ld_vec4(sColR, Ik, cr); ld_vec4(sTS, Ik, t);
                        QAPB_SWITCH4(su, {
_Pragma("unroll")
                            for (int u = 0; u < 4; ++u) if (u != q) U[k][u][q] = cr[u] + t[u];
                        })
                    }
                    if (Ik == R) {
                        int32_t x[4];
                        ld_vec4(sXR, Ik, x);
                        QAPB_SWITCH4(ru, {
_Pragma("unroll")
                            for (int v = 0; v < 4; ++v) if (v != q) U[k][q][v] += x[v];
                        })
                    }
                    if (Ik == S) {
                        int32_t x[4];
                        ld_vec4(sXS, Ik, x);
                        QAPB_SWITCH4(su, {
_Pragma("unroll")
                            for (int v = 0; v < 4; ++v) if (v != q) U[k][q][v] += x[v];
                        })
                    }
                }
                int32_t hI[4];
                ld_vec4(sH, Ik, hI);
                const unsigned tbk = tb[k];
                int32_t bdv = MAXV;
                int bsl = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = u + 1; v < 4; ++v) {
                        const int32_t d = U[k][u][v] + U[k][v][u] - hI[u] - hI[v];
                        const bool adm = !(tbk & (1u << (u * 4 + v))) || (d < thr);
                        if (adm && d < bdv) { bdv = d; bsl = u * 4 + v; }
                    }
                if (PACKED) kd_best = (bdv == MAXV) ? MAXV : (int32_t)((uint32_t)bdv * 16u + (uint32_t)bsl);
                else { kd_best = bdv; slot_best = bsl; }
            }
            if (kd_best != MAXV) {
                const int32_t dk = PACKED ? (kd_best >> 4) : kd_best;
                const int sk = PACKED ? (kd_best & 15) : slot_best;
                const unsigned key = pair_key(4 * Ik + (sk >> 2), 4 * Jk + (sk & 3), 0);
                if (dk < my_d || (dk == my_d && key < my_key)) { my_d = dk; my_key = key; my_k = k; my_slot = sk; }
            }
        }

        int32_t bd = my_d;
        unsigned bkey = my_key;
        warp_argmin(bd, bkey);
        if (lane == 0) { sRedD[warp] = bd; sRedK[warp] = bkey; }
        __syncthreads();  // ---------------------------------------------- sync #1
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
            int32_t mrs = 0, msr = 0;
            unsigned was = 0;
#pragma unroll
            for (int k = 0; k < UPT; ++k) {
                if (k != my_k) continue;
                mrs = pick16(U[k], ru * 4 + su);
                msr = (I[k] != J[k]) ? pick16(L[k], su * 4 + ru) : pick16(U[k], su * 4 + ru);
                was = (tb[k] >> my_slot) & 1u;
                if (tabu) {
                    const int32_t new_exp = (int32_t)(c + ten);
                    tb[k] |= 1u << my_slot;
                    mexp[k] = min(mexp[k], new_exp);
                    sExp[uidv[k] * 16 + my_slot] = new_exp;
                }
            }
            const int32_t hr = sH[r], hs = sH[s];
            sTS[r] = hr + (Drs - Dsr) * Fpspr;  // M'[r][s]
            sTR[s] = hs + (Dsr - Drs) * Fprps;  // M'[s][r]
            sH[r] = mrs + (Dsr - Drs) * Fprps;
            sH[s] = msr + (Drs - Dsr) * Fpspr;
            if (P.tr_i) {  // trail row (_kernels.pyx:182-187); was_tabu = cells[bi][bj] > c (:171)
                const size_t o = (size_t)b * iters + (c - 1);
                P.tr_i[o] = r; P.tr_j[o] = s; P.tr_d[o] = (int64_t)bd;
                if (P.tr_tabu) P.tr_tabu[o] = (int64_t)was;
            }
            if (tabu && P.cells) {
                int64_t *cz = P.cells + (size_t)b * n * n;
                cz[(size_t)r * n + s] = (int64_t)c + ten;
                cz[(size_t)s * n + r] += 1;
            }
        }
        // ---- owners of columns r and s publish them (colR[r] = colS[s] = 0 by the diagonal lanes)
#pragma unroll
        for (int k = 0; k < UPT; ++k) {
            if (!own[k]) continue;
            const int Ik = I[k], Jk = J[k];
            if (Ik != Jk) {
                if (Jk == R) { QAPB_SWITCH4(ru, { st_vec4(sColR, Ik, U[k][0][q], U[k][1][q], U[k][2][q], U[k][3][q]); }) }
                if (Ik == R) { QAPB_SWITCH4(ru, { st_vec4(sColR, Jk, L[k][0][q], L[k][1][q], L[k][2][q], L[k][3][q]); }) }
                if (Jk == S) { QAPB_SWITCH4(su, { st_vec4(sColS, Ik, U[k][0][q], U[k][1][q], U[k][2][q], U[k][3][q]); }) }
                if (Ik == S) { QAPB_SWITCH4(su, { st_vec4(sColS, Jk, L[k][0][q], L[k][1][q], L[k][2][q], L[k][3][q]); }) }
            } else {
                if (Ik == R) {
                    QAPB_SWITCH4(ru, { st_vec4(sColR, Ik, q == 0 ? 0 : U[k][0][q], q == 1 ? 0 : U[k][1][q], q == 2 ? 0 : U[k][2][q], q == 3 ? 0 : U[k][3][q]); })
                }
                if (Ik == S) {
                    QAPB_SWITCH4(su, { st_vec4(sColS, Ik, q == 0 ? 0 : U[k][0][q], q == 1 ? 0 : U[k][1][q], q == 2 ? 0 : U[k][2][q], q == 3 ? 0 : U[k][3][q]); })
                }
            }
        }
        __syncthreads();  // ---------------------------------------------- sync #2
        if (tid == 0) { sP[r] = ps; sP[s] = pr; }
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
