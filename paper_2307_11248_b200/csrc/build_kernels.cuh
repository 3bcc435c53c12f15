// build_kernels.cuh -- start generation and the O(n^3) construction of the placement matrix.
//
//   qap_start_kernel      per start: derive_seed (rng.py:62-70), Fisher-Yates shuffle
//                         (core.py:81-87, rng.py:55-59) -> int32 permutation + stream state,
//                         or conversion of caller-provided int64 permutations.
//   qap_build_m_kernel    M[b] = W + D0.Fp^T-type products (see search_kernel.cuh header) for a
//                         batch of permutations: a tiled integer matrix product -- 64x64 output
//                         tile per CTA, 4x4 micro-tile per thread, k-chunks of 32 staged in shared
//                         memory.  A-tiles are rows of D^T / D (coalesced, already k-major),
//                         B-tiles are rows p_k of F^T / F gathered at columns p_j.  This is the
//                         full evaluator of kernels.all_deltas expressed as a contraction, which
//                         is exactly how the reference's NumPy backend states it
//                         (_purekernels.py:25-56: P = D Fp^T, Q = D^T Fp).
#pragma once
#include "search_kernel.cuh"

namespace qapb {

struct StartParams {
    int n, npad, rng, force_seq_rng;
    unsigned long long master_seed, first_index;
    const unsigned long long *seeds; // [B] explicit per-start states (rng == 1), or null: derive_seed(master, first + b)
    const int64_t *perms;            // [B,n] (rng == 0)
    int32_t *perm32;                 // [B,npad] out
    unsigned long long *state;       // [B] out: SplitMix64 state after the shuffle
};

__global__ void __launch_bounds__(128) qap_start_kernel(const StartParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int32_t *sP = reinterpret_cast<int32_t *>(smem_raw);
    unsigned *sJ = reinterpret_cast<unsigned *>(smem_raw) + P.npad;
    const int tid = threadIdx.x, T = blockDim.x, b = blockIdx.x, n = P.n;
    for (int i = tid; i < P.npad; i += T)
        sP[i] = (P.rng || i >= n) ? (i < n ? i : 0) : (int32_t)P.perms[(size_t)b * n + i];
    unsigned long long st = 0;
    if (P.rng) {
        // draws computed in parallel assuming no rejection; a rejection (probability ~ n^2/2^64)
        // falls back to the exact sequential loop
        const unsigned long long seed =
            P.seeds ? P.seeds[b] : mix64(P.master_seed + QAPB_GAMMA * (P.first_index + (unsigned long long)b + 1ULL));
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
            st = seed;
            if (reject) {
                for (int i = n - 1; i >= 1; --i) {
                    unsigned j = (unsigned)randbelow_seq(st, (unsigned long long)i + 1ULL);
                    int32_t t = sP[i]; sP[i] = sP[j]; sP[j] = t;
                }
            } else {
                for (int i = n - 1; i >= 1; --i) {
                    unsigned j = sJ[i];
                    int32_t t = sP[i]; sP[i] = sP[j]; sP[j] = t;
                }
                st = seed + QAPB_GAMMA * (unsigned long long)(n - 1);
            }
            P.state[b] = st;
        }
    }
    __syncthreads();
    for (int i = tid; i < P.npad; i += T) P.perm32[(size_t)b * P.npad + i] = sP[i];
}

struct BuildParams {
    int n, npad, symmetric;
    const int32_t *F, *FT, *D, *DT, *fd, *dd;
    const int32_t *perm32;           // [B,npad]
    void *M;                         // [B,npad,npad] out (row-major; pads = 2^29 / 2^61, diagonal 0), int32 or int64
    void *h;                         // [B,npad] out
};

enum { BK = 32 };

// Output tile edge of qap_build_m_kernel: the one of {64, 52, 32} that wastes the least work on
// npad (n = 100: 2 x 2 tiles of 52 cover 104 instead of 128 columns -- 1.08x instead of 1.64x the
// useful multiply-adds).  Threads per CTA = (BT / 4)^2, rounded up to a warp multiple.
__host__ __device__ inline int build_tile(int npad)
{
    const int cand[3] = {64, 52, 32};
    int best = 64;
    long long best_cost = -1;
    for (int k = 0; k < 3; ++k) {
        const long long tiles = (npad + cand[k] - 1) / cand[k], cost = tiles * cand[k];
        if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = cand[k]; }
    }
    return best;
}

__device__ __forceinline__ void st_acc4(int32_t *dst, const int32_t (&v)[4])
{
    *reinterpret_cast<int4 *>(dst) = make_int4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void st_acc4(int64_t *dst, const int64_t (&v)[4])
{
    reinterpret_cast<longlong2 *>(dst)[0] = make_longlong2(v[0], v[1]);
    reinterpret_cast<longlong2 *>(dst)[1] = make_longlong2(v[2], v[3]);
}

template <typename acc_t, int BT>
__global__ void __launch_bounds__(256) qap_build_m_kernel(const BuildParams P)
{
    __shared__ __align__(16) int32_t sA[2][BK][BT];  // [term][k][i]
    __shared__ __align__(16) int32_t sB[2][BK][BT];  // [term][k][j]
    constexpr int TW = BT / 4;                         // micro-tiles per tile edge
    const int NT = blockDim.x;
    __shared__ int32_t sPk[BK];
    extern __shared__ __align__(16) unsigned char dyn[];
    int32_t *sPerm = reinterpret_cast<int32_t *>(dyn);  // [npad]
    const int tid = threadIdx.x;
    const int n = P.n, npad = P.npad;
    const int tiles = (npad + BT - 1) / BT;
    const int b = blockIdx.x / (tiles * tiles), tt = blockIdx.x % (tiles * tiles);  // batch on grid.x (no 65535 limit)
    const int ti = tt / tiles, tj = tt % tiles;
    const int i0 = ti * BT, j0 = tj * BT;
    const int32_t *perm = P.perm32 + (size_t)b * npad;
    for (int i = tid; i < npad; i += NT) sPerm[i] = perm[i];
    __syncthreads();
    const bool sym = P.symmetric != 0;
    const int ty = tid / TW, tx = tid % TW;  // micro-tile rows 4*ty.., cols 4*tx..
    const bool active = ty < TW;
    acc_t acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0;

    for (int k0 = 0; k0 < n; k0 += BK) {
        // stage: A[k][i] = D0[i0+i][k0+k] (= row k0+k of D^T), B[k][j] = F0[p_j][p_k] (= row p_k of F^T
        // gathered at p_j); second term (asymmetric only): A2 = D0[k][i] (row of D), B2 = F0[p_k][p_j]
        if (tid < BK) sPk[tid] = (k0 + tid < n) ? sPerm[k0 + tid] : 0;
        __syncthreads();
        for (int e = tid; e < BK * BT; e += NT) {
            const int k = e / BT, x = e % BT;
            const int kk = k0 + k;
            const bool kin = kk < n;
            const int gi = i0 + x, gj = j0 + x;
            const int pk = sPk[k];
            const int pj = (gj < npad) ? sPerm[gj] : 0;
            sA[0][k][x] = (kin && gi < npad) ? P.DT[(size_t)kk * npad + gi] : 0;
            sB[0][k][x] = (kin && gj < n) ? P.FT[(size_t)pk * npad + pj] : 0;
            if (!sym) {
                sA[1][k][x] = (kin && gi < npad) ? P.D[(size_t)kk * npad + gi] : 0;
                sB[1][k][x] = (kin && gj < n) ? P.F[(size_t)pk * npad + pj] : 0;
            }
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < BK && active; ++k) {
            const int4 a = *reinterpret_cast<const int4 *>(&sA[0][k][4 * ty]);
            const int4 bq = *reinterpret_cast<const int4 *>(&sB[0][k][4 * tx]);
            const int32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {bq.x, bq.y, bq.z, bq.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] += (acc_t)av[u] * (acc_t)bv[v];
            if (!sym) {
                const int4 a2 = *reinterpret_cast<const int4 *>(&sA[1][k][4 * ty]);
                const int4 b2 = *reinterpret_cast<const int4 *>(&sB[1][k][4 * tx]);
                const int32_t av2[4] = {a2.x, a2.y, a2.z, a2.w}, bv2[4] = {b2.x, b2.y, b2.z, b2.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] += (acc_t)av2[u] * (acc_t)bv2[v];
            }
        }
        __syncthreads();
    }
    // epilogue: direct term, diagonal products, pads, h on the diagonal
    acc_t *Mb = reinterpret_cast<acc_t *>(P.M) + (size_t)b * npad * npad;
    acc_t *hb = reinterpret_cast<acc_t *>(P.h) + (size_t)b * npad;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int i = i0 + 4 * ty + u;
        if (i >= npad || !active) continue;
        acc_t out[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int j = j0 + 4 * tx + v;
            acc_t val = sym ? 2 * acc[u][v] : acc[u][v];
            if (j < npad) {
                if (i >= n || j >= n) {
                    val = (i == j) ? (acc_t)0 : Acc<acc_t>::bighalf();
                } else {
                    const int pi = sPerm[i], pj = sPerm[j];
                    if (i == j) {
                        hb[i] = val + (acc_t)P.dd[i] * (acc_t)P.fd[pi];
                        val = 0;
                    } else {
                        val += (acc_t)P.D[(size_t)i * npad + j] *
                                   ((acc_t)P.F[(size_t)pi * npad + pj] + (acc_t)P.F[(size_t)pj * npad + pi]) +
                               (acc_t)P.dd[i] * (acc_t)P.fd[pj];
                    }
                }
            }
            out[v] = val;
        }
        const int jb = j0 + 4 * tx;
        if (jb < npad) st_acc4(&Mb[(size_t)i * npad + jb], out);
    }
    if (ti == 0 && tj == 0)
        for (int i = n + tid; i < npad; i += NT) hb[i] = 0;
}

// The same contraction for npad <= 128 with the WHOLE problem of one permutation in one CTA: D^T (40 KB at
// n = 100) and the gathered G[k][j] = F0[p_j][p_k] are staged in shared memory ONCE -- straight 128-bit row
// copies and one gather per entry, instead of re-staging both per 52 x 52 tile and per 32-wide k-chunk with
// two barriers each -- and every thread then runs all n k-steps on an 8 x 4 register tile: three 128-bit
// shared loads feed 32 IMADs per step.  (Asymmetric instances make a second pass with D and F0[p_k][p_j].)
// EMIT (kernels.all_deltas): instead of writing M and h for a search kernel, the CTA parks them in its own
// shared memory (row stride npad + 1: the column reads M[j][i] are conflict-free) and writes the n(n-1)/2
// deltas M[i][j] + M[j][i] - h[i] - h[j] in lexicographic order straight away -- no M round trip through
// global memory and no second kernel.
// (MAXT / MINB: up to 352 threads -- n <= 104 -- two CTAs share an SM, so the register budget is 88.)
template <typename acc_t, bool EMIT, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) qap_build_m_whole_kernel(const BuildParams P, int64_t *__restrict__ deltas)
{
    extern __shared__ __align__(16) unsigned char dyn[];
    const int n = P.n, npad = P.npad, tid = threadIdx.x, NT = blockDim.x, b = blockIdx.x;
    int32_t *sA = reinterpret_cast<int32_t *>(dyn);                 // [npad][npad] (+8 words of slack)
    int32_t *sB = sA + (size_t)npad * npad + 8;                      // [npad][npad]
    int32_t *sPerm = sB + (size_t)npad * npad + 8;                   // [npad]
    const int32_t *perm = P.perm32 + (size_t)b * npad;
    for (int i = tid; i < npad; i += NT) sPerm[i] = perm[i];
    __syncthreads();
    const int CG = npad >> 2;                                        // 4-column groups
    const int rg = tid / CG, cg = tid - rg * CG;                     // rows 8 rg .., columns 4 cg ..
    const bool active = 8 * rg < npad;
    const bool sym = P.symmetric != 0;
    acc_t acc[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0;
    const int nvec = (npad * npad) >> 2;
    for (int pass = 0; pass < (sym ? 1 : 2); ++pass) {
        const int32_t *Asrc = pass == 0 ? P.DT : P.D;                // A[k][i] = D0[i][k]  |  D0[k][i]
        const int32_t *Bsrc = pass == 0 ? P.FT : P.F;                // B[k][j] = F0[p_j][p_k]  |  F0[p_k][p_j]
        if (pass) __syncthreads();
        for (int e = tid; e < nvec; e += NT) reinterpret_cast<int4 *>(sA)[e] = reinterpret_cast<const int4 *>(Asrc)[e];
        for (int e = tid; e < nvec; e += NT) {
            const int k = (4 * e) / npad, j = 4 * e - k * npad;
            const int32_t *row = Bsrc + (size_t)sPerm[k] * npad;
            const bool kin = k < n;
            reinterpret_cast<int4 *>(sB)[e] = make_int4((kin && j < n) ? row[sPerm[j]] : 0, (kin && j + 1 < n) ? row[sPerm[j + 1]] : 0,
                                                        (kin && j + 2 < n) ? row[sPerm[j + 2]] : 0, (kin && j + 3 < n) ? row[sPerm[j + 3]] : 0);
        }
        __syncthreads();
        if (active) {
            const int32_t *pa = sA + 8 * rg, *pb = sB + 4 * cg;
            // software pipeline: the operands of step k + 1 are in flight while the 32 IMADs of step k issue
            int4 a0 = *reinterpret_cast<const int4 *>(pa), a1 = *reinterpret_cast<const int4 *>(pa + 4);
            int4 bq = *reinterpret_cast<const int4 *>(pb);
#pragma unroll 2
            for (int k = 0; k < n; ++k) {
                const int kn = (k + 1 < n) ? k + 1 : k;
                const int4 a0n = *reinterpret_cast<const int4 *>(pa + kn * npad);
                const int4 a1n = *reinterpret_cast<const int4 *>(pa + kn * npad + 4);
                const int4 bqn = *reinterpret_cast<const int4 *>(pb + kn * npad);
                const int32_t av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w}, bv[4] = {bq.x, bq.y, bq.z, bq.w};
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] += (acc_t)av[u] * (acc_t)bv[v];
                a0 = a0n; a1 = a1n; bq = bqn;
            }
        }
    }
    // epilogue: direct term, diagonal products, pads, h on the diagonal.  The matrix entries it needs are in
    // shared memory already: after the last pass sA[i][j] = D0[i][j] and sB[i][j] = F0[p_i][p_j] (by symmetry in
    // the one-pass case), so the direct term D0[i][j] (F0[p_i][p_j] + F0[p_j][p_i]) costs 128-bit shared loads
    // instead of three dependent global loads per entry (they were over half of the kernel's time).
    const int ldm = EMIT ? npad + 1 : npad;
    acc_t *Mb = EMIT ? reinterpret_cast<acc_t *>(dyn) : reinterpret_cast<acc_t *>(P.M) + (size_t)b * npad * npad;
    acc_t *hb = EMIT ? Mb + (size_t)npad * ldm : reinterpret_cast<acc_t *>(P.h) + (size_t)b * npad;
    acc_t hdiag[8];
    if (active) {
        int32_t fdj[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) fdj[v] = (4 * cg + v < n) ? P.fd[sPerm[4 * cg + v]] : 0;
        int32_t ft[4][8];  // F0[p_j][p_i] for the thread's 4 columns j and 8 rows i
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int4 t0 = *reinterpret_cast<const int4 *>(sB + (size_t)(4 * cg + v) * npad + 8 * rg);
            const int4 t1 = *reinterpret_cast<const int4 *>(sB + (size_t)(4 * cg + v) * npad + 8 * rg + 4);
            ft[v][0] = t0.x; ft[v][1] = t0.y; ft[v][2] = t0.z; ft[v][3] = t0.w;
            ft[v][4] = t1.x; ft[v][5] = t1.y; ft[v][6] = t1.z; ft[v][7] = t1.w;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = 8 * rg + u;
            hdiag[u] = 0;
            if (i >= npad) continue;
            const int4 d4 = *reinterpret_cast<const int4 *>(sA + (size_t)i * npad + 4 * cg);
            const int4 f4 = *reinterpret_cast<const int4 *>(sB + (size_t)i * npad + 4 * cg);
            const int32_t dv[4] = {d4.x, d4.y, d4.z, d4.w}, fv[4] = {f4.x, f4.y, f4.z, f4.w};
            const int32_t ddi = i < n ? P.dd[i] : 0;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int j = 4 * cg + v;
                acc_t val = sym ? 2 * acc[u][v] : acc[u][v];
                if (i >= n || j >= n) {
                    val = (i == j) ? (acc_t)0 : Acc<acc_t>::bighalf();
                } else if (i == j) {
                    hdiag[u] = val + (acc_t)ddi * (acc_t)fdj[v];
                    val = 0;
                } else {
                    val += (acc_t)dv[v] * ((acc_t)fv[v] + (acc_t)ft[v][u]) + (acc_t)ddi * (acc_t)fdj[v];
                }
                acc[u][v] = val;
            }
        }
    }
    if (EMIT) __syncthreads();  // every thread is done with sA / sB / sPerm: M may be parked over them
    if (active) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = 8 * rg + u;
            if (i >= npad) continue;
            if (i < n && (i >> 2) == cg) hb[i] = hdiag[u];  // the thread that holds the diagonal entry of row i
            if (EMIT) {
#pragma unroll
                for (int v = 0; v < 4; ++v) Mb[(size_t)i * ldm + 4 * cg + v] = acc[u][v];
            } else {
                st_acc4(&Mb[(size_t)i * npad + 4 * cg], acc[u]);
            }
        }
    }
    for (int i = n + tid; i < npad; i += NT) hb[i] = 0;
    if (EMIT) {
        __syncthreads();
        const int npairs = n * (n - 1) / 2;
        int64_t *ob = deltas + (size_t)b * npairs;
        int i = 0, j = tid + 1;  // pair number k in row-major order of the upper triangle: row i holds j = i+1 .. n-1
        for (int k = tid; k < npairs; k += NT) {
            while (j >= n) { j = j - n + (i + 2); ++i; }  // carry into the following rows
            ob[k] = (int64_t)(Mb[(size_t)i * ldm + j] + Mb[(size_t)j * ldm + i] - hb[i] - hb[j]);
            j += NT;
        }
    }
}

// kernels.all_deltas (_kernels.pyx:58-70) from M and h: out[b][k] = M[i][j] + M[j][i] - h[i] - h[j]
// for the n(n-1)/2 moves in lexicographic (i, j) order, widened to int64.
template <typename acc_t>
__global__ void __launch_bounds__(256) qap_emit_deltas_kernel(int n, int npad, const void *__restrict__ Mv,
                                                              const void *__restrict__ hv, int64_t *__restrict__ out)
{
    const int b = blockIdx.x;
    const acc_t *Mb = reinterpret_cast<const acc_t *>(Mv) + (size_t)b * npad * npad;
    const acc_t *hb = reinterpret_cast<const acc_t *>(hv) + (size_t)b * npad;
    int64_t *ob = out + (size_t)b * ((size_t)n * (n - 1) / 2);
    for (int i = blockIdx.y; i < n - 1; i += gridDim.y) {
        const size_t row0 = (size_t)i * n - ((size_t)i * (i + 1)) / 2 - (size_t)(i + 1);  // + j gives the index
        const acc_t hi = hb[i];
        for (int j = i + 1 + threadIdx.x; j < n; j += blockDim.x)
            ob[row0 + j] = (int64_t)(Mb[(size_t)i * npad + j] + Mb[(size_t)j * npad + i] - hi - hb[j]);
    }
}

}  // namespace qapb
