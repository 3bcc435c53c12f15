// search_warp.cuh -- one WARP per search, n <= 32 (nug12, tai30a: BASELINE configs[0] and configs[1]).
//
// The hybrid kernel (search_hybrid.cuh) spreads a search over a CTA and pays two block barriers, a
// two-level argmin and register-indexed fix-up regions per iteration; at n <= 32 a whole search is 28
// off-diagonal units, so that machinery is all that is left of the iteration.  Here a search is one warp
// and nothing but warp-synchronous code:
//   * lane l is LOCATION l for the publish phase (p[l], h[l] live in its registers), off-diagonal UNIT l
//     (block pair {(I,J),(J,I)}, lexicographic over I < J, 16 pairs) for the pass, and the owner of the
//     diagonal-block pairs l and l + 32 (of 6 per diagonal block), one scalar pair at a time -- every lane
//     runs the same instruction stream, there is no diagonal warp or diagonal path to diverge into;
//   * the placement matrix lives in the warp's slice of shared memory: off-diagonal units in the private
//     layout of the generic kernel (row w of unit l at (w*32 + l)*16 bytes: conflict-free 128-bit LDS/STS),
//     diagonal blocks as plain 4x4 tiles.  Addresses are free to index at run time, so the 4n entries on
//     rows/columns r,s are fixed in place by the lane of their location -- four loads, four stores -- with no
//     column dump, no fix-up vectors and no register-indexed switch;
//   * the argmin is two `redux.sync`; the two barriers of an iteration are `__syncwarp()`;
//   * tenures are drawn 32 at a time, one per lane (exact sequential replay on a rejected draw), and the
//     tenure of an iteration comes out of its lane by shuffle;
//   * searches share nothing, so any number of them can be packed into a CTA (blockDim.x / 32).
// Same integers as every other plan: the formulas of the publish phase are the ones of search_hybrid.cuh.
// int32 state with packed selection keys only (|delta| < 2^27, host-proven); other instances of this size
// keep the hybrid plans.
#pragma once
#include "search_hybrid.cuh"

namespace qapb {

enum {
    WK_M = 0,          // 8 rows x 32 lanes x 16 B: off-diagonal units (rows 0-3: upper block, 4-7: lower block transposed)
    WK_DG = 4096,      // 8 diagonal blocks x 16 words
    WK_XP = 4608,      // 32 units x 16 words: tabu expiry per (unit, slot)
    WK_A = 6656,       // difference vectors of the last move (negated a, c), 32 words each
    WK_B = 6784,
    WK_C = 6912,
    WK_E = 7040,
    WK_HI = 7168,      // packed-key forms of h (search_hybrid.cuh)
    WK_HJ = 7296,
    WK_P = 7424,       // permutation (setup only)
    WK_TOTAL = 7552
};

// word offset (in the warp's slice) of M[x][y] and M[y][x] for location x = this lane and the moved
// location y = 4 Y + yu; X == Y is the diagonal block.  One unit holds both entries, 512 words apart.
__device__ __forceinline__ void wk_pair_words(int X, int xu, int Y, int yu, int nb, int &w_xy, int &w_yx)
{
    const bool up = X < Y;
    const int I = up ? X : Y, J = up ? Y : X;
    const int uid = I * nb - ((I * (I + 1)) >> 1) + (J - I - 1);
    // X < Y: M[x][y] = U[xu][yu] (row xu, column yu), M[y][x] = L[yu][xu] (row 4 + xu, column yu)
    // X > Y: M[y][x] = U[yu][xu] (row yu, column xu), M[x][y] = L[xu][yu] (row 4 + yu, column xu)
    const int row = up ? xu : yu, col = up ? yu : xu;
    const int wU = (row * 32 + uid) * 4 + col;
    w_xy = up ? wU : wU + 512;
    w_yx = up ? wU + 512 : wU;
    if (X == Y) {
        w_xy = WK_DG / 4 + X * 16 + xu * 4 + yu;
        w_yx = WK_DG / 4 + X * 16 + yu * 4 + xu;
    }
}

// 32 tenures (tabu.py:184-186), one per lane: draw k of the chunk is mix64(state + (k+1)*GAMMA); a draw that
// randbelow would reject (probability ~ span / 2^64) makes every lane replay the chunk with the exact rule.
__device__ __forceinline__ int32_t warp_tenure_chunk(unsigned long long &state, unsigned long long span,
                                                     unsigned long long last_ok, long long lo, int force_seq, int lane)
{
    const unsigned long long r = mix64(state + QAPB_GAMMA * ((unsigned long long)lane + 1ULL));
    int32_t t = 0;
    if (__any_sync(0xffffffffu, (r > last_ok) || force_seq)) {
        unsigned long long st = state;
        for (int k = 0; k < 32; ++k) {
            const int32_t v = (int32_t)(lo + (long long)randbelow_seq(st, span));
            if (k == lane) t = v;
        }
        state = st;
    } else {
        t = (int32_t)(lo + (long long)(r % span));
        state += QAPB_GAMMA * 32ULL;
    }
    return t;
}

// SYMM: 1 = both matrices symmetric (one product per entry), 0 = the general two-product update.
// NOTABU: 2opt instantiation (no tabu state at all).  REC: trail / cells / caller-provided tenures.
template <int SYMM, bool NOTABU, bool REC>
__global__ void __launch_bounds__(256) qap_search_warp_kernel(const SearchParams P)
{
    constexpr bool FULLSYM = SYMM == 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= P.batch) return;  // whole warps only
    unsigned char *W = smem_raw + (size_t)(threadIdx.x >> 5) * WK_TOTAL;
    int32_t *sW = reinterpret_cast<int32_t *>(W);
    int32_t *sM = reinterpret_cast<int32_t *>(W + WK_M);
    int32_t *sDG = reinterpret_cast<int32_t *>(W + WK_DG);
    int32_t *xp = reinterpret_cast<int32_t *>(W + WK_XP);
    int32_t *sP = reinterpret_cast<int32_t *>(W + WK_P);
    Vecs V;
    V.A = reinterpret_cast<int32_t *>(W + WK_A);
    V.B = reinterpret_cast<int32_t *>(W + WK_B);
    V.C = reinterpret_cast<int32_t *>(W + WK_C);
    V.E = reinterpret_cast<int32_t *>(W + WK_E);
    V.HI = reinterpret_cast<int32_t *>(W + WK_HI);
    V.HJ = reinterpret_cast<int32_t *>(W + WK_HJ);
    V.H = V.ColR = V.ColS = V.TR = V.TS = V.XR = V.XS = nullptr;

    const int n = P.n, nb = P.nb, npad = P.npad, noff = P.noff;
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
    const bool loc = lane < n;          // this lane is a location
    const int X = lane >> 2, xu = lane & 3;
    int my_p = lane < npad ? P.perm32[(size_t)b * npad + lane] : 0;
    int32_t h = lane < npad ? reinterpret_cast<const int32_t *>(P.initH)[(size_t)b * npad + lane] : 0;
    V.A[lane] = 0; V.B[lane] = 0; V.C[lane] = 0; V.E[lane] = 0;
    V.HI[lane] = 4 * xu - 16 * h;
    V.HJ[lane] = xu - 16 * h;
    sP[lane] = my_p;
    if (REC && P.cells) {
        int64_t *cz = P.cells + (size_t)b * n * n;
        for (int i = lane; i < n * n; i += 32) cz[i] = 0;
    }
    const int32_t *__restrict__ Minit = reinterpret_cast<const int32_t *>(P.initM) + (size_t)b * npad * npad;

    // off-diagonal unit of this lane (lexicographic over I < J)
    const bool own = lane < noff;
    int I = 0, J = 1;
    if (own) {
        int rem = lane;
        while (rem >= nb - 1 - I) { rem -= nb - 1 - I; ++I; }
        J = I + 1 + rem;
    }
    unsigned tb = 0xffffu;
    int32_t mexp = MAXV;
    {
        int32_t U[4][4], L[4][4];
        unsigned dead = 0xffffu;
        if (own) load_unit(Minit, npad, n, I, J, U, L, dead, PADV);
        else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) { U[u][v] = PADV; L[u][v] = PADV; }
        }
        tb = dead;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            reinterpret_cast<int4 *>(sM)[u * 32 + lane] = make_int4(U[u][0], U[u][1], U[u][2], U[u][3]);
            reinterpret_cast<int4 *>(sM)[(4 + u) * 32 + lane] = make_int4(L[0][u], L[1][u], L[2][u], L[3][u]);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) xp[lane * 16 + q] = ((dead >> q) & 1u) ? MAXV : 0;
    }
    if (lane < nb) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) sDG[lane * 16 + u * 4 + v] = Minit[(size_t)(4 * lane + u) * npad + 4 * lane + v];
    }
    // diagonal-block pairs lane and lane + 32 (pair pp of block Bk: (0,1) (0,2) (0,3) (1,2) (1,3) (2,3))
    int di[2], dj[2], dwx[2], dwy[2];
    bool dalive[2];
    int32_t dexp[2] = {0, 0};  // expiry iteration of the pair (cells[i][j]); 0 = never tabu
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int idx = lane + 32 * q;
        const int Bk = idx / 6, pp = idx - 6 * Bk;
        const int u = pp < 3 ? 0 : pp < 5 ? 1 : 2;
        const int v = pp < 3 ? pp + 1 : pp < 5 ? pp - 1 : 3;
        di[q] = 4 * Bk + u; dj[q] = 4 * Bk + v;
        dalive[q] = idx < 6 * nb && dj[q] < n;
        if (!dalive[q]) { di[q] = 0; dj[q] = 1; }
        dwx[q] = (di[q] >> 2) * 16 + (di[q] & 3) * 4 + (dj[q] & 3);
        dwy[q] = (di[q] >> 2) * 16 + (dj[q] & 3) * 4 + (di[q] & 3);
    }
    __syncwarp();

    long long cost;  // _kernels.pyx:18-24, int64, including the diagonal products
    {
        long long part = 0;
        if (loc) {
            for (int j = 0; j < n; ++j) {
                const int pj = sP[j];
                part += (j == lane) ? (long long)P.fd[my_p] * P.dd[lane] : (long long)F[my_p * npad + pj] * D[lane * npad + j];
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(FULL, part, off);
        cost = part;
    }
    long long best_cost = cost;
    int32_t thr = 0;  // best_cost - cost, clamped; aspiration <=> delta < thr  (_kernels.pyx:162)
    int best_p = my_p;
    int steps_done = 0, stopped = 0;
    unsigned long long rstate = (tabu && P.rng) ? P.start_state[b] : 0ULL;
    const unsigned long long span = (unsigned long long)(P.ten_hi - P.ten_lo + 1);
    const unsigned long long last_ok = (tabu && P.rng) ? ~0ULL - (0ULL - span) % span : 0ULL;
    int32_t my_ten = 0;

    for (int c = 1; c <= iters; ++c) {
        if (tabu && ((c - 1) & 31) == 0) {
            if (P.rng) my_ten = warp_tenure_chunk(rstate, span, last_ok, P.ten_lo, P.force_seq_rng, lane);
            else if (REC) my_ten = (c - 1 + lane < iters) ? (int32_t)P.tenures[(size_t)b * iters + (c - 1 + lane)] : 0;
        }
        // ---------------- pass: rank-2 update of the previous move (the difference vectors are zero at its
        // two locations and before the first move), delta, admissibility, first minimum
        int32_t my_d;
        unsigned my_key;
        int my_which = 0, my_slot = 0;  // 0: the off-diagonal unit, 1 / 2: diagonal pair q = 0 / 1
        {
            int32_t U[4][4], L[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int4 a = reinterpret_cast<const int4 *>(sM)[u * 32 + lane];
                const int4 l = reinterpret_cast<const int4 *>(sM)[(4 + u) * 32 + lane];
                U[u][0] = a.x; U[u][1] = a.y; U[u][2] = a.z; U[u][3] = a.w;
                L[0][u] = l.x; L[1][u] = l.y; L[2][u] = l.z; L[3][u] = l.w;
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
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                reinterpret_cast<int4 *>(sM)[u * 32 + lane] = make_int4(U[u][0], U[u][1], U[u][2], U[u][3]);
                reinterpret_cast<int4 *>(sM)[(4 + u) * 32 + lane] = make_int4(L[0][u], L[1][u], L[2][u], L[3][u]);
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
            int32_t x = sDG[dwx[q]], y = sDG[dwy[q]];
            const int32_t ai = V.A[di[q]], bj = V.B[dj[q]], aj = V.A[dj[q]], bi = V.B[di[q]];
            x += ai * bj;
            y += aj * bi;
            if (!FULLSYM) {
                const int32_t ci = V.C[di[q]], ej = V.E[dj[q]], cj = V.C[dj[q]], ei = V.E[di[q]];
                x += ci * ej;
                y += cj * ei;
            }
            const int32_t hi = __shfl_sync(FULL, h, di[q]), hj = __shfl_sync(FULL, h, dj[q]);
            if (dalive[q]) { sDG[dwx[q]] = x; sDG[dwy[q]] = y; }
            const int32_t d = x + y - hi - hj;
            const bool adm = dalive[q] && (NOTABU || dexp[q] <= c || d < thr);
            const unsigned key = pair_key(di[q], dj[q], 0);
            if (adm && (d < my_d || (d == my_d && key < my_key))) { my_d = d; my_key = key; my_which = 1 + q; }
        }
        int32_t bd = my_d;
        unsigned bkey = my_key;
        warp_argmin(bd, bkey);
        if (bd == MAXV) {  // no admissible move: premature stop (_kernels.pyx:168-170)
            stopped = 1;
            break;
        }
        const int r = (int)(bkey >> 17), s = (int)((bkey >> 1) & 0xffffu);
        cost += (long long)bd;
        const bool improved = cost < best_cost;
        if (improved) best_cost = cost;
        thr = Acc<int32_t>::clamp_thr(best_cost - cost);
        steps_done = c;
        const bool is_winner = my_key == bkey;
        const int pr = __shfl_sync(FULL, my_p, r), ps = __shfl_sync(FULL, my_p, s);
        const int32_t hr = __shfl_sync(FULL, h, r), hs = __shfl_sync(FULL, h, s);
        const int32_t ten = tabu ? __shfl_sync(FULL, my_ten, (c - 1) & 31) : 0;
        __syncwarp();  // ------------------------------------------------ sync #1: the pass has stored M

        // ---------------- publish: difference vectors of the move (old permutation), h', and the entries on
        // rows / columns r,s of M fixed in place by the lane of their location
        const int R = r >> 2, S = s >> 2, ru = r & 3, su = s & 3;
        const int i = loc ? lane : 0;
        const int pi = loc ? my_p : 0;
        const bool mid = loc && (lane != r) && (lane != s);
        int w_ir, w_ri, w_is, w_si;
        wk_pair_words(X, xu, R, ru, nb, w_ir, w_ri);
        wk_pair_words(X, xu, S, su, nb, w_is, w_si);
        int32_t m_ir = 0, m_ri = 0, m_is = 0, m_si = 0;
        if (mid) { m_ir = sW[w_ir]; m_ri = sW[w_ri]; m_is = sW[w_is]; m_si = sW[w_si]; }
        if (loc && lane == r) m_is = sW[w_is];  // M[r][s]
        if (loc && lane == s) m_ir = sW[w_ir];  // M[s][r]
        int32_t kr = 0, ks = 0;  // corner terms, zero when both matrices are symmetric
        if (FULLSYM) {
            const int32_t Drs = D[r * npad + s], Fpspr = F[ps * npad + pr];
            const int32_t Dsi = D[s * npad + i], Dri = D[r * npad + i];
            const int32_t Fpspi = F[ps * npad + pi], Fprpi = F[pr * npad + pi];
            const int32_t a = mid ? Dsi - Dri : 0, bb = mid ? Fpspi - Fprpi : 0;
            const int32_t a2 = 2 * a, b2 = 2 * bb;
            V.A[lane] = -a2;
            V.B[lane] = bb;
            if (mid) {
                h -= a2 * bb;
                sW[w_ir] = m_is + a2 * (Fpspr - Fpspi);        // M'[i][r] = M[i][s] + tR[i]
                sW[w_is] = m_ir + a2 * (Fprpi - Fpspr);        // M'[i][s] = M[i][r] + tS[i]
                sW[w_ri] = m_ri + b2 * (Dri - Drs);            // M'[r][i] = M[r][i] + xR[i]
                sW[w_si] = m_si + b2 * (Drs - Dsi);            // M'[s][i] = M[s][i] + xS[i]
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
            V.A[lane] = -a;
            V.B[lane] = bb;
            V.C[lane] = -cc;
            V.E[lane] = e;
            kr = (Drs - Dsr) * Fpspr;
            ks = (Dsr - Drs) * Fprps;
            if (mid) {
                h -= a * bb + cc * e;
                sW[w_ir] = m_is + a * (Fpspr - (Fpips + Fpspi)) + cc * Fprps;
                sW[w_is] = m_ir + a * ((Fpipr + Fprpi) - Fprps) - cc * Fpspr;
                sW[w_ri] = m_ri - Drs * bb - Dsr * e + Dri * be;
                sW[w_si] = m_si + Dsr * bb + Drs * e - Dsi * be;
            }
        }
        // corners: M'[r][s] = h[r] + kr, h'[r] = M[r][s] + ks;  M'[s][r] = h[s] + ks, h'[s] = M[s][r] + kr
        if (loc && lane == r) { sW[w_is] = hr + kr; h = m_is + ks; }
        if (loc && lane == s) { sW[w_ir] = hs + ks; h = m_ir + kr; }
        V.HI[lane] = 4 * xu - 16 * h;
        V.HJ[lane] = xu - 16 * h;
        my_p = (lane == r) ? ps : (lane == s) ? pr : my_p;
        if (improved) best_p = my_p;

        // ---- the lane owning the winning pair: tabu memory, trail
        if (is_winner) {
            const int32_t new_exp = (int32_t)(c + ten);
            unsigned was = 0;
            if (my_which == 0) {
                was = (tb >> my_slot) & 1u;
                if (tabu) {
                    tb |= 1u << my_slot;
                    mexp = min(mexp, new_exp);
                    xp[lane * 16 + my_slot] = new_exp;
                }
            } else {
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    if (my_which == 1 + q) {
                        was = dexp[q] > c ? 1u : 0u;
                        if (tabu) dexp[q] = new_exp;
                    }
            }
            if (REC && P.tr_i) {  // trail row (_kernels.pyx:182-187); was_tabu = cells[bi][bj] > c (:171)
                const size_t o = (size_t)b * iters + (c - 1);
                P.tr_i[o] = r; P.tr_j[o] = s; P.tr_d[o] = (int64_t)bd;
                if (P.tr_tabu) P.tr_tabu[o] = (int64_t)was;
            }
            if (REC && tabu && P.cells) {
                int64_t *cz = P.cells + (size_t)b * n * n;
                cz[(size_t)r * n + s] = (int64_t)c + ten;
                cz[(size_t)s * n + r] += 1;
            }
        }
        // ---- tabu bits that expire at the next iteration are cleared here
        if (!NOTABU && own && c + 1 >= mexp) expire_bits(tb, mexp, c + 1, xp + lane * 16);
        __syncwarp();  // ------------------------------------------------ sync #2
    }

    if (loc) {
        P.best[(size_t)b * n + lane] = best_p;
        P.cur[(size_t)b * n + lane] = my_p;
    }
    if (lane == 0) {
        P.best_cost[b] = best_cost;
        P.cur_cost[b] = cost;
        if (P.stopped) P.stopped[b] = stopped;
        if (P.steps) P.steps[b] = steps_done;
    }
}

}  // namespace qapb
