// clique_kernels.cuh -- bitmap local-graph search (LGS) for k-clique counting
// (k = 3..5) on the degree-oriented DAG (G²Miner LGS, PAPER.md:1040-1075;
// reference _LocalRunner executor.py:415-523, setops.build_local_graph
// setops.py:124-142, mask/popcount helpers setops.py:145-173).
//
// Every k-clique of a DAG has a unique source u (the vertex all others are
// out-neighbours of). With A = N+(u) renamed to local ids 0..d-1 (ascending
// ids, as the reference's LocalGraph), row R[i] is the bitmap of
// A ∩ N+(A[i]); the k-cliques with source u are exactly the (k-1)-cliques of
// the local DAG R, counted with AND + popcount:
//   k=3: Σ_i |R_i|     k=4: Σ_i Σ_{j∈R_i} |R_i & R_j|
//   k=5: Σ_i Σ_{j∈R_i} Σ_{l∈R_i&R_j} |R_i & R_j & R_l|
// so counts equal the reference's sorted-list plan (the same cliques).
//
// The kernels run on the rank-space copy of the DAG (g2m.cu ensure_rank):
// ids are positions in the (degree, id) order, so every out-neighbour has a
// larger id and A spans a narrow window [A0, A_last] for the sources of the
// CTA tiers. Membership + local id of a probed id x is then a direct-address
// lookup in a shared-memory bitmap of that window (one LDS, one POPC, no
// probing loop, no divergence); a linear-probing hash map is the fallback
// for windows wider than the bitmap.
//
// Tiers: d <= 64 -> one warp per source, hash map, single-word rows;
// 64 < d <= 64*W -> one CTA of NW warps per source, W-word rows.
// Sources with d > 1024 are left to the generic plan kernel.
#pragma once

#include "g2m_device.cuh"

namespace g2m_clique {

typedef unsigned short u16;

// ---- probe structures: local id of x in A, or G2M_EMPTY -------------------

struct BitmapProbe {          // direct-address window [base, base + span)
    const u32* bm;            // span bits
    const u16* pre;           // local id of the first member of each word
    u32 base, span;
    __device__ __forceinline__ u32 get(u32 x) const {
        const u32 o = x - base;                    // wraps for x < base
        if (o >= span) return G2M_EMPTY;
        const u32 w = bm[o >> 5];
        const u32 b = 1u << (o & 31u);
        if (!(w & b)) return G2M_EMPTY;
        return (u32)pre[o >> 5] + (u32)__popc(w & (b - 1u));
    }
    __device__ __forceinline__ bool has(u32 x) const {
        const u32 o = x - base;
        return o < span && ((bm[o >> 5] >> (o & 31u)) & 1u);
    }
};

// Two-level window (windows wider than the direct bitmap): one top bit per
// 64-id block, a rank prefix per top word, and one 64-bit member word plus
// first local id for each occupied block -- O(span/64 + d) shared words.
struct TwoLevelProbe {
    const u32* top;           // [ntop] block-occupancy bits
    const u32* tpre;          // [ntop] occupied blocks before each top word
    const u64* blk;           // [occupied] member bits of each occupied block
    const u16* bpre;          // [occupied] local id of each block's first member
    u32 base, span;
    __device__ __forceinline__ u32 get(u32 x) const {
        const u32 o = x - base;
        if (o >= span) return G2M_EMPTY;
        const u32 t = o >> 6;
        const u32 tw = top[t >> 5];
        const u32 tb = 1u << (t & 31u);
        if (!(tw & tb)) return G2M_EMPTY;
        const u32 r = tpre[t >> 5] + (u32)__popc(tw & (tb - 1u));
        const u64 w = blk[r];
        const u64 b = 1ull << (o & 63u);
        if (!(w & b)) return G2M_EMPTY;
        return (u32)bpre[r] + (u32)__popcll(w & (b - 1ull));
    }
    __device__ __forceinline__ bool has(u32 x) const { return get(x) != G2M_EMPTY; }
};

struct HashProbe {            // linear probing, load <= 1/2
    const u32* hk;
    const u32* hv;
    u32 hl, lo, hi;
    __device__ __forceinline__ u32 get(u32 x) const {
        if (x < lo || x > hi) return G2M_EMPTY;
        return g2m_hmap_get(hk, hv, hl, x);
    }
    __device__ __forceinline__ bool has(u32 x) const { return get(x) != G2M_EMPTY; }
};

// Per-edge triangle support (diamond counting, k = 3 only): every triangle
// u -> a -> x (u the source, a = A[i], x = A[pos]) adds 1 to the support of
// its three DAG edges: (a, x) directly in t[] (other sources share it), and
// (u, a), (u, x) through per-source shared row / column counters that are
// flushed once per source.
struct Support {
    u32* t;       // t[slot] over the rank-space DAG slots
    u32* row;     // shared, by local id
    u32* col;
};

// Warp tier: probe the out-lists of rows [i0, i0+32) of A (scratch: 128
// words: end[32] row[32] base[32 u64]). K == 3 returns the number of
// members found (triangles u, A[i], x); otherwise sets the row bits of R
// (row stride Ws words) and returns 0. All 32 lanes share the concatenated
// lists (load-balanced whatever the list lengths).
template <int K, bool SUP = false, typename Probe>
__device__ __forceinline__ u32 probe_rows(const u64* __restrict__ off, const u32* __restrict__ nbr,
                                          const u32* A, u32 d, u32 i0, u64* R, u32 Ws,
                                          u32* scratch, const Probe& P, const Support& S = {}) {
    const u32 lane = g2m_lane();
    u32* fl_end = scratch;
    u32* fl_row = scratch + 32;
    u64* fl_base = (u64*)(scratch + 64);
    const u32 i = i0 + lane;
    const u32 hi = A[d - 1];
    u64 ro = 0;
    u32 rn = 0;
    if (i < d) {
        const u32 v = A[i];
        ro = __ldg(off + v);
        rn = (u32)(__ldg(off + v + 1) - ro);
        // out-neighbours of v are > v >= A0; drop the tail beyond A_last
        if (rn > 64 && __ldg(nbr + ro + rn - 1) > hi) rn = g2m_lb(nbr + ro, rn, hi + 1u);
    }
    const u32 incl = g2m_scan_incl(rn);
    const u32 tot = __shfl_sync(G2M_FULL, incl, 31);
    fl_end[lane] = incl;
    fl_row[lane] = i;
    fl_base[lane] = ro - (u64)(incl - rn);     // nbr index of flattened position e = base + e
    __syncwarp();
    u32 hits = 0;
    u32 ow = 0;   // this lane's owner row, monotone
    auto one = [&](u32 o, u64 xi, u32 x) {
        if constexpr (SUP) {
            const u32 pos = P.get(x);
            if (pos != G2M_EMPTY) {
                atomicAdd(S.t + xi, 1u);
                atomicAdd(S.row + fl_row[o], 1u);
                atomicAdd(S.col + pos, 1u);
            }
        } else if constexpr (K == 3) {
            hits += P.has(x) ? 1u : 0u;
        } else {
            const u32 pos = P.get(x);
            if (pos != G2M_EMPTY)   // 32-bit halves: native ATOMS.OR (64-bit would be a CAS loop)
                atomicOr((u32*)(R + (u64)fl_row[o] * Ws) + (pos >> 5), 1u << (pos & 31u));
        }
    };
    // two elements per lane per step: both loads are in flight before either probe
    for (u32 e0 = 0; e0 < tot; e0 += 64) {
        const u32 ea = e0 + lane, eb = ea + 32;
        u32 oa = ow, ob;
        u64 ia = 0, ib = 0;
        u32 xa = 0, xb = 0;
        if (ea < tot) {
            while (fl_end[oa] <= ea) ++oa;
            ia = fl_base[oa] + ea;
            xa = __ldg(nbr + ia);
        }
        ob = oa;
        if (eb < tot) {
            while (fl_end[ob] <= eb) ++ob;
            ib = fl_base[ob] + eb;
            xb = __ldg(nbr + ib);
        }
        if (ea < tot) one(oa, ia, xa);
        if (eb < tot) one(ob, ib, xb);
        ow = ob;
    }
    __syncwarp();
    return hits;
}

// Number of DEPTH-vertex chains inside candidate set m of a single-word DAG.
template <int DEPTH>
struct Chain1 {
    __device__ static __forceinline__ u64 run(const u64* R, u64 m) {
        u64 c = 0;
        u64 it = m;
        while (it) {
            const int j = __ffsll(it) - 1;
            it &= it - 1;
            c += Chain1<DEPTH - 1>::run(R, m & R[j]);
        }
        return c;
    }
};
template <>
struct Chain1<1> {
    __device__ static __forceinline__ u64 run(const u64*, u64 m) { return (u64)__popcll(m); }
};

// ---------------------------------------------------------------------------
// warp tier: d <= 64, one warp per source vertex
// ---------------------------------------------------------------------------
template <int K, int WPB, bool SUP = false>
__global__ void __launch_bounds__(WPB * 32)
k_clique_warp(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
              u64 nverts, u64* next, u64 grab, u64* count, u32* tsup) {
    __shared__ u32 sA[WPB][64];
    __shared__ u32 sRow[SUP ? WPB : 1][64];
    __shared__ u32 sCol[SUP ? WPB : 1][64];
    __shared__ __align__(8) u64 sR[WPB][64];
    __shared__ __align__(8) u32 sScr[WPB][128];
    __shared__ u32 sHK[WPB][128];
    __shared__ u32 sHV[WPB][128];
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    u32* A = sA[w];
    u64* R = sR[w];
    u64 acc = 0;
    for (;;) {
        u64 t0 = 0;
        if (lane == 0) t0 = atomicAdd(next, grab);
        t0 = __shfl_sync(G2M_FULL, t0, 0);
        if (t0 >= nverts) break;
        const u64 t1 = min(t0 + grab, nverts);
        for (u64 t = t0; t < t1; ++t) {
            const u32 u = __ldg(verts + t);
            const u64 b = __ldg(off + u);
            const u32 d = (u32)(__ldg(off + u + 1) - b);
            A[lane] = lane < d ? __ldg(nbr + b + lane) : 0xffffffffu;
            A[lane + 32] = lane + 32 < d ? __ldg(nbr + b + lane + 32) : 0xffffffffu;
            if constexpr (K > 3) {
                R[lane] = 0;
                R[lane + 32] = 0;
            }
            __syncwarp();
            const u32 hl = g2m_hlog(d);
            g2m_hmap_build(sHK[w], sHV[w], hl, A, d, lane, 32);
            const HashProbe P{sHK[w], sHV[w], hl, A[0], A[d - 1]};
            Support S{};
            if constexpr (SUP) {
                S = Support{tsup, sRow[w], sCol[w]};
                sRow[w][lane] = sRow[w][lane + 32] = 0;
                sCol[w][lane] = sCol[w][lane + 32] = 0;
                __syncwarp();
            }
            u32 h = probe_rows<K, SUP>(off, nbr, A, d, 0, R, 1, sScr[w], P, S);
            if (d > 32) h += probe_rows<K, SUP>(off, nbr, A, d, 32, R, 1, sScr[w], P, S);
            if constexpr (SUP) {
                for (u32 i = lane; i < d; i += 32) {
                    const u32 c = sRow[w][i] + sCol[w][i];
                    if (c) atomicAdd(tsup + b + i, c);
                }
            } else if constexpr (K == 3) {
                acc += h;
            } else {
                for (u32 i = lane; i < d; i += 32) acc += Chain1<K - 2>::run(R, R[i]);
            }
            __syncwarp();
        }
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// ---------------------------------------------------------------------------
// Hub core: the DAG restricted to the top T ranks (rank space: every out-
// neighbour of a core vertex is in the core) as a packed upper-triangular bit
// matrix, row alpha = a - lo holding bits beta - alpha - 1 for the core ranks
// beta > alpha, each row padded to u32 words. T = 2^15 is 64 MB: L2-resident.
// An edge test a -> b with a in the core is one bit read instead of a
// binary search of N+(a) (a chain of dependent L2 reads).
// ---------------------------------------------------------------------------
struct HubCore {
    const u32* bits;    // nullptr: no core
    u32 lo, T;
    // words of rows 0..alpha-1: S(T-1) - S(T-1-alpha), S(N) = sum_{m<=N} ceil(m/32)
    __device__ __forceinline__ static u64 S(u64 N) {
        const u64 q = N >> 5, r = N & 31u;
        return 16ull * q * (q + 1) + r * (q + 1);
    }
    __device__ __forceinline__ bool has(u32 a, u32 b) const {
        const u32 al = a - lo, be = b - lo;
        const u32 bit = be - al - 1u;
        const u64 w = S((u64)T - 1) - S((u64)T - 1 - al) + (bit >> 5);
        return (__ldg(bits + w) >> (bit & 31u)) & 1u;
    }
};

// ---------------------------------------------------------------------------
// pair tier: d <= 64, one warp per source; the local edges a -> b (a, b in A)
// are found by testing every pair of A directly, b in N+(a) by binary search
// -- d(d-1)/2 lane-parallel tests instead of streaming the out-lists of A,
// which for small sources are mostly far longer than A itself.
// ---------------------------------------------------------------------------
template <int K, int WPB, int MAXD = 64, int PU = 1>
__global__ void __launch_bounds__(WPB * 32)
k_clique_pairs(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
               u64 nverts, u64* next, u64 grab, u64* count, HubCore core = HubCore{nullptr, 0, 0}) {
    static_assert(K == 3 || MAXD <= 64 || (K == 4 && MAXD <= 128), "row width");
    constexpr int RW = MAXD > 64 ? 2 : 1;      // u64 words per local row
    __shared__ u32 sA[WPB][MAXD];
    __shared__ __align__(8) u64 sR[WPB][K > 3 ? MAXD * RW : 1];
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    u32* A = sA[w];
    u64* R = sR[w];
    u64 acc = 0;
    for (;;) {
        u64 t0 = 0;
        if (lane == 0) t0 = atomicAdd(next, grab);
        t0 = __shfl_sync(G2M_FULL, t0, 0);
        if (t0 >= nverts) break;
        const u64 t1 = min(t0 + grab, nverts);
        for (u64 t = t0; t < t1; ++t) {
            const u32 u = __ldg(verts + t);
            const u64 b = __ldg(off + u);
            const u32 d = (u32)(__ldg(off + u + 1) - b);
#pragma unroll
            for (u32 x = lane; x < (u32)MAXD; x += 32) A[x] = x < d ? __ldg(nbr + b + x) : 0u;
            if constexpr (K > 3)
                for (u32 x = lane; x < (u32)(MAXD * RW); x += 32) R[x] = 0;
            __syncwarp();
            const u32 np = d * (d - 1) / 2;
            const float D = 2.f * (float)d - 1.f;
            // PU pairs per lane per step: their core-word loads are all in flight
            // before any is used (the core reads are the latency of this tier)
            for (u32 p0 = lane; p0 < np; p0 += 32 * PU) {
                u32 ii[PU], jj[PU], cw[PU];
                bool vv[PU], cc[PU];
#pragma unroll
                for (int q = 0; q < PU; ++q) {
                    const u32 p = p0 + 32u * q;
                    vv[q] = p < np;
                    cc[q] = false;
                    ii[q] = jj[q] = cw[q] = 0u;
                    if (vv[q]) {
                        // row i of pair p in the row-major upper triangle: closed form + fix-up
                        u32 i = (u32)((D - sqrtf(D * D - 8.f * (float)p)) * 0.5f);
                        while (i > 0 && i * (2 * d - i - 1) / 2 > p) --i;
                        while ((i + 1) * (2 * d - i - 2) / 2 <= p) ++i;
                        ii[q] = i;
                        jj[q] = i + 1 + (p - i * (2 * d - i - 1) / 2);
                        const u32 a = A[i];
                        if (core.bits && a >= core.lo) {
                            cc[q] = true;
                            const u32 al = a - core.lo, bit = A[jj[q]] - a - 1u;
                            cw[q] = __ldg(core.bits + HubCore::S((u64)core.T - 1) -
                                          HubCore::S((u64)core.T - 1 - al) + (bit >> 5)) >> (bit & 31u);
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < PU; ++q) {
                    if (!vv[q]) continue;
                    bool e;
                    if (cc[q]) {
                        e = cw[q] & 1u;
                    } else {
                        const u32 a = A[ii[q]];
                        const u64 ao = __ldg(off + a);
                        e = g2m_has_g(nbr + ao, (u32)(__ldg(off + a + 1) - ao), A[jj[q]]);
                    }
                    if (e) {
                        if constexpr (K == 3) acc += 1;
                        else atomicOr((u32*)(R + ii[q] * RW) + (jj[q] >> 5), 1u << (jj[q] & 31u));
                    }
                }
            }
            if constexpr (K > 3 && RW == 1) {
                __syncwarp();
                if (lane < d) acc += Chain1<K - 2>::run(R, R[lane]);
                if (lane + 32 < d) acc += Chain1<K - 2>::run(R, R[lane + 32]);
            } else if constexpr (K == 4) {   // two-word rows: Σ_i Σ_{j in R_i} |R_i & R_j|
                __syncwarp();
                for (u32 i = lane; i < d; i += 32) {
                    const u64 r0 = R[2 * i], r1 = R[2 * i + 1];
                    u64 it = r0;
                    while (it) {
                        const int j = __ffsll(it) - 1;
                        it &= it - 1;
                        acc += (u64)__popcll(r0 & R[2 * j]) + (u64)__popcll(r1 & R[2 * j + 1]);
                    }
                    it = r1;
                    while (it) {
                        const int j = 64 + __ffsll(it) - 1;
                        it &= it - 1;
                        acc += (u64)__popcll(r1 & R[2 * j + 1]);
                    }
                }
            }
            __syncwarp();
        }
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// ---------------------------------------------------------------------------
// staged pair tier (G2M_PAIR_BULK): the pair tier's local-edge tests with
// the searched lists brought into shared memory by the TMA engine. Row i of
// A (a = A[i], nk = d-1-i keys A[i+1..d), list L = N+(a) of length l) is
// *staged* when nk * (ceil log2 l - 4) * 8 >= l, i.e. when its nk global
// binary searches would fetch more 32-byte sectors (less the ~4 top levels
// the lanes share in L1) than copying the l * 4 list bytes once: one lane
// issues a 1-D cp.async.bulk of the list (completion on an mbarrier),
// double-buffered so the next staged row's copy is in flight while this
// row's keys are searched in shared memory (~30-cycle LDS steps instead of
// dependent L2/DRAM round trips). The first copy overlaps the global
// searches of the unstaged rows (few keys, or lists longer than CAPB - 4).
// ---------------------------------------------------------------------------
template <int K, int MAXD, int CAPB>
struct PairBulkSmem {
    static constexpr int RW = MAXD > 64 ? 2 : 1;
    u32 buf[2][CAPB];                   // staged lists, 16-byte aligned
    u64 R[K > 3 ? MAXD * RW : 2];
    u64 ro[MAXD];                       // list start of row i
    u64 bar[2];
    u32 A[MAXD];
    u32 rl[MAXD];                       // list length of row i
    u32 pre[MAXD + 4];                  // exclusive prefix of nk over the global rows
    u32 grow[MAXD];                     // global-search rows
    u32 srow[MAXD];                     // staged rows
};

template <int K, int WPB, int MAXD, int CAPB>
__global__ void __launch_bounds__(WPB * 32)
k_clique_pairs_bulk(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
                    u64 nverts, u64* next, u64 grab, u64* count) {
    static_assert(K == 3 || MAXD <= 64 || (K == 4 && MAXD <= 128), "row width");
    static_assert(CAPB % 4 == 0, "16-byte staging buffers");
    using SM = PairBulkSmem<K, MAXD, CAPB>;
    constexpr int RW = SM::RW;
    static_assert(sizeof(SM) % 16 == 0, "per-warp region keeps 16-byte alignment");
    extern __shared__ __align__(16) unsigned char pb_smem[];
    SM& S = reinterpret_cast<SM*>(pb_smem)[threadIdx.x >> 5];
    const u32 lane = g2m_lane();
    const u32 lt = g2m_lanemask_lt();
    u32* A = S.A;
    u64* R = S.R;
    if (lane == 0) {
        g2m_mbar_init(&S.bar[0], 1);
        g2m_mbar_init(&S.bar[1], 1);
        g2m_fence_barrier_init();
    }
    __syncwarp();
    u32 ph0 = 0, ph1 = 0;     // completed phases per buffer
    u64 acc = 0;
    for (;;) {
        u64 t0 = 0;
        if (lane == 0) t0 = atomicAdd(next, grab);
        t0 = __shfl_sync(G2M_FULL, t0, 0);
        if (t0 >= nverts) break;
        const u64 t1 = min(t0 + grab, nverts);
        for (u64 t = t0; t < t1; ++t) {
            const u32 u = __ldg(verts + t);
            const u64 b = __ldg(off + u);
            const u32 d = (u32)(__ldg(off + u + 1) - b);
            for (u32 x = lane; x < d; x += 32) A[x] = __ldg(nbr + b + x);
            if constexpr (K > 3)
                for (u32 x = lane; x < d * RW; x += 32) R[x] = 0;
            __syncwarp();
            // classify rows: staged / global-search
            u32 nst = 0, ng = 0, carry = 0;
            for (u32 i0 = 0; i0 + 1 < d; i0 += 32) {
                const u32 i = i0 + lane;
                const bool valid = i + 1 < d;
                u64 ro = 0;
                u32 l = 0, nk = 0;
                if (valid) {
                    const u32 a = A[i];
                    ro = __ldg(off + a);
                    l = (u32)(__ldg(off + a + 1) - ro);
                    nk = d - 1 - i;
                    S.ro[i] = ro;
                    S.rl[i] = l;
                }
                const u32 lg = l > 1 ? 32u - (u32)__clz(l - 1) : 1u;
                const bool st = valid && l > 0 && l + 4 <= (u32)CAPB && nk * (lg > 4 ? lg - 4 : 1u) * 8u >= l;
                const bool gl = valid && l > 0 && !st;
                const u32 ms = __ballot_sync(G2M_FULL, st), mg = __ballot_sync(G2M_FULL, gl);
                if (st) S.srow[nst + __popc(ms & lt)] = i;
                const u32 gk = gl ? nk : 0u;
                const u32 incl = g2m_scan_incl(gk);
                if (gl) {
                    const u32 q = ng + __popc(mg & lt);
                    S.grow[q] = i;
                    S.pre[q] = carry + incl - gk;
                }
                nst += __popc(ms);
                ng += __popc(mg);
                carry += __shfl_sync(G2M_FULL, incl, 31);
            }
            if (lane == 0) S.pre[ng] = carry;
            __syncwarp();
            // first staged copy in flight during the global searches
            if (nst && lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const u32 i = S.srow[0];
                g2m_bulk_list(S.buf[0], nbr + S.ro[i], S.rl[i], &S.bar[0]);
            }
            // global-search rows: pairs flattened over the lanes
            for (u32 p = lane; p < carry; p += 32) {
                u32 lo = 0, n = ng;        // last q with pre[q] <= p
                while (n > 1) {
                    const u32 h = n >> 1;
                    lo = S.pre[lo + h] <= p ? lo + h : lo;
                    n -= h;
                }
                const u32 i = S.grow[lo];
                const u32 j = i + 1 + (p - S.pre[lo]);
                if (g2m_has_g(nbr + S.ro[i], S.rl[i], A[j])) {
                    if constexpr (K == 3) acc += 1;
                    else atomicOr((u32*)(R + i * RW) + (j >> 5), 1u << (j & 31u));
                }
            }
            // staged rows, double-buffered
            for (u32 s2 = 0; s2 < nst; ++s2) {
                const u32 bs = s2 & 1u;
                if (s2 + 1 < nst && lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const u32 i = S.srow[s2 + 1];
                    g2m_bulk_list(S.buf[bs ^ 1u], nbr + S.ro[i], S.rl[i], &S.bar[bs ^ 1u]);
                }
                g2m_mbar_wait(&S.bar[bs], (bs ? ph1 : ph0) & 1u);
                if (bs) ++ph1; else ++ph0;
                const u32 i = S.srow[s2];
                const u32 l = S.rl[i];
                const u32* L = S.buf[bs] + (u32)(S.ro[i] & 3ull);
                for (u32 j = i + 1 + lane; j < d; j += 32) {
                    if (g2m_has(L, l, A[j])) {
                        if constexpr (K == 3) acc += 1;
                        else atomicOr((u32*)(R + i * RW) + (j >> 5), 1u << (j & 31u));
                    }
                }
                __syncwarp();
            }
            if constexpr (K > 3 && RW == 1) {
                __syncwarp();
                if (lane < d) acc += Chain1<K - 2>::run(R, R[lane]);
                if (lane + 32 < d) acc += Chain1<K - 2>::run(R, R[lane + 32]);
            } else if constexpr (K == 4) {
                __syncwarp();
                for (u32 i = lane; i < d; i += 32) {
                    const u64 r0 = R[2 * i], r1 = R[2 * i + 1];
                    u64 it = r0;
                    while (it) {
                        const int j = __ffsll(it) - 1;
                        it &= it - 1;
                        acc += (u64)__popcll(r0 & R[2 * j]) + (u64)__popcll(r1 & R[2 * j + 1]);
                    }
                    it = r1;
                    while (it) {
                        const int j = 64 + __ffsll(it) - 1;
                        it &= it - 1;
                        acc += (u64)__popcll(r1 & R[2 * j + 1]);
                    }
                }
            }
            __syncwarp();
        }
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// Warp-cooperative compaction of the set bits of words[q0, q1) (shared,
// read by broadcast) into out[] as bit positions; returns the count.
__device__ __forceinline__ u32 compact_bits(const u64* words, u32 q0, u32 q1, u32* out) {
    const u32 lane = g2m_lane();
    const u32 lt = g2m_lanemask_lt();
    u32 n = 0;
    for (u32 q = q0; q < q1; ++q) {
        const u64 wv = words[q];
        if (!wv) continue;
        const u32 lo = (u32)wv, hi = (u32)(wv >> 32);
        if ((lo >> lane) & 1u) out[n + __popc(lo & lt)] = q * 64 + lane;
        if ((hi >> lane) & 1u) out[n + __popc(lo) + __popc(hi & lt)] = q * 64 + 32 + lane;
        n += __popcll(wv);
    }
    __syncwarp();
    return n;
}

// Per-warp scratch of the CTA tier (u32 words): L1[256] (k >= 4), L2[256] (k = 5).
__host__ __device__ constexpr u32 cta_warp_words(int K) { return K > 4 ? 512u : (K == 4 ? 256u : 0u); }

// The fallback hash map (keys + vals, 256W words) is only live while rows are
// probed, the per-warp candidate lists only while they are counted: they
// share one region.
__host__ __device__ constexpr size_t cta_union_words(int K, int W, int NW) {
    return (size_t)256 * W > (size_t)NW * cta_warp_words(K) ? (size_t)256 * W : (size_t)NW * cta_warp_words(K);
}

// u64 words of the local-graph rows R and the per-warp row buffers T.
__host__ __device__ constexpr size_t cta_row_words(int K, int W, int NW) {
    return K > 3 ? (size_t)(64 * W + NW) * (W + 1) : 0;
}

// Shared-memory bytes of one CTA-tier block (layout in k_clique_cta); with
// GR the rows live in a global (L2-resident) slab per block instead.
__host__ __device__ constexpr size_t cta_smem_bytes(int K, int W, int NW, u32 bmw, bool GR = false,
                                                    bool SUP = false) {
    return (GR ? 0 : (size_t)8 * cta_row_words(K, W, NW))        // R, T
           + (SUP ? (size_t)4 * 2 * 64 * W : 0)                  // support row / column counters
           + (size_t)8 * 64 * W                                  // RB
           + (size_t)4 * 64 * W * 3 + (size_t)4 * 2 * W          // A, RE, LR, BT
           + (size_t)4 * cta_union_words(K, W, NW)               // hash (probe) | per-warp scratch (count)
           + (size_t)4 * bmw + (size_t)2 * ((bmw + 1) & ~1u);    // bitmap, pre
}

// Rows with at least kLongRow candidates are probed row by row (a warp per
// row, lanes striding, no owner search); the rest are concatenated.
constexpr u32 kLongRow = 128;

// One probed element x (nbr index xi) of row `row` of source A.
template <int K, bool SUP, typename Probe>
__device__ __forceinline__ void probe_one(u32 row, u64 xi, u32 x, u64* R, u32 Ws, const Probe& P,
                                          const Support& S, u32& hits) {
    if constexpr (SUP) {
        const u32 pos = P.get(x);
        if (pos != G2M_EMPTY) {
            atomicAdd(S.t + xi, 1u);
            atomicAdd(S.row + row, 1u);
            atomicAdd(S.col + pos, 1u);
        }
    } else if constexpr (K == 3) {
        hits += P.has(x) ? 1u : 0u;
    } else {
        const u32 pos = P.get(x);
        if (pos != G2M_EMPTY)   // 32-bit halves: native ATOMS.OR (64-bit would be a CAS loop)
            atomicOr((u32*)(R + (u64)row * Ws) + (pos >> 5), 1u << (pos & 31u));
    }
}

// CTA-wide probe of all out-lists N+(A[i]), i < d. Long rows (list LR,
// nlong entries) go first, one warp per row in dynamic grabs; then the warps
// take 64-element steps of the concatenation of the short rows in dynamic
// grabs (RE[i]: inclusive end of row i in the concatenation, 0-length for
// long rows; RB[i]: nbr index of its position 0). K == 3 counts members;
// otherwise sets the row bits of R.
template <int K, int NW, bool SUP, typename Probe>
__device__ __forceinline__ u32 cta_probe(const u64* __restrict__ off, const u32* __restrict__ nbr,
                                         const u32* A, const u32* RE, const u64* RB, const u32* LR, u32 nlong,
                                         u32 alast, u32 d, u32 tot, u32* s_lrow, u32* s_flat, u64* R, u32 Ws,
                                         const Probe& P, const Support& S) {
    const u32 lane = g2m_lane();
    u32 hits = 0;
    for (;;) {
        u32 k = 0;
        if (lane == 0) k = atomicAdd(s_lrow, 1u);
        k = __shfl_sync(G2M_FULL, k, 0);
        if (k >= nlong) break;
        const u32 i = LR[k];
        const u32 v = A[i];
        const u64 ro = __ldg(off + v);
        u32 rn = (u32)(__ldg(off + v + 1) - ro);
        if (__ldg(nbr + ro + rn - 1) > alast) rn = g2m_lb(nbr + ro, rn, alast + 1u);
        for (u32 e0 = 0; e0 < rn; e0 += 64) {
            const u32 ea = e0 + lane, eb = ea + 32;
            const u32 xa = ea < rn ? __ldg(nbr + ro + ea) : 0u;
            const u32 xb = eb < rn ? __ldg(nbr + ro + eb) : 0u;
            if (ea < rn) probe_one<K, SUP>(i, ro + ea, xa, R, Ws, P, S, hits);
            if (eb < rn) probe_one<K, SUP>(i, ro + eb, xb, R, Ws, P, S, hits);
        }
    }
    u32 o0 = 0;      // first row whose end is beyond the warp's first element (warp-uniform)
    for (;;) {
        u32 e0 = 0;
        if (lane == 0) e0 = atomicAdd(s_flat, 64u);
        e0 = __shfl_sync(G2M_FULL, e0, 0);     // increasing per warp, so o0 only moves forward
        if (e0 >= tot) break;
        for (;;) {   // RE is non-decreasing, so "RE[r] <= e0" holds on a prefix
            const u32 r = o0 + lane;
            const u32 n = __popc(__ballot_sync(G2M_FULL, r < d && RE[r] <= e0));
            o0 += n;
            if (n < 32) break;
        }
        const u32 ea = e0 + lane, eb = ea + 32;
        u32 oa = o0, ob = o0;
        u32 xa = 0, xb = 0;
        u64 ia = 0, ib = 0;
        if (ea < tot) {
            while (RE[oa] <= ea) ++oa;
            ia = RB[oa] + ea;
            xa = __ldg(nbr + ia);
        }
        if (eb < tot) {
            ob = oa;
            while (RE[ob] <= eb) ++ob;
            ib = RB[ob] + eb;
            xb = __ldg(nbr + ib);
        }
        if (ea < tot) probe_one<K, SUP>(oa, ia, xa, R, Ws, P, S, hits);
        if (eb < tot) probe_one<K, SUP>(ob, ib, xb, R, Ws, P, S, hits);
    }
    return hits;
}

// ---------------------------------------------------------------------------
// CTA tier: 64 < d <= 64*W, one CTA of NW warps per source vertex, W-word
// rows with an odd stride. Local-graph construction is one CTA-wide pass
// over all out-lists (cta_probe: long rows whole, short rows concatenated);
// rows are counted in
// dynamic single-row grabs, so the CTA barrier does not wait on the
// unluckiest warp. The candidates j of R_i are compacted (CH words at a
// time) into a shared list so every lane gets a candidate; R_j has no bits
// below j (rank-space DAG), so only words >= j/64 are ANDed. k=5:
// t2 = R_i & R_j stays in the lane's registers when small; large ones are
// compacted again and shared by the whole warp.
// bmw: u32 words of the window bitmap (0 = hash only).
// ---------------------------------------------------------------------------
// k = 5: local sources i with 128 < |R_i| <= 256 deferred to a CTA-wide phase
// that compresses R_i's sub-DAG to 4-word rows (set by the host per launch,
// G2M_CL5_BIG=1). Off by default: measured slower on RMAT-22 (W=16 tier
// 597 -> 670 ms; the per-big-row CTA barriers serialise what the per-warp
// path overlaps).
__device__ u32 g_cl5_big = 0;

// Blocks per SM the narrow tiers are launched at (g2m.cu): keeps the register
// budget at what that occupancy allows (the window/hash variants add live values).
__host__ __device__ constexpr int cta_min_blocks(int K, int W) {
    return K == 3 ? (W <= 16 ? 4 : 1) : (K == 4 ? (W <= 8 ? 3 : 1) : (W == 4 ? 2 : (W <= 8 ? 3 : 1)));
}

template <int K, int W, int NW, bool GR = false, bool SUP = false>
__global__ void __launch_bounds__(NW * 32, cta_min_blocks(K, W))
k_clique_cta(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
             u64 nverts, u64* next, u64* count, u32 bmw, u64* grows, u32* tsup, u32 split, u32 direct_max,
             HubCore core = HubCore{nullptr, 0, 0}) {
    constexpr u32 CH = 4;             // words compacted per round (<= 256 candidates)
    extern __shared__ __align__(16) u64 smem[];
    // layout: R [64W x (W+1)] u64 | T [NW x (W+1)] u64   (K > 3 only)
    //         RB [64W] u64 | A [64W] u32 | RE [64W] u32 | BT [2W] u32
    //         hash keys, vals [128W] u32 each | per-warp scratch | bitmap [bmw] u32 | pre [bmw] u16
    u64* R = GR ? grows + (u64)blockIdx.x * cta_row_words(K, W, NW) : smem;
    u64* T = R + (K > 3 ? 64 * W * (W + 1) : 0);
    u64* RB = GR ? smem : T + (K > 3 ? NW * (W + 1) : 0);
    u32* A = (u32*)(RB + 64 * W);
    u32* RE = A + 64 * W;
    u32* LR = RE + 64 * W;
    u32* BT = LR + 64 * W;
    u32* HK = BT + 2 * W;             // probe phase
    u32* HV = HK + 128 * W;
    u32* scr = HK;                    // count phase (same region, after the barrier)
    u32* BM = HK + cta_union_words(K, W, NW);
    u16* PRE = (u16*)(BM + bmw);
    u32* SROW = (u32*)(PRE + ((bmw + 1) & ~1u));     // SUP only: [64W] row, [64W] column counters
    u32* SCOL = SROW + 64 * W;
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    u32* L1 = scr + w * cta_warp_words(K);
    u32* L2 = L1 + 256;
    u64* t2s = T + w * (W + 1);
    __shared__ u64 s_u;
    __shared__ u32 s_cnt, s_tot, s_nlong, s_lrow, s_flat, s_nbig, s_n1;
    for (u32 x = threadIdx.x; x < bmw; x += NW * 32) BM[x] = 0;
    u64 acc = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            s_u = atomicAdd(next, 1ull);
            s_cnt = 0;
            s_nbig = 0;
            s_nlong = 0;
            s_lrow = 0;
            s_flat = 0;
        }
        __syncthreads();
        // work item s_u = (source, part): with split > 1 every part builds the
        // source's local graph and counts the rows i = part (mod split)
        const u64 t = s_u / split;
        const u32 part = (u32)(s_u % split);
        if (t >= nverts) break;
        const u32 u = __ldg(verts + t);
        const u64 b = __ldg(off + u);
        const u32 d = (u32)(__ldg(off + u + 1) - b);
        const u32 Wd = (d + 63) >> 6;
        const u32 Ws = Wd | 1u;          // odd row stride (bank spread)
        const u32 a0 = __ldg(nbr + b), alast = __ldg(nbr + b + d - 1);
        const u32 span = alast - a0 + 1u;
        const bool use_bm = span <= bmw * 32u && span <= direct_max;
        // two-level window inside the (idle) bitmap region: top [ntop] | tpre [ntop] |
        // blk [d] u64 | bpre [d] u16
        const u32 ntop = ((((span + 63u) >> 6) + 31u) >> 5) + 1u & ~1u;
        const bool use_tl = !use_bm && 2u * ntop + 2u * d + (d + 1u) / 2u + 2u <= bmw;
        u32* TT = BM;
        u32* TP = BM + ntop;
        u64* TB = (u64*)(BM + 2 * ntop);
        u16* TBP = (u16*)(TB + d);
        // A, window bits, and per-32-row batches of the flattened out-lists
        for (u32 bt = w; bt * 32 < d; bt += NW) {
            const u32 i = bt * 32 + lane;
            u64 ro = 0;
            u32 rn = 0;
            if (i < d) {
                const u32 y = __ldg(nbr + b + i);
                A[i] = y;
                if (use_bm) {
                    const u32 o = y - a0;
                    atomicOr(BM + (o >> 5), 1u << (o & 31u));
                    // first member of its word: local id base of that word
                    if (i == 0 || ((__ldg(nbr + b + i - 1) - a0) >> 5) != (o >> 5)) PRE[o >> 5] = (u16)i;
                } else if (use_tl) {
                    const u32 t = (y - a0) >> 6;
                    atomicOr(TT + (t >> 5), 1u << (t & 31u));
                }
                // hub-core rows (a suffix of A) are filled from the core bits below,
                // not probed (no support counters through the core)
                if (SUP || !core.bits || y < core.lo) {
                    ro = __ldg(off + y);
                    rn = (u32)(__ldg(off + y + 1) - ro);
                    // out-neighbours of y are > y >= A0; drop the tail beyond A_last
                    if (rn > 64 && __ldg(nbr + ro + rn - 1) > alast) rn = g2m_lb(nbr + ro, rn, alast + 1u);
                }
            }
            const bool lng = rn >= kLongRow;     // probed row by row, not concatenated
            const u32 lm = __ballot_sync(G2M_FULL, lng);
            if (lm) {
                u32 lb0 = 0;
                if (lane == 0) lb0 = atomicAdd(&s_nlong, (u32)__popc(lm));
                lb0 = __shfl_sync(G2M_FULL, lb0, 0);
                if (lng) LR[lb0 + __popc(lm & g2m_lanemask_lt())] = i;
                if (lng) rn = 0;
            }
            const u32 incl = g2m_scan_incl(rn);
            if (i < d) {
                RE[i] = incl;
                RB[i] = ro - (u64)(incl - rn);
            }
            if (lane == 31) BT[bt] = incl;
        }
        if constexpr (K > 3)
            for (u32 x = threadIdx.x; x < d * Ws; x += NW * 32) R[x] = 0;
        if constexpr (SUP)
            for (u32 x = threadIdx.x; x < d; x += NW * 32) SROW[x] = SCOL[x] = 0;
        __syncthreads();
        u32 hl = 0;
        if (use_tl) {
            // rank prefix of the top words (warp 0 scans, 32 words per step), then
            // each member sets its bit in its block's word
            if (w == 0) {
                u32 carry = 0;
                for (u32 q0 = 0; q0 < ntop; q0 += 32) {
                    const u32 q = q0 + lane;
                    const u32 c = q < ntop ? (u32)__popc(TT[q]) : 0u;
                    const u32 incl = g2m_scan_incl(c);
                    if (q < ntop) TP[q] = carry + incl - c;
                    carry += __shfl_sync(G2M_FULL, incl, 31);
                }
            }
            __syncthreads();
            for (u32 x = threadIdx.x; x < d; x += NW * 32) {
                const u32 o = A[x] - a0, t = o >> 6;
                const u32 r = TP[t >> 5] + (u32)__popc(TT[t >> 5] & ((1u << (t & 31u)) - 1u));
                atomicOr((u32*)(TB + r) + ((o >> 5) & 1u), 1u << (o & 31u));
                if (x == 0 || ((A[x - 1] - a0) >> 6) != t) TBP[r] = (u16)x;
            }
        } else if (!use_bm) {
            hl = g2m_hlog(d);
            g2m_hmap_build(HK, HV, hl, A, d, threadIdx.x, NW * 32);
        }
        if (w == 0) {   // batch offsets (<= 2W batches, 4 per lane)
            const u32 nb = (d + 31) >> 5;
            u32 v[4], sum = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const u32 idx = lane * 4 + q;
                v[q] = idx < nb ? BT[idx] : 0u;
                sum += v[q];
            }
            const u32 incl = g2m_scan_incl(sum);
            u32 ex = incl - sum;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const u32 idx = lane * 4 + q;
                if (idx < nb) BT[idx] = ex;
                ex += v[q];
            }
            if (lane == 31) s_tot = incl;
        }
        __syncthreads();
        for (u32 x = threadIdx.x; x < d; x += NW * 32) {
            const u32 bo = BT[x >> 5];
            RE[x] += bo;
            RB[x] -= bo;
        }
        __syncthreads();
        // ---- build rows (K > 3) / count triangles (K == 3)
        const u32 tot = s_tot;
        u32 hits;
        const Support S{tsup, SROW, SCOL};
        const u32 nlong = s_nlong;
        if (use_bm)
            hits = cta_probe<K, NW, SUP>(off, nbr, A, RE, RB, LR, nlong, alast, d, tot, &s_lrow, &s_flat, R, Ws,
                                         BitmapProbe{BM, PRE, a0, span}, S);
        else if (use_tl)
            hits = cta_probe<K, NW, SUP>(off, nbr, A, RE, RB, LR, nlong, alast, d, tot, &s_lrow, &s_flat, R, Ws,
                                         TwoLevelProbe{TT, TP, TB, TBP, a0, span}, S);
        else
            hits = cta_probe<K, NW, SUP>(off, nbr, A, RE, RB, LR, nlong, alast, d, tot, &s_lrow, &s_flat, R, Ws,
                                         HashProbe{HK, HV, hl, a0, alast}, S);
        if constexpr (!SUP) {
            // hub-core rows i (A[i] >= core.lo; every A[j], j > i, is then in the
            // core too): R_i by one bit test per j > i, 32 j's per ballot, no probing
            if (core.bits && alast >= core.lo) {
                const u32 ic = g2m_lb(A, d, core.lo);
                for (u32 i = ic + w; i < d; i += NW) {
                    const u32 a = A[i];
                    const u64 rowb = HubCore::S((u64)core.T - 1) - HubCore::S((u64)core.T - 1 - (a - core.lo));
                    // four 32-member chunks per step: four independent core-word loads in
                    // flight per lane before the ballots (the loads are the latency)
                    for (u32 j0 = (i + 1) & ~31u; j0 < d; j0 += 128) {
                        u32 wv[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const u32 j = j0 + 32u * q + lane;
                            wv[q] = 0u;
                            if (j > i && j < d) {
                                const u32 bit = A[j] - a - 1u;
                                wv[q] = __ldg(core.bits + rowb + (bit >> 5)) >> (bit & 31u);
                            }
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const u32 m = __ballot_sync(G2M_FULL, wv[q] & 1u);
                            if constexpr (K == 3) {
                                hits += lane == 0 ? (u32)__popc(m) : 0u;
                            } else {
                                if (lane == 0 && m) ((u32*)(R + (u64)i * Ws))[(j0 >> 5) + q] = m;
                            }
                        }
                    }
                }
            }
        }
        if constexpr (K == 3) acc += hits;
        __syncthreads();
        if constexpr (SUP)
            for (u32 x = threadIdx.x; x < d; x += NW * 32) {
                const u32 c = SROW[x] + SCOL[x];
                if (c) atomicAdd(tsup + b + x, c);
            }
        if constexpr (K > 3) {
            for (;;) {
                constexpr u32 G = K == 4 ? 4u : 1u;   // rows per grab (k = 5 rows are heavy)
                u32 ig = 0;
                if (lane == 0) ig = atomicAdd(&s_cnt, G);
                ig = __shfl_sync(G2M_FULL, ig, 0);
                const u32 nmine = (d - part + split - 1) / split;   // rows part, part+split, ...
                if (ig >= nmine) break;
                const u32 ie = min(ig + G, nmine);
                for (u32 ii = ig; ii < ie; ++ii) {
                const u32 i = part + ii * split;
                const u64* Ri = R + (u64)i * Ws;
                const u64 myw = lane < Wd ? Ri[lane] : 0ull;
                const u32 nzw = __ballot_sync(G2M_FULL, myw != 0ull);
                if (!nzw) continue;
                if constexpr (K == 5) {
                    // 4-cliques with local source i = triangles of the sub-DAG on
                    // R_i. With n1 = |R_i| <= 128 its rows fit two words:
                    // S_k bit m <=> L1[m] in R_{L1[k]}, four ballots per k.
                    const u32 n1 = __reduce_add_sync(G2M_FULL, (u32)__popcll(myw));
                    if (n1 > 128 && n1 <= 256 && W >= 4 && g_cl5_big) {
                        // CTA-wide compressed phase below (LR is free after the probe)
                        if (lane == 0) LR[atomicAdd(&s_nbig, 1u)] = i;
                        continue;
                    }
                    if (n1 <= 128) {
                        // sub-DAG rows of up to 128 bits (two words): lane q*32+l holds
                        // candidate c[q]; S_k = ballots of "c in R_{L1[k]}"
                        compact_bits(Ri, 0, Wd, L1);
                        u32 c[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) c[q] = lane + 32u * q < n1 ? L1[lane + 32 * q] : 0u;
                        __syncwarp();
                        u64* SS = (u64*)L1;          // [n1][2] u64, over L1 and L2
                        for (u32 k = 0; k < n1; ++k) {
                            const u32 qk = k >> 5;
                            const u32 src = qk == 0 ? c[0] : (qk == 1 ? c[1] : (qk == 2 ? c[2] : c[3]));
                            const u64* Rk = R + (u64)__shfl_sync(G2M_FULL, src, k & 31u) * Ws;
                            u32 sw[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const bool bq = lane + 32u * q < n1 && (u32)q >= qk &&
                                                ((Rk[c[q] >> 6] >> (c[q] & 63u)) & 1ull);
                                sw[q] = __ballot_sync(G2M_FULL, bq);
                            }
                            if (lane == 0) {
                                SS[2 * k] = ((u64)sw[1] << 32) | sw[0];
                                SS[2 * k + 1] = ((u64)sw[3] << 32) | sw[2];
                            }
                        }
                        __syncwarp();
                        for (u32 k = lane; k < n1; k += 32) {
                            const u64 S0 = SS[2 * k], S1 = SS[2 * k + 1];
                            u64 it = S0;
                            while (it) {
                                const int l = __ffsll(it) - 1;
                                it &= it - 1;
                                acc += (u64)__popcll(S0 & SS[2 * l]) + (u64)__popcll(S1 & SS[2 * l + 1]);
                            }
                            it = S1;
                            while (it) {
                                const int l = 64 + __ffsll(it) - 1;
                                it &= it - 1;
                                acc += (u64)__popcll(S1 & SS[2 * l + 1]);
                            }
                        }
                        __syncwarp();
                        continue;
                    }
                }
                for (u32 c0 = 0; c0 < Wd; c0 += CH) {
                    if (!((nzw >> c0) & ((1u << CH) - 1u))) continue;
                    const u32 n1 = compact_bits(Ri, c0, min(c0 + CH, Wd), L1);
                    for (u32 e0 = 0; e0 < n1; e0 += 32) {
                        const u32 e = e0 + lane;
                        const bool isj = e < n1;
                        const u32 j = isj ? L1[e] : 0u;
                        const u64* Rj = R + (u64)j * Ws;
                        if constexpr (K == 4) {
                            if (isj) {
                                u32 m = nzw & ~((1u << (j >> 6)) - 1u);   // R_j is zero below word j/64
                                while (m) {
                                    const int q = __ffs(m) - 1;
                                    m &= m - 1;
                                    acc += (u64)__popcll(Ri[q] & Rj[q]);
                                }
                            }
                        } else {   // K == 5, rows with |R_i| > 64
                            u64 t2[W];
                            u32 c = 0;
#pragma unroll
                            for (int r = 0; r < W; ++r) {
                                t2[r] = (isj && r < (int)Wd && r >= (int)(j >> 6)) ? (Ri[r] & Rj[r]) : 0ull;
                                c += (u32)__popcll(t2[r]);
                            }
                            const bool heavy = c > 32;
                            if (isj && !heavy) {
#pragma unroll
                                for (int r = 0; r < W; ++r) {
                                    u64 bits = t2[r];
                                    while (bits) {
                                        const u32 l = r * 64 + (__ffsll(bits) - 1);
                                        bits &= bits - 1;
                                        const u64* Rl = R + (u64)l * Ws;
                                        const int lw = (int)(l >> 6);   // R_l is zero below word l/64
#pragma unroll
                                        for (int r2 = 0; r2 < W; ++r2)
                                            if (r2 >= lw && t2[r2]) acc += (u64)__popcll(t2[r2] & Rl[r2]);
                                    }
                                }
                            }
                            u32 hm = __ballot_sync(G2M_FULL, isj && heavy);
                            while (hm) {
                                const int hj = __ffs(hm) - 1;
                                hm &= hm - 1;
                                if ((int)lane == hj) {
#pragma unroll
                                    for (int r = 0; r < W; ++r) if (r < (int)Wd) t2s[r] = t2[r];
                                }
                                __syncwarp();
                                const u32 nz2 = __ballot_sync(G2M_FULL, lane < Wd && t2s[lane < Wd ? lane : 0] != 0ull);
                                for (u32 c2 = 0; c2 < Wd; c2 += CH) {
                                    if (!((nz2 >> c2) & ((1u << CH) - 1u))) continue;
                                    const u32 n2 = compact_bits(t2s, c2, min(c2 + CH, Wd), L2);
                                    for (u32 f = lane; f < n2; f += 32) {
                                        const u32 l = L2[f];
                                        const u64* Rl = R + (u64)l * Ws;
                                        u32 mq = nz2 & ~((1u << (l >> 6)) - 1u);   // R_l is zero below word l/64
                                        while (mq) {
                                            const int q3 = __ffs(mq) - 1;
                                            mq &= mq - 1;
                                            acc += (u64)__popcll(t2s[q3] & Rl[q3]);
                                        }
                                    }
                                    __syncwarp();
                                }
                            }
                        }
                    }
                    __syncwarp();
                }
                }
            }
            if constexpr (K == 5 && W >= 4) {
                // Deferred rows (128 < |R_i| <= 256): the whole CTA compresses R_i's
                // sub-DAG to 4-word rows S_k (bit m <=> CS[m] in R_{CS[k]}, 8 ballots
                // per k), then counts its triangles warp-per-k, lanes over the set bits
                // of S_k: 4 words per (k, l) instead of W per (j, l) on the per-warp path.
                // The union region is free once every warp has left the row loop.
                __syncthreads();
                const u32 nbig = s_nbig;
                u64* SS = (u64*)scr;                    // [256][4] u64
                u32* CS = scr + 2048;                   // [256] candidates of R_i
                u32* LW = CS + 256 + w * 256;           // per-warp set-bit list
                for (u32 bi = 0; bi < nbig; ++bi) {
                    const u32 i = LR[bi];
                    if (w == 0) {
                        const u32 n1 = compact_bits(R + (u64)i * Ws, 0, Wd, CS);
                        if (lane == 0) s_n1 = n1;
                    }
                    __syncthreads();
                    const u32 n1 = s_n1;
                    const u32 ng = (n1 + 31) >> 5;
                    for (u32 k = w; k < n1; k += NW) {
                        const u64* Rk = R + (u64)CS[k] * Ws;
                        u32 sw[8];
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            const u32 m = (u32)g * 32u + lane;
                            const bool bq = (u32)g < ng && (u32)g >= (k >> 5) && m < n1 &&
                                            ((Rk[CS[m] >> 6] >> (CS[m] & 63u)) & 1ull);
                            sw[g] = __ballot_sync(G2M_FULL, bq);
                        }
                        if (lane == 0) {
                            SS[4 * k] = ((u64)sw[1] << 32) | sw[0];
                            SS[4 * k + 1] = ((u64)sw[3] << 32) | sw[2];
                            SS[4 * k + 2] = ((u64)sw[5] << 32) | sw[4];
                            SS[4 * k + 3] = ((u64)sw[7] << 32) | sw[6];
                        }
                    }
                    __syncthreads();
                    for (u32 k = w; k < n1; k += NW) {
                        const u64* Sk = SS + 4 * k;
                        const u32 nl = compact_bits(Sk, 0, 4, LW);
                        for (u32 f = lane; f < nl; f += 32) {
                            const u32 l = LW[f];
                            const u64* Sl = SS + 4 * l;
#pragma unroll
                            for (u32 q = 0; q < 4; ++q)
                                if (q >= (l >> 6)) acc += (u64)__popcll(Sk[q] & Sl[q]);
                        }
                        __syncwarp();
                    }
                    __syncthreads();
                }
            }
        }
        // clear the window bits of this source (the bitmap stays all-zero between sources)
        if (use_bm)
            for (u32 x = threadIdx.x; x < d; x += NW * 32) BM[(A[x] - a0) >> 5] = 0;
        else if (use_tl)   // everything the two-level window wrote
            for (u32 x = threadIdx.x; x < 2u * ntop + 2u * d + (d + 1u) / 2u + 2u; x += NW * 32) BM[x] = 0;
        __syncthreads();
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// Bucket the sources of this partition by local-graph size class.
// class 0: d < K-1 (no clique), 8: d <= pair_maxd (pairs), 1: d <= 64 (warp), 2..5: d <= 128..1024
// (CTA, W = 2,4,8,16), 7: 1024 < d <= max_cta_d (CTA, W = 64; k = 3 only),
// 6: d > max_cta_d (generic kernel). span_max[c]: widest id window of class c.
__global__ void k_clique_bucket(const u64* off, const u32* nbr, u64 nv, int kmin1, u64 max_cta_d, u64 pair_maxd,
                                u64 rr_chunk, u32 parts, u32 part, const u64* wpre, u64 wchunk, u32* lists,
                                u64 list_stride, u64* sizes, u32* span_max) {
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x) {
        if (!g2m_owns(v, rr_chunk, parts, part, wpre, wchunk)) continue;
        const u64 b = off[v];
        const u64 d = off[v + 1] - b;
        int c;
        if (d < (u64)kmin1 || d == 0) continue;
        if (max_cta_d == 0) c = 6;   // every source to the generated plan kernel
        else if (d <= pair_maxd) c = 8;
        else if (d <= 64) c = 1;
        else if (d <= 128) c = 2;
        else if (d <= 256) c = 3;
        else if (d <= 512) c = 4;
        else if (d <= 1024) c = 5;
        else if (d <= max_cta_d) c = 7;
        else c = 6;
        // warp-aggregated append: one atomic per (warp, class) instead of per vertex
        const u32 peers = __match_any_sync(__activemask(), c);
        const u32 leader = __ffs(peers) - 1;
        u64 base = 0;
        if (g2m_lane() == leader) base = atomicAdd(sizes + c, (u64)__popc(peers));
        base = __shfl_sync(peers, base, leader);
        const u64 slot = base + __popc(peers & g2m_lanemask_lt());
        lists[(u64)c * list_stride + slot] = (u32)v;
        if (c >= 2 && c != 6) atomicMax(span_max + c, __ldg(nbr + b + d - 1) - __ldg(nbr + b) + 1u);
    }
}

// Σ_e C(t_e, 2): diamonds from per-edge triangle support (diamond = an edge
// plus an unordered pair of its common neighbours).
__global__ void k_sum_choose2(const u32* t, u64 n, u64* count) {
    u64 acc = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 c = t[i];
        acc += c * (c - 1) / 2;
    }
    acc = g2m_wsum(acc);
    if ((threadIdx.x & 31) == 0 && acc) g2m_add128(count, acc, 0);
}

// Hub-core bits (HubCore): one warp per core vertex a, a bit per out-neighbour.
__global__ void k_core_build(const u64* off, const u32* nbr, u64 nv, u32 lo, u32 T, u32* bits) {
    const u32 lane = g2m_lane();
    for (u64 al = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; al < T;
         al += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u64 a = lo + al;
        const u64 b0 = off[a], b1 = off[a + 1];
        const u64 base = HubCore::S((u64)T - 1) - HubCore::S((u64)T - 1 - al);
        for (u64 s = b0 + lane; s < b1; s += 32) {
            const u32 bit = nbr[s] - (u32)a - 1u;
            atomicOr(bits + base + (bit >> 5), 1u << (bit & 31u));
        }
    }
}

}  // namespace g2m_clique
