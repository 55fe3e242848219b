// cycle4_kernels.cuh -- 4-cycle counting by wedge aggregation (count mode of
// subgraph listing with the 4-cycle pattern; reference plan: PAPER.md §A.2
// "4-cycle (buffers=0, Ω reduced)", executor.py:218-325).
//
// The reference enumerates, per 4-cycle, its unique symmetry-broken
// embedding (v1 > v2 > v3, v4 < v1) and counts |N(v2) ∩ N(v3) ∩ [0, v1)|.
// The number of 4-cycles is invariant under vertex renaming,
// so the kernels count the same set with v1 = the highest-ranked vertex of
// the cycle in the (degree, id) order (rank-space CSR, g2m.cu ensure_rank):
//
//   #C4 = Σ_{v1} Σ_{x < v1} C(c(x), 2),
//   c(x) = |{ v ∈ N(v1) : v < v1, x ∈ N(v) }|        (x < v1, ranks)
//
// i.e. every wedge v1 - v - x below v1 increments c(x); a cycle is a pair of
// wedges with the same ends. C(c,2) accumulates incrementally: an increment
// that finds the old value k adds k (C(k+1,2) - C(k,2) = k). In rank space
// N(v) ∩ [0, v1) is a prefix of the sorted row, so the wedge work is
// Σ_{v1} Σ_{v ∈ N<(v1)} |N(v) ∩ [0, v1)| (Chiba-Nishizeki ordering). Wedge
// ends of degree 1 (ranks below lo_x) can never close a cycle and are skipped.
//
// Tiers by the wedge bound W(v1) = Σ_{v ∈ N<(v1)} d(v):
//   1: W <= 512       one warp per v1, counters in a per-warp shared hash
//   2: W <= 8192      one CTA per v1, counters in a CTA shared hash
//   3: W <= stage cap one CTA per v1: the wedge ends are bucketed by id range
//                     into an HBM staging area (histogram, scan, scatter) and
//                     each 1024-id bucket is counted by one warp in shared
//                     memory -- streaming HBM traffic instead of random
//                     counter updates
//   4: larger         all blocks on one v1 at a time, dense counters shared
//                     by the grid, one L2-sized id range per pass, cleared
//                     by memset
#pragma once

#include "g2m_device.cuh"

namespace g2m_c4 {

constexpr u32 kBucketBits = 10;          // tier 3: ids per bucket = 1024 (one warp's counters)
constexpr u32 kBucketIds = 1u << kBucketBits;

// Counter table: increment the count of x, return its old value.
__device__ __forceinline__ u32 hinc(u32* keys, u32* cnt, u32 mask, u32 x) {
    u32 h = (x * 0x9E3779B1u) & mask;
    for (;;) {
        const u32 k = keys[h];
        if (k == x) return atomicAdd(cnt + h, 1u);
        if (k == G2M_EMPTY) {
            const u32 p = atomicCAS(keys + h, G2M_EMPTY, x);
            if (p == G2M_EMPTY || p == x) return atomicAdd(cnt + h, 1u);
        }
        h = (h + 1) & mask;
    }
}

// Walk the wedges v1 - L[i] - x (lo_x <= x < r1) of rows [i0, i0+32) of L
// (all 32 lanes share the concatenated row segments) and apply f(x).
template <typename F>
__device__ __forceinline__ void wedges32(const u64* __restrict__ off, const u32* __restrict__ nbr,
                                         const u32* L, u32 l1, u32 i0, u32 r1, u32 lo_x, u32* scratch, F&& f) {
    const u32 lane = g2m_lane();
    u32* fl_end = scratch;
    u64* fl_base = (u64*)(scratch + 32);
    const u32 i = i0 + lane;
    u64 ro = 0;
    u32 rn = 0;
    if (i < l1) {
        const u32 v = L[i];
        ro = __ldg(off + v);
        const u32 dv = (u32)(__ldg(off + v + 1) - ro);
        const u32 s0 = (dv && __ldg(nbr + ro) < lo_x) ? g2m_lb(nbr + ro, dv, lo_x) : 0u;
        const u32 e1 = (dv && __ldg(nbr + ro + dv - 1) < r1) ? dv : g2m_lb(nbr + ro, dv, r1);
        rn = e1 > s0 ? e1 - s0 : 0u;
        ro += s0;
    }
    const u32 incl = g2m_scan_incl(rn);
    const u32 tot = __shfl_sync(G2M_FULL, incl, 31);
    fl_end[lane] = incl;
    fl_base[lane] = ro - (u64)(incl - rn);
    __syncwarp();
    u32 ow = 0;
    for (u32 e0 = 0; e0 < tot; e0 += 64) {   // two elements per lane in flight
        const u32 ea = e0 + lane, eb = ea + 32;
        u32 xa = 0, xb = 0;
        if (ea < tot) {
            while (fl_end[ow] <= ea) ++ow;
            xa = __ldg(nbr + (fl_base[ow] + ea));
        }
        if (eb < tot) {
            u32 ob = ow;
            while (fl_end[ob] <= eb) ++ob;
            xb = __ldg(nbr + (fl_base[ob] + eb));
            ow = ob;
        }
        if (ea < tot) f(xa);
        if (eb < tot) f(xb);
    }
    __syncwarp();
}

// Row batches of L in dynamic 32-row grabs from a shared (CTA) or global
// (grid) counter; f as in wedges32.
template <typename F>
__device__ __forceinline__ void wedge_rows(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* L,
                                           u32 l1, u32 r1, u32 lo_x, u32* ctr, u32* scratch, F&& f) {
    const u32 lane = g2m_lane();
    for (;;) {
        u32 i0 = 0;
        if (lane == 0) i0 = atomicAdd(ctr, 32u);
        i0 = __shfl_sync(G2M_FULL, i0, 0);
        if (i0 >= l1) break;
        wedges32(off, nbr, L, l1, i0, r1, lo_x, scratch, f);
    }
}

// ---- tier 1: warp per v1 ---------------------------------------------------
template <int WPB>
__global__ void __launch_bounds__(WPB * 32)
k_c4_warp(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
          const u32* __restrict__ lows, u64 nverts, u64* next, u64* count, u32 lo_x) {
    constexpr u32 CAP = 1024;
    __shared__ u32 sK[WPB][CAP];
    __shared__ u32 sC[WPB][CAP];
    __shared__ __align__(8) u32 sScr[WPB][96];
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    u32* K = sK[w];
    u32* Cn = sC[w];
    for (u32 x = lane; x < CAP; x += 32) { K[x] = G2M_EMPTY; Cn[x] = 0; }
    __syncwarp();
    u64 acc = 0;
    for (;;) {
        u64 t = 0;
        if (lane == 0) t = atomicAdd(next, 1ull);
        t = __shfl_sync(G2M_FULL, t, 0);
        if (t >= nverts) break;
        const u32 r1 = __ldg(verts + t);
        const u32 l1 = __ldg(lows + t);
        const u32* L = nbr + __ldg(off + r1);
        for (u32 i0 = 0; i0 < l1; i0 += 32)
            wedges32(off, nbr, L, l1, i0, r1, lo_x, sScr[w], [&](u32 x) { acc += hinc(K, Cn, CAP - 1, x); });
        for (u32 x = lane; x < CAP; x += 32) { K[x] = G2M_EMPTY; Cn[x] = 0; }
        __syncwarp();
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// ---- tier 2: CTA per v1, shared hash of `cap` counters ----------------------
template <int NW>
__global__ void __launch_bounds__(NW * 32)
k_c4_cta(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
         const u32* __restrict__ lows, u64 nverts, u64* next, u64* count, u32 cap, u32 lo_x) {
    extern __shared__ __align__(16) u32 smem_c4[];
    u32* K = smem_c4;                 // keys [cap], counts [cap], per-warp scratch [NW x 96]
    u32* Cn = K + cap;
    u32* wscr = Cn + cap + (threadIdx.x >> 5) * 96;
    const u32 lane = g2m_lane();
    __shared__ u64 s_t;
    __shared__ u32 s_row;
    for (u32 x = threadIdx.x; x < cap; x += NW * 32) { K[x] = G2M_EMPTY; Cn[x] = 0; }
    u64 acc = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            s_t = atomicAdd(next, 1ull);
            s_row = 0;
        }
        __syncthreads();
        const u64 t = s_t;
        if (t >= nverts) break;
        const u32 r1 = __ldg(verts + t);
        const u32 l1 = __ldg(lows + t);
        const u32* L = nbr + __ldg(off + r1);
        wedge_rows(off, nbr, L, l1, r1, lo_x, &s_row, wscr, [&](u32 x) { acc += hinc(K, Cn, cap - 1, x); });
        __syncthreads();
        for (u32 x = threadIdx.x; x < cap; x += NW * 32) { K[x] = G2M_EMPTY; Cn[x] = 0; }
        __syncthreads();
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// CTA-wide exclusive scan of H[0, nb) in place (every warp scans one chunk,
// warp 0 scans the chunk totals) and the compaction of the non-empty buckets
// into NBL (ascending), *nne of them. WT: 2 * NW words of scratch.
template <int NW>
__device__ __forceinline__ void cta_scan_compact(u32* H, u32 nb, u32* NBL, u32* WT, u32* nne) {
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    const u32 ch = ((nb + NW - 1) / NW + 31u) & ~31u;         // chunk per warp, multiple of 32
    const u32 c0 = min(nb, w * ch), c1 = min(nb, c0 + ch);
    u32 sum = 0, cnt = 0;
    for (u32 b0 = c0; b0 < c1; b0 += 32) {
        const u32 b = b0 + lane;
        const u32 v = b < c1 ? H[b] : 0u;
        const u32 incl = g2m_scan_incl(v);
        sum += __shfl_sync(G2M_FULL, incl, 31);
        cnt += __popc(__ballot_sync(G2M_FULL, v != 0u));
    }
    if (lane == 0) { WT[w] = sum; WT[NW + w] = cnt; }
    __syncthreads();
    if (w == 0) {
        const u32 a = lane < NW ? WT[lane] : 0u, c = lane < NW ? WT[NW + lane] : 0u;
        const u32 ia = g2m_scan_incl(a), ic = g2m_scan_incl(c);
        if (lane < NW) { WT[lane] = ia - a; WT[NW + lane] = ic - c; }
        if (lane == 31) *nne = ic;
    }
    __syncthreads();
    u32 carry = WT[w], ccarry = WT[NW + w];
    for (u32 b0 = c0; b0 < c1; b0 += 32) {
        const u32 b = b0 + lane;
        const u32 v = b < c1 ? H[b] : 0u;
        const u32 incl = g2m_scan_incl(v);
        const u32 m = __ballot_sync(G2M_FULL, v != 0u);
        if (b < c1) H[b] = carry + incl - v;
        if (v) NBL[ccarry + __popc(m & g2m_lanemask_lt())] = b;
        carry += __shfl_sync(G2M_FULL, incl, 31);
        ccarry += __popc(m);
    }
    __syncthreads();
}

// ---- tier 3: CTA per v1, bucketed staging ------------------------------------
// Shared memory: bucket histogram -> cursors -> bucket ends [nbmax] u32 |
// per-warp counters [NW x 1024] u32 | per-warp scratch [NW x 96] u32.
// stage: this block's slab of stage_cap u32 in HBM.
__host__ __device__ constexpr size_t stage_smem_bytes(int NW, u32 nbmax) {
    return (size_t)4 * nbmax + (size_t)4 * NW * kBucketIds + (size_t)4 * NW * 96 + (size_t)4 * nbmax +
           (size_t)4 * 2 * NW;
}

template <int NW>
__global__ void __launch_bounds__(NW * 32)
k_c4_stage(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
           const u32* __restrict__ lows, u64 nverts, u64* next, u64* count, u32* stage_all, u64 stage_cap,
           u32 nbmax, u32 lo_x) {
    extern __shared__ __align__(16) u32 smem_c4[];
    u32* H = smem_c4;
    u32* WC = H + nbmax;
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    u32* wcnt = WC + w * kBucketIds;
    u32* wscr = WC + NW * kBucketIds + w * 96;
    u32* NBL = WC + NW * kBucketIds + NW * 96;   // non-empty buckets [nbmax]
    u32* WT = NBL + nbmax;                       // scan scratch [2 NW]
    u32* stage = stage_all + (u64)blockIdx.x * stage_cap;
    __shared__ u64 s_t;
    __shared__ u32 s_row, s_row2, s_bkt, s_nne;
    for (u32 x = lane; x < kBucketIds; x += 32) wcnt[x] = 0;
    u64 acc = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            s_t = atomicAdd(next, 1ull);
            s_row = s_row2 = s_bkt = 0;
        }
        __syncthreads();
        const u64 t = s_t;
        if (t >= nverts) break;
        const u32 r1 = __ldg(verts + t);
        const u32 l1 = __ldg(lows + t);
        const u32* L = nbr + __ldg(off + r1);
        const u32 nb = (r1 >> kBucketBits) + 1;
        for (u32 b = threadIdx.x; b < nb; b += NW * 32) H[b] = 0;
        __syncthreads();
        // 1: histogram of the wedge ends by bucket
        wedge_rows(off, nbr, L, l1, r1, lo_x, &s_row, wscr, [&](u32 x) { atomicAdd(H + (x >> kBucketBits), 1u); });
        __syncthreads();
        // 2: exclusive scan of the histogram (CTA-wide): cursors = bucket starts;
        //    the non-empty buckets listed for step 4
        cta_scan_compact<NW>(H, nb, NBL, WT, &s_nne);
        const u32 nne = s_nne;
        // 3: scatter the wedge ends into their buckets (cursors end as bucket ends)
        wedge_rows(off, nbr, L, l1, r1, lo_x, &s_row2, wscr, [&](u32 x) {
            stage[atomicAdd(H + (x >> kBucketBits), 1u)] = x;
        });
        __syncthreads();
        // 4: one warp per bucket counts it in its private shared counters
        for (;;) {
            u32 b = 0;
            if (lane == 0) b = atomicAdd(&s_bkt, 1u);
            b = __shfl_sync(G2M_FULL, b, 0);
            if (b >= nne) break;
            b = NBL[b];
            const u32 s0 = b ? H[b - 1] : 0u, s1 = H[b];
            for (u32 e = s0 + lane; e < s1; e += 32) acc += atomicAdd(wcnt + (stage[e] & (kBucketIds - 1)), 1u);
            __syncwarp();
            for (u32 e = s0 + lane; e < s1; e += 32) wcnt[stage[e] & (kBucketIds - 1)] = 0;
            __syncwarp();
        }
        __syncthreads();
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// ---- tier 3, coarse buckets ----------------------------------------------------
// As k_c4_stage, but the wedge ends are partitioned into 32K-id buckets (a
// few hundred per v1 instead of r1/1024): the scatter then has few enough
// open write cursors per block that L2 combines the partial-sector writes
// instead of evicting them to DRAM. Each bucket is counted by the whole CTA
// in dense shared counters, cleared by a re-walk (or densely when the
// bucket is large).
constexpr u32 kCoarseBits = 15;
constexpr u32 kCoarseIds = 1u << kCoarseBits;

// Count-phase rounds (G2M_C4_ROUNDS): consecutive small buckets (<= kRoundEntries
// entries in total, <= kRoundBuckets buckets) are counted together, warp-privately:
// the round's entries are counting-sorted in shared memory by (bucket, 1024-id
// sub-range), and each warp counts its (bucket, sub-range) groups in its own
// 1024-counter slice of C -- a few CTA barriers per round instead of two per
// bucket (a top vertex of RMAT-27 has up to 4096 coarse buckets, most of them
// holding a handful of wedge ends).
constexpr u32 kRoundEntries = 8192;
constexpr u32 kRoundBuckets = 64;
constexpr u32 kRoundKeys = kRoundBuckets * (kCoarseIds >> 10);   // (bucket, sub-range) groups

__host__ __device__ constexpr size_t stage2_smem_bytes(int NW, u32 nbmax) {
    return (size_t)4 * nbmax + (size_t)4 * kCoarseIds + (size_t)4 * NW * 96 + (size_t)4 * kRoundEntries +
           (size_t)4 * (kRoundKeys + 1) + (size_t)4 * nbmax + (size_t)4 * 2 * NW;
}

__device__ u32 g_c4_rounds = 1;



template <int NW>
__global__ void __launch_bounds__(NW * 32, 1)
k_c4_stage2(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
            const u32* __restrict__ lows, u64 nverts, u64* next, u64* count, u32* stage_all, u64 stage_cap,
            u32 nbmax, u32 lo_x) {
    extern __shared__ __align__(16) u32 smem_c4[];
    constexpr u32 NT = NW * 32;
    u32* H = smem_c4;
    u32* C = H + nbmax;
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    u32* wscr = C + kCoarseIds + w * 96;
    u32* RS = C + kCoarseIds + NW * 96;          // round staging [kRoundEntries]
    u32* RK = RS + kRoundEntries;                // round group cursors [kRoundKeys + 1]
    u32* NBL = RK + kRoundKeys + 1;              // non-empty buckets [nbmax]
    u32* WT = NBL + nbmax;                       // scan scratch [2 NW]
    __shared__ u32 s_nne;
    u32* stage = stage_all + (u64)blockIdx.x * stage_cap;
    __shared__ u64 s_t;
    __shared__ u32 s_row, s_row2;
    for (u32 x = threadIdx.x; x < kCoarseIds; x += NT) C[x] = 0;
    u64 acc = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            s_t = atomicAdd(next, 1ull);
            s_row = s_row2 = 0;
        }
        __syncthreads();
        const u64 t = s_t;
        if (t >= nverts) break;
        const u32 r1 = __ldg(verts + t);
        const u32 l1 = __ldg(lows + t);
        const u32* L = nbr + __ldg(off + r1);
        const u32 nb = (r1 >> kCoarseBits) + 1;
        for (u32 b = threadIdx.x; b < nb; b += NT) H[b] = 0;
        __syncthreads();
        wedge_rows(off, nbr, L, l1, r1, lo_x, &s_row, wscr, [&](u32 x) { atomicAdd(H + (x >> kCoarseBits), 1u); });
        __syncthreads();
        // CTA-wide scan (bucket starts) + the list of non-empty buckets: the count
        // phase visits only those (a warp-0 scan and a walk over every bucket id
        // were 38 % of the stall samples, profiles/r02/hotspots_r02t.txt)
        cta_scan_compact<NW>(H, nb, NBL, WT, &s_nne);
        const u32 nne = s_nne;
        wedge_rows(off, nbr, L, l1, r1, lo_x, &s_row2, wscr, [&](u32 x) {
            stage[atomicAdd(H + (x >> kCoarseBits), 1u)] = x;
        });
        __syncthreads();
        for (u32 k = 0; k < nne;) {
            const u32 b = NBL[k];
            const u32 s0 = b ? H[b - 1] : 0u, s1 = H[b];
            if (g_c4_rounds && s1 - s0 <= kRoundEntries) {
                // a round: non-empty buckets NBL[k, ke) within kRoundBuckets ids of b,
                // <= kRoundEntries entries in total; they end at bucket be - 1
                u32 ke = k + 1;
                while (ke < nne && NBL[ke] - b < kRoundBuckets && H[NBL[ke]] - s0 <= kRoundEntries) ++ke;
                const u32 be = NBL[ke - 1] + 1;
                const u32 tot = H[be - 1] - s0;
                const u32 nkey = (be - b) << (kCoarseBits - 10);
                for (u32 x = threadIdx.x; x <= nkey; x += NT) RK[x] = 0;
                __syncthreads();
                // key = (bucket - b) * 32 + 1024-id sub-range; bucket of entry e from its id
                for (u32 e = threadIdx.x; e < tot; e += NT) {
                    const u32 x = stage[s0 + e];
                    const u32 key = (((x >> kCoarseBits) - b) << (kCoarseBits - 10)) | ((x >> 10) & 31u);
                    atomicAdd(RK + key + 1, 1u);
                }
                __syncthreads();
                if (w == 0) {       // inclusive scan of RK[1..nkey] -> group starts RK[0..nkey]
                    u32 carry = 0;
                    for (u32 q0 = 1; q0 <= nkey; q0 += 32) {
                        const u32 q = q0 + lane;
                        const u32 v = q <= nkey ? RK[q] : 0u;
                        const u32 incl = g2m_scan_incl(v);
                        if (q <= nkey) RK[q] = carry + incl;
                        carry += __shfl_sync(G2M_FULL, incl, 31);
                    }
                }
                __syncthreads();
                // scatter into the round staging area (group cursors start at RK[key])
                for (u32 e = threadIdx.x; e < tot; e += NT) {
                    const u32 x = stage[s0 + e];
                    const u32 key = (((x >> kCoarseBits) - b) << (kCoarseBits - 10)) | ((x >> 10) & 31u);
                    RS[atomicAdd(RK + key, 1u)] = x;
                }
                __syncthreads();
                // RK[key] is now the end of group key (its start is RK[key - 1], 0 for key 0)
                u32* Cw = C + w * 1024u;
                for (u32 key = w; key < nkey; key += NW) {
                    const u32 g0 = key ? RK[key - 1] : 0u, g1 = RK[key];
                    if (g0 == g1) continue;
                    for (u32 e = g0 + lane; e < g1; e += 32) acc += atomicAdd(Cw + (RS[e] & 1023u), 1u);
                    __syncwarp();
                    for (u32 e = g0 + lane; e < g1; e += 32) Cw[RS[e] & 1023u] = 0;
                    __syncwarp();
                }
                __syncthreads();
                k = ke;
                continue;
            }
            for (u32 e = s0 + threadIdx.x; e < s1; e += NT) acc += atomicAdd(C + (stage[e] & (kCoarseIds - 1)), 1u);
            __syncthreads();
            if (s1 - s0 > kCoarseIds / 4) {
                for (u32 x = threadIdx.x; x < kCoarseIds; x += NT) C[x] = 0;
            } else {
                for (u32 e = s0 + threadIdx.x; e < s1; e += NT) C[stage[e] & (kCoarseIds - 1)] = 0;
            }
            __syncthreads();
            ++k;
        }
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// ---- tier 4: the whole grid on one v1, shared dense counters -----------------
// The v1's wedges are flattened over the grid: k_c4_rows writes each row's
// wedge count and first nbr index, a scan makes the ends, and k_c4_grid's
// warps take 1024-element steps (owner row by binary search over the ends),
// so a few huge rows do not serialise the grid. The wedge ends are counted
// one id range [lo, hi) at a time: dense counters for the range only, sized
// to stay L2-resident whatever |V| is (RMAT-27: 134 M ids would be 537 MB of
// counters, random atomics in HBM). Rows are sorted, so N(v) ∩ [lo, hi) is
// one contiguous segment: the passes partition the wedges, the only extra
// work per pass is two binary searches per row.
__global__ void k_c4_rows(const u64* __restrict__ off, const u32* __restrict__ nbr, u32 r1, u32 l1, u32 lo,
                          u32 hi, u64* rn_out, u64* rb_out) {
    const u32* L = nbr + __ldg(off + r1);
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < l1; i += gridDim.x * blockDim.x) {
        const u32 v = __ldg(L + i);
        u64 ro = __ldg(off + v);
        const u32 dv = (u32)(__ldg(off + v + 1) - ro);
        const u32 s0 = (dv && __ldg(nbr + ro) < lo) ? g2m_lb(nbr + ro, dv, lo) : 0u;
        const u32 e1 = (dv && __ldg(nbr + ro + dv - 1) < hi) ? dv : g2m_lb(nbr + ro, dv, hi);
        rn_out[i] = e1 > s0 ? e1 - s0 : 0u;
        rb_out[i] = ro + s0;
    }
}

// rb[i] -= start of row i in the flattening, so element e of row i is nbr[rb[i] + e]
__global__ void k_c4_base(u32 l1, const u64* __restrict__ rn, u64* rb, const u64* __restrict__ re) {
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < l1; i += gridDim.x * blockDim.x)
        rb[i] -= re[i] - rn[i];
}

// RED variant (template RED): increments without a return value (fire-and-
// forget L2 reductions); the pair counts C(c, 2) come from k_c4_sweep, which
// also clears the range.
template <bool RED>
__global__ void __launch_bounds__(512)
k_c4_grid(const u32* __restrict__ nbr, u32 l1, const u64* __restrict__ rn, const u64* __restrict__ rb,
          const u64* __restrict__ re, u64* ctr, u32* dense, u32 lo, u64* count) {
    const u32 lane = g2m_lane();
    const u64 tot = re[l1 - 1];
    u64 acc = 0;
    for (;;) {
        u64 e0 = 0;
        if (lane == 0) e0 = atomicAdd(ctr, 1024ull);
        e0 = __shfl_sync(G2M_FULL, e0, 0);
        if (e0 >= tot) break;
        // owner of e0: first row with end > e0
        u32 ow = 0, n = l1;
        while (n > 0) {
            const u32 h = n >> 1;
            if (__ldg(re + ow + h) <= e0) { ow += h + 1; n -= h + 1; } else n = h;
        }
#pragma unroll 4
        for (u32 k = 0; k < 1024; k += 32) {
            const u64 e = e0 + k + lane;
            if (e < tot) {
                while (__ldg(re + ow) <= e) ++ow;
                if constexpr (RED) atomicAdd(dense + (__ldg(nbr + __ldg(rb + ow) + e) - lo), 1u);
                else acc += atomicAdd(dense + (__ldg(nbr + __ldg(rb + ow) + e) - lo), 1u);
            }
        }
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// Σ C(c, 2) over counters [0, n) (u32, 4 per thread as one u128 load) and clear them.
__global__ void k_c4_sweep(u32* dense, u64 n, u64* count) {
    u64 acc = 0;
    const u64 n4 = n >> 2;
    uint4* d4 = reinterpret_cast<uint4*>(dense);
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n4; i += (u64)gridDim.x * blockDim.x) {
        const uint4 v = d4[i];
        if (v.x | v.y | v.z | v.w) {
            acc += (u64)v.x * (v.x - 1) / 2 + (u64)v.y * (v.y - 1) / 2 + (u64)v.z * (v.z - 1) / 2 +
                   (u64)v.w * (v.w - 1) / 2;
            d4[i] = make_uint4(0, 0, 0, 0);
        }
    }
    for (u64 i = (n4 << 2) + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 c = dense[i];
        acc += c * (c - (c ? 1 : 0)) / 2;
        dense[i] = 0;
    }
    acc = g2m_wsum(acc);
    if ((threadIdx.x & 31) == 0 && acc) g2m_add128(count, acc, 0);
}

// Per v1 (rank r, this partition): l1 = |N(r) ∩ [0, r)| and the wedge bound
// W = Σ_{v ∈ N<(r)} d(v); class 1..4 as above (0: l1 < 2, no cycle).
// One warp per vertex.
__global__ void k_c4_bucket(const u64* off, const u32* nbr, u64 nv, u64 rr_chunk, u32 parts, u32 part,
                            const u64* wpre, u64 wchunk, u64 stage_cap, u32* lists, u32* lows, u64* wkeys,
                            u64 stride, u64* sizes) {
    const u32 lane = g2m_lane();
    for (u64 r = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; r < nv;
         r += ((u64)gridDim.x * blockDim.x) >> 5) {
        if (!g2m_owns(r, rr_chunk, parts, part, wpre, wchunk)) continue;
        const u64 b = off[r];
        const u32 d = (u32)(off[r + 1] - b);
        const u32 l1 = g2m_wlb(nbr + b, d, (u32)r);
        if (l1 < 2) continue;
        u64 wsum = 0;
        for (u32 i = lane; i < l1; i += 32) {
            const u32 v = __ldg(nbr + b + i);
            wsum += __ldg(off + v + 1) - __ldg(off + v);
        }
        wsum = g2m_wsum(wsum);
        if (lane == 0) {
            const int c = wsum <= 512 ? 1 : (wsum <= 8192 ? 2 : (wsum <= stage_cap ? 3 : 4));
            const u64 slot = atomicAdd(sizes + c, 1ull);
            atomicAdd(sizes + 5 + c, wsum);     // wedge bound per tier (debug / balance)
            lists[(u64)c * stride + slot] = (u32)r;
            lows[(u64)c * stride + slot] = l1;
            if (c == 3)   // descending W (LPT order)
                wkeys[slot] = ((u64)(0xffffffffu - (u32)min(wsum, 0xffffffffull)) << 32) | r;
        }
    }
}

__global__ void k_c4_unpack(const u64* keys, u64 n, const u64* off, const u32* nbr, u32* verts, u32* lows) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u32 r = (u32)keys[i];
        verts[i] = r;
        const u64 b = off[r];
        lows[i] = g2m_lb(nbr + b, (u32)(off[r + 1] - b), r);
    }
}

}  // namespace g2m_c4
