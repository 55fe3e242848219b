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
// Σ_{v1} Σ_{v ∈ N<(v1)} |N(v) ∩ [0, v1)| (Chiba-Nishizeki ordering).
//
// Tiers by the wedge bound W(v1) = Σ_{v ∈ N<(v1)} d(v):
//   1: W <= 512   one warp per v1, counters in a per-warp shared hash (1024)
//   2: W <= 8192  one CTA per v1, counters in a CTA shared hash (16384)
//   3: larger     one CTA per v1, dense u32 counters in a per-CTA HBM slab,
//                 cleared by a second walk over the same wedges.
#pragma once

#include "g2m_device.cuh"

namespace g2m_c4 {

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

// Walk the wedges v1 - L[i] - x (x < r1) of rows [i0, i0+32) of L (all 32
// lanes share the concatenated row prefixes) and apply f(x) to each x.
template <typename F>
__device__ __forceinline__ void wedges32(const u64* __restrict__ off, const u32* __restrict__ nbr,
                                         const u32* L, u32 l1, u32 i0, u32 r1, u32* scratch, F&& f) {
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
        rn = (dv && __ldg(nbr + ro + dv - 1) < r1) ? dv : g2m_lb(nbr + ro, dv, r1);
    }
    const u32 incl = g2m_scan_incl(rn);
    const u32 tot = __shfl_sync(G2M_FULL, incl, 31);
    fl_end[lane] = incl;
    fl_base[lane] = ro - (u64)(incl - rn);
    __syncwarp();
    u32 ow = 0;
    for (u32 e = lane; e < tot; e += 32) {
        while (fl_end[ow] <= e) ++ow;
        f(__ldg(nbr + (fl_base[ow] + e)));
    }
    __syncwarp();
}

// ---- tier 1: warp per v1 ---------------------------------------------------
template <int WPB>
__global__ void __launch_bounds__(WPB * 32)
k_c4_warp(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
          const u32* __restrict__ lows, u64 nverts, u64* next, u64* count) {
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
            wedges32(off, nbr, L, l1, i0, r1, sScr[w], [&](u32 x) { acc += hinc(K, Cn, CAP - 1, x); });
        for (u32 x = lane; x < CAP; x += 32) { K[x] = G2M_EMPTY; Cn[x] = 0; }
        __syncwarp();
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// ---- tier 2/3: CTA per v1 -----------------------------------------------------
// GLOBAL = false: counters in a shared hash of CAP entries (dynamic smem);
// GLOBAL = true: dense counters cnt[x] in this block's HBM slab (n words).
template <int NW, bool GLOBAL>
__global__ void __launch_bounds__(NW * 32)
k_c4_cta(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
         const u32* __restrict__ lows, u64 nverts, u64* next, u64* count, u32* slab, u64 slab_words,
         u32 cap) {
    extern __shared__ __align__(16) u32 smem_c4[];
    u32* K = smem_c4;                 // shared hash keys [cap], counts [cap]   (!GLOBAL)
    u32* Cn = K + (GLOBAL ? 0 : cap);
    u32* scr = Cn + (GLOBAL ? 0 : cap);
    u32* dense = slab + (u64)blockIdx.x * slab_words;
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    u32* wscr = scr + w * 96;
    __shared__ u64 s_t;
    __shared__ u32 s_row, s_row2;
    if (!GLOBAL)
        for (u32 x = threadIdx.x; x < cap; x += NW * 32) { K[x] = G2M_EMPTY; Cn[x] = 0; }
    u64 acc = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            s_t = atomicAdd(next, 1ull);
            s_row = 0;
            s_row2 = 0;
        }
        __syncthreads();
        const u64 t = s_t;
        if (t >= nverts) break;
        const u32 r1 = __ldg(verts + t);
        const u32 l1 = __ldg(lows + t);
        const u32* L = nbr + __ldg(off + r1);
        for (;;) {
            u32 i0 = 0;
            if (lane == 0) i0 = atomicAdd(&s_row, 32u);
            i0 = __shfl_sync(G2M_FULL, i0, 0);
            if (i0 >= l1) break;
            if (GLOBAL)
                wedges32(off, nbr, L, l1, i0, r1, wscr, [&](u32 x) { acc += atomicAdd(dense + x, 1u); });
            else
                wedges32(off, nbr, L, l1, i0, r1, wscr, [&](u32 x) { acc += hinc(K, Cn, cap - 1, x); });
        }
        __syncthreads();
        if (GLOBAL) {   // clear the counters this v1 touched
            for (;;) {
                u32 i0 = 0;
                if (lane == 0) i0 = atomicAdd(&s_row2, 32u);
                i0 = __shfl_sync(G2M_FULL, i0, 0);
                if (i0 >= l1) break;
                wedges32(off, nbr, L, l1, i0, r1, wscr, [&](u32 x) { dense[x] = 0; });
            }
        } else {
            for (u32 x = threadIdx.x; x < cap; x += NW * 32) { K[x] = G2M_EMPTY; Cn[x] = 0; }
        }
        __syncthreads();
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// Per v1 (rank r, this partition): l1 = |N(r) ∩ [0, r)| and the wedge bound
// W = Σ_{v ∈ N<(r)} d(v); class 1..3 as above (0: l1 < 2, no cycle).
// One warp per vertex.
__global__ void k_c4_bucket(const u64* off, const u32* nbr, u64 nv, u64 rr_chunk, u32 parts, u32 part,
                            u32* lists, u32* lows, u64* wkeys, u64 stride, u64* sizes) {
    const u32 lane = g2m_lane();
    for (u64 r = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; r < nv;
         r += ((u64)gridDim.x * blockDim.x) >> 5) {
        if (rr_chunk && ((r / rr_chunk) % parts) != part) continue;
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
            const int c = wsum <= 512 ? 1 : (wsum <= 8192 ? 2 : 3);
            const u64 slot = atomicAdd(sizes + c, 1ull);
            lists[(u64)c * stride + slot] = (u32)r;
            lows[(u64)c * stride + slot] = l1;
            if (c == 3) wkeys[slot] = ((u64)(0xffffffffu - (u32)min(wsum, 0xffffffffull)) << 32) | r;   // descending W (LPT order)
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
