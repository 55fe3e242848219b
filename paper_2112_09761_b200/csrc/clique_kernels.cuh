// clique_kernels.cuh -- bitmap local-graph search (LGS) for k-clique counting
// on the degree-oriented DAG (G²Miner LGS; reference
// _LocalRunner executor.py:415-523, setops.build_local_graph
// setops.py:124-142, mask/popcount helpers setops.py:145-173).
//
// Every k-clique of an oriented graph has a unique source u (its minimum in
// the (degree, id) order). With A = N+(u) renamed to local ids 0..d-1
// (ascending ids, as the reference's LocalGraph), row R[i] is the bitmap of
// A ∩ N+(A[i]); the k-cliques with source u are exactly the (k-1)-cliques of
// the local DAG R, counted with AND + popcount:
//   k=3: Σ_i |R_i|     k=4: Σ_i Σ_{j∈R_i} |R_i & R_j|
//   k=5: Σ_i Σ_{j∈R_i} Σ_{l∈R_i&R_j} |R_i & R_j & R_l|
// so counts equal the reference's sorted-list plan (the same cliques).
//
// Tiers: d <= 64 -> one warp per source, single-word rows in shared memory;
// 64 < d <= 64*W -> one CTA per source, W-word rows in shared memory.
// Sources with d > 1024 are left to the generic plan kernel.
#pragma once

#include "g2m_device.cuh"

namespace g2m_clique {

// Stream the neighbour lists of rows [i0, i0+32) of A, test each element for
// membership in A (shared, sorted) and set the row bits (row stride W words).
// A's local ids come from a shared hash map (hk/hv, 2^hl slots); rows have
// an odd u64 stride W so that lanes reading different rows spread over banks.
__device__ __forceinline__ void build_rows(const u64* __restrict__ off, const u32* __restrict__ nbr,
                                           const u32* A, u32 d, u32 i0, u64* R, u32 W,
                                           u32* fl_end, u64* fl_off, u32* fl_row,
                                           const u32* hk, const u32* hv, u32 hl) {
    const u32 lane = g2m_lane();
    const u32 i = i0 + lane;
    const u32 lo = A[0], hi = A[d - 1];
    u64 ro = 0;
    u32 rn = 0;
    if (i < d) {
        const u32 v = A[i];
        ro = __ldg(off + v);
        rn = (u32)(__ldg(off + v + 1) - ro);
        if (rn > 48) {   // cut the parts of long lists that cannot hit [A0, A(d-1)]
            const u32* p = nbr + ro;
            const u32 s = g2m_lb(p, rn, lo);
            const u32 e = g2m_lb(p, rn, hi + 1u);
            ro += s;
            rn = e - s;
        }
    }
    const u32 incl = g2m_scan_incl(rn);
    const u32 tot = __shfl_sync(G2M_FULL, incl, 31);
    fl_end[lane] = incl;
    fl_off[lane] = ro;
    fl_row[lane] = i;
    __syncwarp();
    u32 ow = 0;
    for (u32 e = lane; e < tot; e += 32) {
        while (fl_end[ow] <= e) ++ow;
        const u32 st = ow ? fl_end[ow - 1] : 0u;
        const u32 x = __ldg(nbr + fl_off[ow] + (e - st));
        if (x >= lo && x <= hi) {
            const u32 pos = g2m_hmap_get(hk, hv, hl, x);
            if (pos != G2M_EMPTY)   // 32-bit halves: native ATOMS.OR (64-bit would be a CAS loop)
                atomicOr((u32*)(R + (u64)fl_row[ow] * W) + (pos >> 5), 1u << (pos & 31));
        }
    }
    __syncwarp();
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
template <int K, int WPB>
__global__ void __launch_bounds__(WPB * 32)
k_clique_warp(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
              u64 nverts, u64* next, u64 grab, u64* count) {
    __shared__ u32 sA[WPB][64];
    __shared__ __align__(8) u64 sR[WPB][64];
    __shared__ u32 sEnd[WPB][32];
    __shared__ __align__(8) u64 sOff[WPB][32];
    __shared__ u32 sRow[WPB][32];
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
            R[lane] = 0;
            R[lane + 32] = 0;
            __syncwarp();
            const u32 hl = g2m_hlog(d);
            g2m_hmap_build(sHK[w], sHV[w], hl, A, d, lane, 32);
            build_rows(off, nbr, A, d, 0, R, 1, sEnd[w], sOff[w], sRow[w], sHK[w], sHV[w], hl);
            if (d > 32) build_rows(off, nbr, A, d, 32, R, 1, sEnd[w], sOff[w], sRow[w], sHK[w], sHV[w], hl);
            for (u32 i = lane; i < d; i += 32) acc += Chain1<K - 2>::run(R, R[i]);
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

// ---------------------------------------------------------------------------
// CTA tier: 64 < d <= 64*W, one CTA of NW warps per source vertex, W-word
// rows with an odd stride. Each warp takes rows i; the candidates j of R_i
// are compacted (CH words at a time) into a shared list so every lane gets
// a candidate. k=5: t2 = R_i & R_j stays in the lane's registers when small;
// large ones are compacted again and shared by the whole warp.
// ---------------------------------------------------------------------------
template <int K, int W, int NW>
__global__ void __launch_bounds__(NW * 32)
k_clique_cta(const u64* __restrict__ off, const u32* __restrict__ nbr, const u32* __restrict__ verts,
             u64 nverts, u64* next, u64* count) {
    constexpr u32 CH = 4;             // words compacted per round (<= 256 candidates)
    extern __shared__ __align__(16) u64 smem[];
    // layout: R [64W x (W+1)] u64 | T [NW x (W+1)] u64 | A [64W] u32 |
    //         hash keys, vals [128W] u32 each | per-warp: end[32] row[32] off[32 u64] L1[256] L2[256]
    u64* R = smem;
    u64* T = R + 64 * W * (W + 1);
    u32* A = (u32*)(T + NW * (W + 1));
    u32* HK = A + 64 * W;
    u32* HV = HK + 128 * W;
    u32* base = HV + 128 * W;
    const u32 lane = g2m_lane();
    const u32 w = threadIdx.x >> 5;
    u32* fl_end = base + w * 640;
    u32* fl_row = fl_end + 32;
    u64* fl_off = (u64*)(fl_end + 64);
    u32* L1 = fl_end + 128;
    u32* L2 = L1 + 256;
    u64* t2s = T + w * (W + 1);
    __shared__ u64 s_u;
    u64 acc = 0;
    for (;;) {
        if (threadIdx.x == 0) s_u = atomicAdd(next, 1ull);
        __syncthreads();
        const u64 t = s_u;
        if (t >= nverts) break;
        const u32 u = __ldg(verts + t);
        const u64 b = __ldg(off + u);
        const u32 d = (u32)(__ldg(off + u + 1) - b);
        const u32 Wd = (d + 63) >> 6;
        const u32 Ws = Wd | 1u;          // odd row stride (bank spread)
        for (u32 x = threadIdx.x; x < d; x += NW * 32) A[x] = __ldg(nbr + b + x);
        for (u32 x = threadIdx.x; x < d * Ws; x += NW * 32) R[x] = 0;
        __syncthreads();
        const u32 hl = g2m_hlog(d);
        g2m_hmap_build(HK, HV, hl, A, d, threadIdx.x, NW * 32);
        for (u32 i0 = w * 32; i0 < d; i0 += NW * 32)
            build_rows(off, nbr, A, d, i0, R, Ws, fl_end, fl_off, fl_row, HK, HV, hl);
        __syncthreads();
        for (u32 i = w; i < d; i += NW) {
            const u64* Ri = R + (u64)i * Ws;
            const u64 myw = lane < Wd ? Ri[lane] : 0ull;
            if (K == 3) {
                acc += (u64)__popcll(myw);
                continue;
            }
            const u32 nzw = __ballot_sync(G2M_FULL, myw != 0ull);
            if (!nzw) continue;
            for (u32 c0 = 0; c0 < Wd; c0 += CH) {
                if (!((nzw >> c0) & ((1u << CH) - 1u))) continue;
                const u32 n1 = compact_bits(Ri, c0, min(c0 + CH, Wd), L1);
                for (u32 e0 = 0; e0 < n1; e0 += 32) {
                    const u32 e = e0 + lane;
                    const bool isj = e < n1;
                    const u32 j = isj ? L1[e] : 0u;
                    const u64* Rj = R + (u64)j * Ws;
                    if (K == 4) {
                        if (isj) {
                            u32 m = nzw;
                            while (m) {
                                const int q = __ffs(m) - 1;
                                m &= m - 1;
                                acc += (u64)__popcll(Ri[q] & Rj[q]);
                            }
                        }
                    } else {   // K == 5
                        u64 t2[W];
                        u32 c = 0;
#pragma unroll
                        for (int r = 0; r < W; ++r) {
                            t2[r] = (isj && r < (int)Wd) ? (Ri[r] & Rj[r]) : 0ull;
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
#pragma unroll
                                    for (int r2 = 0; r2 < W; ++r2)
                                        if (t2[r2]) acc += (u64)__popcll(t2[r2] & Rl[r2]);
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
                                    const u64* Rl = R + (u64)L2[f] * Ws;
                                    u32 m = nz2;
                                    while (m) {
                                        const int q3 = __ffs(m) - 1;
                                        m &= m - 1;
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
        __syncthreads();
    }
    acc = g2m_wsum(acc);
    if (lane == 0 && acc) g2m_add128(count, acc, 0);
}

// Bucket the sources of this partition by local-graph size class.
// class 0: d < K-1 (no clique), 1: d <= 64 (warp), 2..5: W = 2,4,8,16 (CTA),
// 6: d > 1024 (generic kernel).
__global__ void k_clique_bucket(const u64* off, u64 nv, int kmin1, u64 rr_chunk, u32 parts, u32 part,
                                u32* lists, u64 list_stride, u64* sizes) {
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < nv; v += (u64)gridDim.x * blockDim.x) {
        if (rr_chunk && ((v / rr_chunk) % parts) != part) continue;
        const u64 d = off[v + 1] - off[v];
        int c;
        if (d < (u64)kmin1) continue;
        if (d <= 64) c = 1;
        else if (d <= 128) c = 2;
        else if (d <= 256) c = 3;
        else if (d <= 512) c = 4;
        else if (d <= 1024) c = 5;
        else c = 6;
        const u64 slot = atomicAdd(sizes + c, 1ull);
        lists[(u64)c * list_stride + slot] = (u32)v;
    }
}

}  // namespace g2m_clique
