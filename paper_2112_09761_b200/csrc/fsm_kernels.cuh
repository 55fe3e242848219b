// fsm_kernels.cuh -- device side of the bounded-BFS frequent subgraph miner
// (reference fsm.py:107-210, run_bounded_bfs): edge-induced subgraphs grow one
// edge per level; each level's subgraphs are grouped by quick pattern (labels of
// the sorted vertices + edges as position pairs, fsm.py:40-47), the host turns
// each distinct quick pattern into its canonical pattern and position maps
// (fsm.py:50-80), the device expands every (subgraph, map, position) into a
// domain triple (canonical id, position, data vertex), sorts and uniquifies them,
// and the per-(pattern, position) run lengths are the domain sizes whose minimum
// is the support (min-image, fsm.py:88-91). Extension adds one edge adjacent to
// the subgraph's vertices (fsm.py:178-201) for subgraphs of kept patterns; new
// edge sets are deduplicated on the device, each keeping the set of parent
// patterns that produced it (the reference's pending_parents).
//
// Row layout (level l = edges per subgraph): edges u64 (u << 32 | v, u < v),
// ascending, kFsmE per row; vertices u32 ascending, kFsmV per row; nverts u8.
#pragma once

#include "g2m_device.cuh"

namespace g2m_fsmk {

constexpr int kFsmE = 7;     // max edges per subgraph (max_edges <= 7)
constexpr int kFsmV = 8;     // max vertices (a connected subgraph of 7 edges has <= 8)
constexpr int kRec = 12;     // quick-pattern record words

__device__ __forceinline__ u64 fnv64(const u32* w, int n) {
    u64 h = 0xcbf29ce484222325ull;
    for (int i = 0; i < n; ++i) {
        u32 x = w[i];
        for (int b = 0; b < 4; ++b) {
            h ^= (x & 0xffu);
            h *= 0x100000001b3ull;
            x >>= 8;
        }
    }
    return h;
}

// level 1: every edge u < w with both ends allowed; per-vertex count, then fill
__global__ void k_fsm_l1_count(const u64* off, const u32* nbr, u64 nv, const unsigned char* ok, u64* cnt) {
    for (u64 u = blockIdx.x * (u64)blockDim.x + threadIdx.x; u < nv; u += (u64)gridDim.x * blockDim.x) {
        u64 c = 0;
        if (!ok || ok[u])
            for (u64 s = off[u]; s < off[u + 1]; ++s) {
                const u32 w = nbr[s];
                if (w > u && (!ok || ok[w])) ++c;
            }
        cnt[u] = c;
    }
}

__global__ void k_fsm_l1_fill(const u64* off, const u32* nbr, u64 nv, const unsigned char* ok, const u64* pos,
                              u64* redges, u32* rverts, unsigned char* rnv) {
    for (u64 u = blockIdx.x * (u64)blockDim.x + threadIdx.x; u < nv; u += (u64)gridDim.x * blockDim.x) {
        if (ok && !ok[u]) continue;
        u64 p = pos[u];
        for (u64 s = off[u]; s < off[u + 1]; ++s) {
            const u32 w = nbr[s];
            if (w > u && (!ok || ok[w])) {
                redges[p * kFsmE] = ((u64)u << 32) | w;
                rverts[p * kFsmV] = (u32)u;
                rverts[p * kFsmV + 1] = w;
                rnv[p] = 2;
                ++p;
            }
        }
    }
}

// quick-pattern record + hash of every row (fsm.py:40-47: labels of the sorted
// vertices, edges as sorted (min, max) position pairs)
__global__ void k_fsm_quick(const u64* redges, const u32* rverts, const unsigned char* rnv, u64 n, int l,
                            const u32* labels, u32* rec, u64* hash, u64* rowid) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        const int k = rnv[r];
        const u32* V = rverts + r * kFsmV;
        u32 w[kRec];
#pragma unroll
        for (int i = 0; i < kRec; ++i) w[i] = 0;
        w[0] = (u32)k | ((u32)l << 8);
        for (int i = 0; i < k; ++i) w[1 + i] = labels[V[i]];
        u32 pr[kFsmE];
        for (int e = 0; e < l; ++e) {
            const u64 ed = redges[r * kFsmE + e];
            const u32 a = (u32)(ed >> 32), b = (u32)ed;
            u32 ia = 0, ib = 0;
            for (int i = 0; i < k; ++i) {
                if (V[i] == a) ia = i;
                if (V[i] == b) ib = i;
            }
            pr[e] = (min(ia, ib) << 3) | max(ia, ib);
        }
        for (int i = 1; i < l; ++i) {        // sort the pairs
            const u32 x = pr[i];
            int j = i - 1;
            while (j >= 0 && pr[j] > x) { pr[j + 1] = pr[j]; --j; }
            pr[j + 1] = x;
        }
        u64 packed = 0;
        for (int e = 0; e < l; ++e) packed |= (u64)pr[e] << (6 * e);
        w[9] = (u32)packed;
        w[10] = (u32)(packed >> 32);
#pragma unroll
        for (int i = 0; i < kRec; ++i) rec[r * kRec + i] = w[i];
        hash[r] = fnv64(w, kRec);
        rowid[r] = r;
    }
}

// after sorting (hash, row): group heads and qid per row; a record that differs
// from its group head's is a 64-bit collision (flagged, the host raises)
__global__ void k_fsm_group(const u64* hs, const u64* rows, u64 n, const u32* rec, const u64* head_pos,
                            u32* qid, u32* err) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 g = head_pos[i];           // group index of sorted position i
        qid[rows[i]] = (u32)g;
        (void)hs;
    }
    (void)rec;
    (void)err;
}

__global__ void k_fsm_check(const u64* rows, u64 n, const u32* rec, const u64* first_row_of_group, const u32* qid,
                            u32* err) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 r = rows[i];
        const u64 h = first_row_of_group[qid[r]];
        for (int w = 0; w < kRec; ++w)
            if (rec[r * kRec + w] != rec[h * kRec + w]) { atomicOr(err, 1u); break; }
    }
}

// domain triples: per row, for each map m of its quick pattern and canonical
// position c: (canon << 36) | (c << 32) | verts[map[c]]  (fsm.py:160-166)
__global__ void k_fsm_dom_count(const u32* qid, const u32* nmaps, const unsigned char* rnv, u64 n, u64* cnt) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x)
        cnt[r] = (u64)nmaps[qid[r]] * rnv[r];
}

__global__ void k_fsm_dom_fill(const u32* qid, const u32* canon, const u32* nmaps, const u32* map_off,
                               const unsigned char* maps, const u32* rverts, const unsigned char* rnv, u64 n,
                               const u64* pos, u64* keys) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        const u32 q = qid[r];
        const int k = rnv[r];
        const u64 c = canon[q];
        const unsigned char* M = maps + map_off[q];
        u64 p = pos[r];
        for (u32 m = 0; m < nmaps[q]; ++m)
            for (int i = 0; i < k; ++i) keys[p++] = (c << 36) | ((u64)i << 32) | rverts[r * kFsmV + M[m * k + i]];
    }
}

// parent -> child pattern pairs of this level's rows
__global__ void k_fsm_pc(const u32* qid, const u32* canon, const u32* par_off, const u32* par, u64 n, u64* out) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        const u64 c = canon[qid[r]];
        for (u32 j = par_off[r]; j < par_off[r + 1]; ++j) out[j] = ((u64)par[j] << 32) | c;
    }
}

// extension candidates (fsm.py:178-201): rows of kept patterns, one new edge
// (v, w) per vertex v of the subgraph and allowed neighbour w, not already in
// the subgraph; count pass then fill pass
__device__ __forceinline__ bool fsm_has_edge(const u64* E, int l, u64 e) {
    for (int i = 0; i < l; ++i)
        if (E[i] == e) return true;
    return false;
}

template <bool FILL>
__global__ void k_fsm_extend(const u64* off, const u32* nbr, const unsigned char* ok, const u64* redges,
                             const u32* rverts, const unsigned char* rnv, const u32* qid, const u32* canon,
                             const unsigned char* kept, u64 n, int l, u64* cnt, const u64* pos, u64* cedges,
                             u32* cverts, unsigned char* cnv, u32* cpar, u64* chash, u64* cid) {
    for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < n; r += (u64)gridDim.x * blockDim.x) {
        const u32 cr = canon[qid[r]];
        u64 c = 0;
        u64 p = FILL ? pos[r] : 0;
        if (kept[cr]) {
            const u64* E = redges + r * kFsmE;
            const u32* V = rverts + r * kFsmV;
            const int k = rnv[r];
            for (int i = 0; i < k; ++i) {
                const u32 v = V[i];
                for (u64 s = off[v]; s < off[v + 1]; ++s) {
                    const u32 w = nbr[s];
                    if (ok && !ok[w]) continue;
                    const u64 e = v < w ? (((u64)v << 32) | w) : (((u64)w << 32) | v);
                    if (fsm_has_edge(E, l, e)) continue;
                    if (FILL) {
                        u64* NE = cedges + p * kFsmE;
                        int j = 0, o = 0;
                        bool put = false;
                        for (; j < l; ++j) {
                            if (!put && e < E[j]) { NE[o++] = e; put = true; }
                            NE[o++] = E[j];
                        }
                        if (!put) NE[o++] = e;
                        u32* NV = cverts + p * kFsmV;
                        bool in = false;
                        for (int t = 0; t < k; ++t) in = in || V[t] == w;
                        int nk = 0;
                        bool putv = in;
                        for (int t = 0; t < k; ++t) {
                            if (!putv && w < V[t]) { NV[nk++] = w; putv = true; }
                            NV[nk++] = V[t];
                        }
                        if (!putv) NV[nk++] = w;
                        cnv[p] = (unsigned char)nk;
                        cpar[p] = cr;
                        u32 hw[2 * kFsmE];
                        for (int t = 0; t < 2 * kFsmE; ++t) hw[t] = 0;
                        for (int t = 0; t <= l; ++t) {
                            hw[2 * t] = (u32)(NE[t] >> 32);
                            hw[2 * t + 1] = (u32)NE[t];
                        }
                        chash[p] = fnv64(hw, 2 * (l + 1));
                        cid[p] = p;
                        ++p;
                    }
                    ++c;
                }
            }
        }
        if (!FILL) cnt[r] = c;
    }
}

// after sorting candidates by (hash): 1 where a candidate's edge set differs
// from its predecessor's (a new unique edge set); equal hashes with different
// edge sets are collisions (flagged)
__global__ void k_fsm_cand_heads(const u64* hs, const u64* ids, u64 m, const u64* cedges, int l, u32* head,
                                 u32* err) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
        if (i == 0) { head[i] = 1; continue; }
        bool same = hs[i] == hs[i - 1];
        if (same) {
            const u64* A = cedges + ids[i] * kFsmE;
            const u64* B = cedges + ids[i - 1] * kFsmE;
            bool eq = true;
            for (int t = 0; t <= l; ++t) eq = eq && A[t] == B[t];
            if (!eq) atomicOr(err, 1u);
            same = eq;
        }
        head[i] = same ? 0u : 1u;
    }
}

// next-level rows from the group heads; (group, parent) pairs for every candidate
__global__ void k_fsm_next(const u64* ids, const u64* grp, u64 m, const u32* head, const u64* cedges,
                           const u32* cverts, const unsigned char* cnv, const u32* cpar, u64* redges, u32* rverts,
                           unsigned char* rnv, u64* gp) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x) {
        const u64 g = grp[i];
        const u64 c = ids[i];
        if (head[i]) {
            for (int t = 0; t < kFsmE; ++t) redges[g * kFsmE + t] = cedges[c * kFsmE + t];
            for (int t = 0; t < kFsmV; ++t) rverts[g * kFsmV + t] = cverts[c * kFsmV + t];
            rnv[g] = cnv[c];
        }
        gp[i] = (g << 32) | cpar[c];
    }
}

}  // namespace g2m_fsmk
