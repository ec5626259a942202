// split.cuh -- hot-key splitting across blocks with a final combine.
//
// New mechanism (not in the paper nor the reference package): the
// reference Assignment is a bijection group -> thread (partition.py:72-87),
// so the best any reference policy can reach is max/mean = P x (hottest
// group's share) -- 56.85 at Zipf s=1.5, P=148.
//
// Split mode plans, from batch t's OWN counts (on the side stream while
// batch t's placement runs; the window update waits for it), how batch t
// executes:
//   1. hot groups: min(count, W) > mean/2 (so at most 2P of them);
//      everything else is cold and stays whole on its partition;
//   2. the configured policy moves COLD groups between partitions on the
//      cold-only loads (same device loop as the reference policies); those
//      moves keep the reference's one-batch delay (in force from t+1);
//   3. the hot groups' tuples are water-filled onto the least loaded
//      partitions: find the level L with sum_p max(0, L - load_p) >= hot
//      tuples, lay partition capacities and hot groups' runs on one axis
//      and cut -- each overlap is a share (group, partition, run slice).
// Loads are in values to store, min(count, W) per group: a hot group's
// tuples before its last W are never stored, so planning on tuple counts
// left partitions holding those slices idle (C3, W = 1e6 and a top group
// of ~6M tuples per batch: measured partition time max/mean 1.7 with a
// tuple-balanced plan).  A share covers the slice [s*lo/den, s*hi/den) of
// its group's s = min(count, W) stored values (den = the planned s), so
// the shares tile the stored range exactly.
// Every share does independent window exchanges (window.cuh) and adds its
// delta to the group's batch accumulator; K5 (k_finalize) folds them once
// per batch.
#pragma once

#include "common.cuh"

namespace ss {

struct SplitPlan {
    int* n_split;          // device scalar
    int* n_share;          // device scalar
    int32_t* split_of;     // [G] split index or -1
    int32_t* split_g;      // [maxS]
    long long* split_den;  // [maxS] planned count
    int32_t* part_soff;    // [P+1] shares of each partition (axis order)
    int32_t* share_grp;    // [maxSh] split index
    long long* share_lo;   // [maxSh] numerators
    long long* share_hi;
};

struct SplitScratch {
    int32_t* hot_g;        // [maxS] unsorted hot list
    int* n_hot;
    unsigned long long* base;   // [P] cold loads
    uint8_t* hot_flag;     // [G]
    unsigned long long* n_stored;   // sum of min(count, W) of the batch
};

// Phase 0: the batch's values to store, sum of min(count, W) (the hot
// threshold is half the mean block load in these units)
__global__ void __launch_bounds__(256)
k_split_sum(const int32_t* __restrict__ gcount, uint32_t G, int64_t W, unsigned long long* __restrict__ n_stored,
            const unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    if (*bad != (unsigned long long)kNoBad) return;
    unsigned long long s = 0;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x)
        s += (unsigned long long)min64(gcount[g], W);
    // one atomic per CTA (one per warp serialised ~31K same-address
    // atomics at 1M groups)
    __shared__ unsigned long long sh[8];
    s = warp_sum(s);
    if (lane_id() == 0) sh[warp_id()] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += sh[q];
        if (t) atomicAdd(n_stored, t);
    }
}

// Phase 1: hot detection + cold loads.  grid-stride over G; cold loads
// accumulate per CTA in shared memory (P <= 4096) before one flush.
__global__ void __launch_bounds__(256)
k_split_hot(const int32_t* __restrict__ gcount, uint32_t G, const int32_t* __restrict__ pmap,
            const unsigned long long* __restrict__ n_stored, int maxS, SplitScratch sc, int P,
            const unsigned long long* __restrict__ bad, int64_t W) { SS_PDL_ENTRY();
    extern __shared__ uint32_t sh_base[];
    if (*bad != (unsigned long long)kNoBad) return;
    // hot: more values to store than half the mean block load
    const long long hot_min = max(1LL, (long long)(*n_stored / (2ull * (unsigned long long)P)));
    for (int i = threadIdx.x; i < P; i += blockDim.x) sh_base[i] = 0;
    __syncthreads();
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
        const int32_t c = gcount[g];
        uint8_t hot = 0;
        if (min64(c, W) > hot_min) {
            const int slot = atomicAdd(sc.n_hot, 1);
            if (slot < maxS) {
                sc.hot_g[slot] = (int32_t)g;
                hot = 1;
            }
        }
        sc.hot_flag[g] = hot;
        if (c && !hot) atomicAdd(&sh_base[pmap[g]], (uint32_t)min64(c, W));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x)
        if (sh_base[i]) atomicAdd(&sc.base[i], (unsigned long long)sh_base[i]);
}

// Phase 3: water-fill the hot groups onto the loads left by the cold
// moves and write the next plan.  One CTA.
__global__ void __launch_bounds__(1024)
k_split_fill(const int32_t* __restrict__ gcount, const long long* __restrict__ loads, int P, int maxS,
             SplitScratch sc, SplitPlan prev, SplitPlan nx, const unsigned long long* __restrict__ bad, int64_t W) { SS_PDL_ENTRY();
    extern __shared__ long long fsm[];
    long long* hot_c = fsm;                 // [maxS]
    long long* hot_s = hot_c + maxS;        // [maxS + 1] axis starts
    int32_t* hot_g = (int32_t*)(hot_s + maxS + 1);   // [maxS]
    int32_t* cnt = hot_g + maxS;            // [P + 1] shares per partition -> offsets
    __shared__ long long red[33];
    __shared__ long long sh_L;
    __shared__ int sh_n;
    if (*bad != (unsigned long long)kNoBad) return;
    // clear the split marks this buffer held two batches ago
    const int nprev = *prev.n_split;
    for (int i = threadIdx.x; i < nprev; i += blockDim.x) prev.split_of[prev.split_g[i]] = -1;
    const int nh = min(*sc.n_hot, maxS);
    // sort hot groups by (count desc, id asc): rank by counting (nh <= 2P+1)
    for (int i = threadIdx.x; i < nh; i += blockDim.x) {
        const int g = sc.hot_g[i];
        const long long c = min64(gcount[g], W);
        int r = 0;
        for (int j = 0; j < nh; ++j) {
            const int g2 = sc.hot_g[j];
            const long long c2 = min64(gcount[g2], W);
            r += (c2 > c) || (c2 == c && g2 < g);
        }
        hot_g[r] = g;
        hot_c[r] = c;
    }
    __syncthreads();
    // axis starts of the hot runs
    if (threadIdx.x == 0) {
        long long run = 0;
        for (int j = 0; j < nh; ++j) { hot_s[j] = run; run += hot_c[j]; }
        hot_s[nh] = run;
        sh_n = nh;
    }
    __syncthreads();
    const long long T = hot_s[nh];
    // water level: smallest L with sum max(0, L - load) >= T
    long long lo = LLONG_MAX, hi = 0;
    for (int p = threadIdx.x; p < P; p += blockDim.x) { lo = min(lo, loads[p]); hi = max(hi, loads[p]); }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(SS_FULL, lo, o));
        hi = max(hi, __shfl_xor_sync(SS_FULL, hi, o));
    }
    if (lane_id() == 0) { red[warp_id()] = lo; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) lo = min(lo, red[w]);
        sh_L = lo;
    }
    __syncthreads();
    long long a = sh_L, b = sh_L + T + 1;   // f(a) = 0 < T (if T > 0), f(b) >= T
    while (T > 0 && a + 1 < b) {
        const long long mid = a + (b - a) / 2;
        long long f = 0;
        for (int p = threadIdx.x; p < P; p += blockDim.x) f += max(0LL, mid - loads[p]);
        long long tot;
        block_excl_scan(f, red, &tot);
        if (tot >= T) b = mid; else a = mid;
    }
    const long long L = b;
    // partition p covers axis [C_p, C_p + cap_p) clipped to T
    // count shares per partition
    long long carry = 0;
    for (int p0 = 0; p0 < P; p0 += blockDim.x) {
        const int p = p0 + threadIdx.x;
        long long cap = (T > 0 && p < P) ? max(0LL, L - loads[p]) : 0;
        long long tot;
        long long ex = block_excl_scan(cap, red, &tot) + carry;
        if (p < P) {
            long long x0 = min(ex, T), x1 = min(ex + cap, T);
            int k = 0;
            if (x1 > x0) {
                // hot runs overlapping [x0, x1): j0 = last start <= x0, j1 = last start < x1
                int l = 0, r = nh - 1;
                while (l < r) { const int m = (l + r + 1) >> 1; if (hot_s[m] <= x0) l = m; else r = m - 1; }
                const int j0 = l;
                l = j0; r = nh - 1;
                while (l < r) { const int m = (l + r + 1) >> 1; if (hot_s[m] < x1) l = m; else r = m - 1; }
                k = l - j0 + 1;
            }
            cnt[p] = k;
        }
        carry += tot;
    }
    __syncthreads();
    // partition offsets
    {
        int run = 0;
        for (int p0 = 0; p0 < P; p0 += blockDim.x) {
            const int p = p0 + threadIdx.x;
            long long v = (p < P) ? cnt[p] : 0;
            long long tot;
            long long ex = block_excl_scan(v, red, &tot);
            __syncthreads();
            if (p < P) nx.part_soff[p] = run + (int)ex;
            run += (int)tot;
        }
        if (threadIdx.x == 0) { nx.part_soff[P] = run; *nx.n_share = run; *nx.n_split = nh; }
    }
    __syncthreads();
    // emit shares
    carry = 0;
    for (int p0 = 0; p0 < P; p0 += blockDim.x) {
        const int p = p0 + threadIdx.x;
        long long cap = (T > 0 && p < P) ? max(0LL, L - loads[p]) : 0;
        long long tot;
        long long ex = block_excl_scan(cap, red, &tot) + carry;
        if (p < P) {
            const long long x0 = min(ex, T), x1 = min(ex + cap, T);
            if (x1 > x0) {
                int l = 0, r = nh - 1;
                while (l < r) { const int m = (l + r + 1) >> 1; if (hot_s[m] <= x0) l = m; else r = m - 1; }
                int out = nx.part_soff[p];
                for (int j = l; j < nh && hot_s[j] < x1; ++j) {
                    const long long s0 = max(x0, hot_s[j]), s1 = min(x1, hot_s[j + 1]);
                    if (s1 <= s0) continue;
                    nx.share_grp[out] = j;
                    nx.share_lo[out] = s0 - hot_s[j];
                    nx.share_hi[out] = s1 - hot_s[j];
                    ++out;
                }
            }
        }
        carry += tot;
    }
    for (int j = threadIdx.x; j < nh; j += blockDim.x) {
        nx.split_g[j] = hot_g[j];
        nx.split_den[j] = hot_c[j];
        nx.split_of[hot_g[j]] = j;
    }
}

// Loads of the current batch under the current plan (report / max-mean).
__global__ void __launch_bounds__(256)
k_split_loads(const int32_t* __restrict__ gcount, uint32_t G, const int32_t* __restrict__ pmap, int P,
              SplitPlan cur, unsigned long long* __restrict__ loads, const unsigned long long* __restrict__ bad,
              int64_t W) { SS_PDL_ENTRY();
    extern __shared__ uint32_t sh_load[];
    if (*bad != (unsigned long long)kNoBad) return;
    for (int i = threadIdx.x; i < P; i += blockDim.x) sh_load[i] = 0;
    __syncthreads();
    const int nsh = *cur.n_share;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
        const int32_t c = gcount[g];
        if (c && cur.split_of[g] < 0) atomicAdd(&sh_load[pmap[g]], (uint32_t)min64(c, W));
    }
    // shares: one thread per share, find its partition by binary search
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nsh; i += gridDim.x * blockDim.x) {
        int l = 0, r = P - 1;
        while (l < r) { const int m = (l + r + 1) >> 1; if (cur.part_soff[m] <= i) l = m; else r = m - 1; }
        const int j = cur.share_grp[i];
        const long long kt = min64(gcount[cur.split_g[j]], W), den = cur.split_den[j];
        const long long a = kt * cur.share_lo[i] / den, b = kt * cur.share_hi[i] / den;
        if (b > a) atomicAdd(&sh_load[l], (uint32_t)(b - a));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x)
        if (sh_load[i]) atomicAdd(&loads[i], (unsigned long long)sh_load[i]);
}

}  // namespace ss
