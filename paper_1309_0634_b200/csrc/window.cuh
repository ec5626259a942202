// window.cuh -- K4 (per-partition incremental window update), K5 (combine
// of split hot keys), store growth and the per-batch result emission.
//
// Reference semantics (engine.py:185-250): a group with
// prior (fill f0, next_pos p0, sum S0) receiving k values a_0..a_{k-1} in
// arrival order ends with
//     fill = min(f0+k, W),  next_pos = (p0 + max(f0+k-W, 0)) mod W,
//     sum  = sum of the last `fill` values of  old-window ++ run,
// and only a_j with j >= k-W are stored, at ring slot (p0+f0+j) mod W.
//
// B200 formulation: slot (p0+f0+j) mod W held, at batch start, the old
// timeline position q = (f0+j) mod W, which is live iff q < f0.  So every
// stored value is an independent exchange
//     old = live ? ring[slot] : 0;  ring[slot] = a_j;  delta += a_j - old
// and sum = S0 + sum(delta): integer arithmetic, bit-exact in any order,
// which is what lets split hot keys be updated by several CTAs at once.
#pragma once

#include "common.cuh"

namespace ss {

constexpr int kIngestThreads = 1024;
constexpr int kILP = 8;                      // stored values in flight per thread
constexpr int kMemberChunk = 2048;          // members staged per CTA round
constexpr int kMPT = kMemberChunk / kIngestThreads;
constexpr size_t kIngestSmem = (size_t)kMemberChunk * (8 + 8 + 4 * 8) + 16;

struct IngestArgs {
    const int32_t* order;       // partition lists, concatenated   [G]
    const int32_t* offsets;     // CSR offsets                     [P+1]
    int32_t* gcnt;              // group counts of this sub-batch  [G] (reset after use)
    const int32_t* gstart;      // run start of each group in the placed sub-batch
    const int32_t* vals;        // placed (group-sorted, arrival-stable) values
    int32_t* fill;
    int32_t* next_pos;
    long long* wsum;
    int32_t* mn;
    int32_t* mx;
    const int64_t* off;         // ring region of each group
    int32_t* ring;
    int64_t W;
    int minmax;                 // maintain MIN/MAX
    const int32_t* split_of;    // >= 0: group executed as split shares (K5 finalises)
    const int32_t* share_off;   // [P+1] split shares of each partition
    const int32_t* share_grp;   // split-group index per share
    const long long* share_lo;  // run slice [k*lo/den, k*hi/den) of the share
    const long long* share_hi;
    const int32_t* split_g;     // split-group index -> group
    const long long* split_den; // split-group index -> planned count
    const int* n_split;
    unsigned long long* split_delta;   // per split-group delta (K5)
    int32_t* split_min;
    int32_t* split_max;
    int32_t* rescan;            // groups whose MIN/MAX need a rescan
    unsigned* n_rescan;
    unsigned long long* part_ns;       // per-partition (CTA) time, ns
    const unsigned long long* bad;
};

// segmented (contiguous-lane segments) suffix reduction; the first lane
// of each segment ends with the segment total.
__device__ __forceinline__ long long seg_sum(long long v, unsigned seg_end) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long n = __shfl_down_sync(SS_FULL, v, o);
        if (lane + o <= seg_end) v += n;
    }
    return v;
}

__global__ void __launch_bounds__(kIngestThreads)
k_ingest(IngestArgs a) {
    extern __shared__ __align__(16) unsigned char ingest_sm[];
    int64_t* m_off = (int64_t*)ingest_sm;
    unsigned long long* m_delta = (unsigned long long*)(m_off + kMemberChunk);
    int32_t* m_g = (int32_t*)(m_delta + kMemberChunk);
    int32_t* m_scan = m_g + kMemberChunk;            // kMemberChunk + 1
    int32_t* m_start = m_scan + kMemberChunk + 4;
    int32_t* m_q0 = m_start + kMemberChunk;
    int32_t* m_s0 = m_q0 + kMemberChunk;
    int32_t* m_f0 = m_s0 + kMemberChunk;
    int32_t* m_min = m_f0 + kMemberChunk;
    int32_t* m_max = m_min + kMemberChunk;
    __shared__ int32_t sh_red[33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    uint64_t t0 = 0;
    if (threadIdx.x == 0) t0 = globaltimer();
    const int p = blockIdx.x;
    const int lo = a.offsets[p], hi = a.offsets[p + 1];
    const int s_lo = a.share_off ? a.share_off[p] : 0;
    const int s_hi = a.share_off ? a.share_off[p + 1] : 0;
    const int n_items = (hi - lo) + (s_hi - s_lo);   // members, then split shares
    const int W = (int)a.W;
    const unsigned lane = lane_id();

    for (int c0 = 0; c0 < n_items; c0 += kMemberChunk) {
        const int m = min(kMemberChunk, n_items - c0);
        int32_t wk[kMPT];
        int32_t tsum = 0;
#pragma unroll
        for (int q = 0; q < kMPT; ++q) {
            const int i = threadIdx.x * kMPT + q;
            wk[q] = 0;
            if (i < m) {
                const int it = c0 + i;
                int g, k, kb = 0;   // kb: first run index of this item
                if (it < hi - lo) {
                    g = a.order[lo + it];
                    k = (a.split_of && a.split_of[g] >= 0) ? 0 : a.gcnt[g];
                } else {
                    const int sh = s_lo + (it - (hi - lo));
                    const int sg = a.share_grp[sh];
                    g = a.split_g[sg];
                    const int kt = a.gcnt[g];
                    const long long den = a.split_den[sg];
                    kb = (int)((long long)kt * a.share_lo[sh] / den);
                    const int ke = (int)((long long)kt * a.share_hi[sh] / den);
                    // the slice is [kb, ke) of a run of kt; stored part is j >= kt - W
                    const int w0 = max(kb, kt - W);
                    k = max(0, ke - w0);
                    kb = w0;
                    if (k > 0) {
                        const int f0 = a.fill[g];
                        m_g[i] = -1 - sg;          // marks a share
                        m_start[i] = a.gstart[g] + kb;
                        m_q0[i] = (int)(((int64_t)f0 + kb) % W);
                        m_s0[i] = (int)(((int64_t)a.next_pos[g] + f0 + kb) % W);
                        m_f0[i] = f0;
                        m_off[i] = a.off[g];
                        m_delta[i] = 0;
                        m_min[i] = 0x7fffffff;
                        m_max[i] = (int32_t)0x80000000;
                        wk[q] = k;
                    }
                    k = -1;   // handled
                }
                if (k > 0) {
                    const int f0 = a.fill[g];
                    const int w0 = max(0, k - W);
                    m_g[i] = g;
                    m_start[i] = a.gstart[g] + w0;
                    m_q0[i] = (int)(((int64_t)f0 + w0) % W);
                    m_s0[i] = (int)(((int64_t)a.next_pos[g] + f0 + w0) % W);
                    m_f0[i] = f0;
                    m_off[i] = a.off[g];
                    m_delta[i] = 0;
                    m_min[i] = 0x7fffffff;
                    m_max[i] = (int32_t)0x80000000;
                    wk[q] = k - w0;
                } else if (k == 0) {
                    m_g[i] = 0x7fffffff;   // nothing to do
                }
            }
            tsum += wk[q];
        }
        int32_t total;
        int32_t ex = block_excl_scan(tsum, sh_red, &total);
#pragma unroll
        for (int q = 0; q < kMPT; ++q) {
            const int i = threadIdx.x * kMPT + q;
            if (i < m) m_scan[i] = ex;
            ex += wk[q];
        }
        if (threadIdx.x == 0) m_scan[m] = total;
        __syncthreads();

        // ---- exchange: kILP stored values per thread per round, all loads
        // issued before any store (distinct slots within a round) -----------
        for (int base = 0; base < total; base += kIngestThreads * kILP) {
            int mi[kILP];
            int32_t v[kILP], old[kILP];
            int64_t cell[kILP];
#pragma unroll
            for (int u = 0; u < kILP; ++u) {
                const int t = base + u * kIngestThreads + threadIdx.x;
                mi[u] = -1;
                if (t < total) {
                    // last member with m_scan[l] <= t; fixed trip count so the
                    // kILP searches interleave
                    int l = 0;
#pragma unroll
                    for (int step = kMemberChunk / 2; step >= 1; step >>= 1) {
                        const int c = l + step;
                        if (c < m && m_scan[c] <= t) l = c;
                    }
                    mi[u] = l;
                }
            }
#pragma unroll
            for (int u = 0; u < kILP; ++u) {
                if (mi[u] >= 0) {
                    const int t = base + u * kIngestThreads + threadIdx.x;
                    const int rr = t - m_scan[mi[u]];
                    v[u] = a.vals[m_start[mi[u]] + rr];
                    int sl = m_s0[mi[u]] + rr;
                    if (sl >= W) sl -= W;
                    cell[u] = m_off[mi[u]] + sl;
                }
            }
#pragma unroll
            for (int u = 0; u < kILP; ++u) {
                old[u] = 0;
                if (mi[u] >= 0) {
                    const int t = base + u * kIngestThreads + threadIdx.x;
                    int q = m_q0[mi[u]] + (t - m_scan[mi[u]]);
                    if (q >= W) q -= W;
                    if (q < m_f0[mi[u]]) old[u] = a.ring[cell[u]];
                }
            }
#pragma unroll
            for (int u = 0; u < kILP; ++u)
                if (mi[u] >= 0) a.ring[cell[u]] = v[u];
#pragma unroll
            for (int u = 0; u < kILP; ++u) {
                const bool valid = mi[u] >= 0;
                const long long d = valid ? (long long)v[u] - (long long)old[u] : 0;
                const unsigned key = valid ? (unsigned)mi[u] : 0xffffffffu;
                const unsigned peers = __match_any_sync(SS_FULL, key);
                const unsigned seg_end = 31u - __clz(peers);
                const long long tot = seg_sum(d, seg_end);
                const bool leader = valid && lane == (unsigned)(__ffs(peers) - 1);
                if (leader) atomicAdd(&m_delta[mi[u]], (unsigned long long)tot);
                if (a.minmax && valid) {
                    const int32_t mnv = __reduce_min_sync(peers, v[u]);
                    const int32_t mxv = __reduce_max_sync(peers, v[u]);
                    if (leader) {
                        atomicMin(&m_min[mi[u]], mnv);
                        atomicMax(&m_max[mi[u]], mxv);
                    }
                }
            }
        }
        __syncthreads();

        // ---- finalise each member's state (shares go to K5) -----------------
        for (int i = threadIdx.x; i < m; i += kIngestThreads) {
            const int g = m_g[i];
            if (g == 0x7fffffff) continue;
            if (m_scan[i + 1] == m_scan[i]) continue;     // no stored value
            if (g < 0) {
                const int sg = -1 - g;
                atomicAdd(&a.split_delta[sg], m_delta[i]);
                if (a.minmax) {
                    atomicMin(&a.split_min[sg], m_min[i]);
                    atomicMax(&a.split_max[sg], m_max[i]);
                }
                continue;
            }
            const int k = a.gcnt[g];
            const int f0 = m_f0[i];
            const int64_t tot = (int64_t)f0 + k;
            const int p0 = a.next_pos[g];
            a.fill[g] = (int32_t)min64(tot, W);
            a.next_pos[g] = (int32_t)((p0 + max64(tot - W, 0)) % W);
            a.wsum[g] = a.wsum[g] + (long long)m_delta[i];
            if (a.minmax) {
                if (tot <= W || k >= W) {
                    // no old value survives alongside an eviction: monotone update
                    const bool keep_old = (f0 > 0) && (k < W);
                    a.mn[g] = keep_old ? min(a.mn[g], m_min[i]) : m_min[i];
                    a.mx[g] = keep_old ? max(a.mx[g], m_max[i]) : m_max[i];
                } else {
                    a.rescan[atomicAdd(a.n_rescan, 1u)] = g;
                }
            }
            a.gcnt[g] = 0;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && a.part_ns) atomicAdd(&a.part_ns[p], (unsigned long long)(globaltimer() - t0));
}

// K5: finalise split groups after all their shares ran.  One thread each.
__global__ void k_split_finalize(IngestArgs a) {
    const int sg = blockIdx.x * blockDim.x + threadIdx.x;
    if (sg >= *a.n_split || *a.bad != (unsigned long long)kNoBad) return;
    const int g = a.split_g[sg];
    const int k = a.gcnt[g];
    if (k > 0) {
        const int W = (int)a.W;
        const int f0 = a.fill[g];
        const int64_t tot = (int64_t)f0 + k;
        const int p0 = a.next_pos[g];
        a.fill[g] = (int32_t)min64(tot, W);
        a.next_pos[g] = (int32_t)((p0 + max64(tot - W, 0)) % W);
        a.wsum[g] = a.wsum[g] + (long long)a.split_delta[sg];
        if (a.minmax) {
            if (tot <= W || k >= W) {
                const bool keep_old = (f0 > 0) && (k < W);
                a.mn[g] = keep_old ? min(a.mn[g], a.split_min[sg]) : a.split_min[sg];
                a.mx[g] = keep_old ? max(a.mx[g], a.split_max[sg]) : a.split_max[sg];
            } else {
                a.rescan[atomicAdd(a.n_rescan, 1u)] = g;
            }
        }
        a.gcnt[g] = 0;
    }
    a.split_delta[sg] = 0;
    a.split_min[sg] = 0x7fffffff;
    a.split_max[sg] = (int32_t)0x80000000;
}

// MIN/MAX of a full window after a partial eviction: every ring slot is
// live, so the slot order does not matter.  One CTA per listed group.
__global__ void __launch_bounds__(256)
k_minmax_rescan(const int32_t* __restrict__ rescan, const unsigned* __restrict__ n_rescan,
                const int32_t* __restrict__ ring, const int64_t* __restrict__ off, int64_t W,
                int32_t* __restrict__ mn, int32_t* __restrict__ mx) {
    __shared__ int32_t s_mn[8], s_mx[8];
    const unsigned n = *n_rescan;
    for (unsigned i = blockIdx.x; i < n; i += gridDim.x) {
        const int g = rescan[i];
        const int32_t* r = ring + off[g];
        int32_t lo = 0x7fffffff, hi = (int32_t)0x80000000;
        for (int64_t j = threadIdx.x; j < W; j += blockDim.x) {
            const int32_t v = r[j];
            lo = min(lo, v);
            hi = max(hi, v);
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        if (lane_id() == 0) { s_mn[warp_id()] = lo; s_mx[warp_id()] = hi; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; ++w) { lo = min(lo, s_mn[w]); hi = max(hi, s_mx[w]); }
            mn[g] = lo;
            mx[g] = hi;
        }
        __syncthreads();
    }
}

// Occupancy-proportional store: grow the ring region of every group whose
// window will hold more values than its capacity (capacity doubles up to
// W; a window that has not reached W is linear, next_pos == 0, so growth
// copies `fill` values).  One warp per group.
__global__ void __launch_bounds__(256)
k_reserve(const int32_t* __restrict__ gcnt, uint32_t G, int64_t W, const int32_t* __restrict__ fill,
          int64_t* __restrict__ off, int32_t* __restrict__ cap, int32_t* __restrict__ ring,
          unsigned long long* __restrict__ pool_top, unsigned long long pool_cap,
          int* __restrict__ oom, const unsigned long long* __restrict__ bad) {
    if (*bad != (unsigned long long)kNoBad) return;
    const unsigned lane = lane_id();
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t g0 = (blockIdx.x * (blockDim.x >> 5) + warp_id()) * 32; g0 < G; g0 += nwarps * 32) {
        const uint32_t g = g0 + lane;
        int64_t need = 0, ncap = 0, noff = 0;
        int c = 0, f = 0;
        if (g < G) {
            const int k = gcnt[g];
            if (k) {
                f = fill[g];
                c = cap[g];
                need = min64((int64_t)f + k, W);
                if (need > c) {
                    ncap = min64(W, max64(max64(need, 2 * (int64_t)c), 16));
                }
            }
        }
        // warp-aggregated reservation
        const int64_t incl = warp_incl_scan(ncap);
        const int64_t wtot = __shfl_sync(SS_FULL, incl, 31);
        unsigned long long base = 0;
        if (lane == 31 && wtot) base = atomicAdd(pool_top, (unsigned long long)wtot);
        base = __shfl_sync(SS_FULL, base, 31);
        if (ncap) {
            noff = (int64_t)base + incl - ncap;
            if ((unsigned long long)(noff + ncap) > pool_cap) {
                *oom = 1;
                ncap = 0;
            }
        }
        // copy live prefix (linear while filling), one group at a time per warp
        unsigned todo = __ballot_sync(SS_FULL, ncap != 0);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t so = __shfl_sync(SS_FULL, off[g0 + src < G ? g0 + src : 0], src);
            const int64_t doff = __shfl_sync(SS_FULL, noff, src);
            const int ff = __shfl_sync(SS_FULL, f, src);
            for (int j = lane; j < ff; j += 32) ring[doff + j] = ring[so + j];
        }
        __syncwarp();
        if (ncap) {
            off[g] = noff;
            cap[g] = (int32_t)ncap;
        }
    }
}

// Per-batch result emission: every group touched by the batch gets a row
// (group, COUNT, SUM, AVG, MIN, MAX); AVG is the correctly rounded double
// quotient.  Also clears the batch counts for the next batch.
__global__ void __launch_bounds__(256)
k_emit(int32_t* __restrict__ gcount, uint32_t G, const int32_t* __restrict__ fill,
       const long long* __restrict__ wsum, const int32_t* __restrict__ mn, const int32_t* __restrict__ mx,
       int minmax, unsigned* __restrict__ n_res, int32_t* __restrict__ r_g, int32_t* __restrict__ r_cnt,
       long long* __restrict__ r_sum, double* __restrict__ r_avg, int32_t* __restrict__ r_mn,
       int32_t* __restrict__ r_mx, const unsigned long long* __restrict__ bad) {
    if (*bad != (unsigned long long)kNoBad) return;
    const unsigned lane = lane_id();
    for (uint32_t g0 = blockIdx.x * blockDim.x; g0 < G; g0 += gridDim.x * blockDim.x) {
        const uint32_t g = g0 + threadIdx.x;
        const bool t = (g < G) && gcount[g] != 0;
        const unsigned bal = __ballot_sync(SS_FULL, t);
        unsigned base = 0;
        if (lane == 0 && bal) base = atomicAdd(n_res, (unsigned)__popc(bal));
        base = __shfl_sync(SS_FULL, base, 0);
        if (t) {
            const unsigned slot = base + __popc(bal & lanemask_lt());
            const int32_t c = fill[g];
            const long long s = wsum[g];
            r_g[slot] = (int32_t)g;
            r_cnt[slot] = c;
            r_sum[slot] = s;
            r_avg[slot] = c ? __ll2double_rn(s) / (double)c : 0.0;
            if (minmax) {
                r_mn[slot] = mn[g];
                r_mx[slot] = mx[g];
            }
            gcount[g] = 0;
        }
    }
}

}  // namespace ss
