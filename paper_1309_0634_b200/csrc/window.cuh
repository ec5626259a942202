// window.cuh -- K4 (per-partition window exchange), K5 (batch finalisation
// and per-batch result emission), store growth and MIN/MAX rescans.
//
// Reference semantics (engine.py:185-250): a group with
// prior (fill f0, next_pos p0, sum S0) receiving k values a_0..a_{k-1} in
// arrival order ends with
//     fill = min(f0+k, W),  next_pos = (p0 + max(f0+k-W, 0)) mod W,
//     sum  = sum of the last `fill` values of  old-window ++ run,
// and only a_j with j >= k-W are stored, at ring slot (p0+f0+j) mod W.
//
// B200 formulation, per BATCH (k = the group's count in the whole batch,
// j = a tuple's rank inside its group over the whole batch): slot
// (p0+f0+j) mod W held, at batch start, the old timeline position
// q = (f0+j) mod W, which is live iff q < f0.  Every stored value is an
// independent exchange
//     old = live ? ring[slot] : 0;  ring[slot] = a_j;  delta += a_j - old
// and sum = S0 + sum(delta) (or sum(a_j) when k >= W: every old value is
// evicted).  Integer arithmetic, bit-exact in any order, so the batch's
// L2-resident sub-batches, the partitions' CTAs and the shares of a split
// hot key all work independently; K5 folds the deltas into the state once
// per batch.  Only min(k, W) values per group and batch are ever stored.
#pragma once

#include "common.cuh"

namespace ss {

constexpr int kIngestThreads = 512;       // 2 CTAs/SM fit, so the balancer's CTA never blocks a partition
constexpr int kILP = 8;                     // stored values in flight per thread
constexpr int kMemberChunk = 2048;          // members staged per CTA round
constexpr int kMPT = kMemberChunk / kIngestThreads;
constexpr size_t kIngestSmem = (size_t)kMemberChunk * (8 + 8 + 4 * 10) + 64;

struct IngestArgs {
    const int32_t* order;       // partition lists, concatenated   [G]
    const int32_t* offsets;     // CSR offsets                     [P+1]
    const int32_t* gcnt;        // kept tuples of each group (a suffix of its batch tuples) [G]
    const int32_t* gcount;      // group counts of the whole batch
    const int32_t* gstart;      // run start of each group in the placed kept set
    const int32_t* vals;        // placed (group-sorted, arrival-stable) values
    const int32_t* fill;        // batch-start state (read only in K4)
    const int32_t* next_pos;
    const int64_t* off;         // ring region of each group
    int32_t* ring;
    long long* bdelta;          // per-group batch delta (K5 folds it)
    int32_t* bmin;              // per-group batch min / max of stored values
    int32_t* bmax;
    int64_t W;
    int minmax;                 // maintain MIN/MAX
    const int32_t* split_of;    // >= 0: group executed as split shares
    const int32_t* share_off;   // [P+1] split shares of each partition
    const int32_t* share_grp;   // split-group index per share
    const long long* share_lo;  // run slice [k*lo/den, k*hi/den) of the share
    const long long* share_hi;
    const int32_t* split_g;     // split-group index -> group
    const long long* split_den; // split-group index -> planned count
    unsigned long long* part_ns;       // per-partition (CTA) time, ns
    unsigned long long* part_work;     // per-partition stored values
    const int32_t* n_live;      // live tuples of this sub-batch (0: nothing to do)
    int cpp;                    // CTAs sharing one partition's work (grid = P * cpp)
    const int4* cta_map;        // or: work-proportional CTAs, (partition, sub, CTAs of it) per CTA
    const int* n_used;          // CTAs in use (with cta_map)
    const unsigned long long* bad;
};

// Work-proportional K4 grid, for the group-reassignment policy without
// hot-key splitting (a partition hosting a top group carries several times
// the mean): partition p gets max(1, floor(total * work_p / sum)) CTAs,
// partition-major; map[b] = (partition, sub, its CTA count) of CTA b, so a
// CTA finds its slot with one load; n_used = CTAs used (<= total + P).
// work_p comes from k_batch_stats; it is cleared for the next batch.
__global__ void __launch_bounds__(1024)
k_cta_map(uint32_t* __restrict__ pwork, int P, int total, int4* __restrict__ map, int* __restrict__ n_used) { SS_PDL_ENTRY();
    __shared__ unsigned long long sh_sum[32];
    __shared__ int32_t sh_red[33];
    const int t = threadIdx.x;
    const unsigned lane = lane_id(), wp = warp_id();
    const uint32_t w = t < P ? pwork[t] : 0u;
    if (t < P) pwork[t] = 0;
    unsigned long long v = warp_sum((unsigned long long)w);
    if (lane == 0) sh_sum[wp] = v;
    __syncthreads();
    if (wp == 0) {
        v = lane < (blockDim.x >> 5) ? sh_sum[lane] : 0ull;
        v = warp_sum(v);
        if (lane == 0) sh_sum[0] = v;
    }
    __syncthreads();
    const unsigned long long tot = sh_sum[0];
    int c = 0;
    if (t < P) c = tot ? max(1, (int)((double)total * (double)w / (double)tot)) : 1;
    int all;
    const int ex = block_excl_scan(c, sh_red, &all);
    // CTA slots of partition t: (t, sub, c) at [ex, ex + c)
    for (int k = 0; k < c; ++k) map[ex + k] = make_int4(t, k, c, 0);
    if (t == 0) *n_used = all;
}

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

// per-member 64-bit delta kept as two native 32-bit shared words (64-bit
// shared atomics are CAS loops on sm_100): low word + carries into high
__device__ __forceinline__ void add_delta(uint32_t* lo, uint32_t* hi, long long v) {
    const unsigned long long x = (unsigned long long)v;
    const uint32_t lo32 = (uint32_t)x;
    const uint32_t prev = atomicAdd(lo, lo32);
    const uint32_t carry = (prev + lo32 < prev) ? 1u : 0u;
    atomicAdd(hi, (uint32_t)(x >> 32) + carry);
}

constexpr int kLILP = 8;                    // values in flight per lane for long members
constexpr int kUnit = 32 * kLILP;           // values of one warp unit (long members)

#ifdef SS_K4_PROF
__device__ unsigned long long g_k4_prof[8];
#endif

__global__ void __launch_bounds__(kIngestThreads, 2)
k_ingest(IngestArgs a) { SS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char ingest_sm[];
    int64_t* m_off = (int64_t*)ingest_sm;
    uint32_t* m_dlo = (uint32_t*)(m_off + kMemberChunk);
    uint32_t* m_dhi = m_dlo + kMemberChunk;
    int32_t* m_g = (int32_t*)(m_dhi + kMemberChunk);
    int32_t* m_scan = m_g + kMemberChunk;            // short members: value scan  [kMemberChunk + 1]
    int32_t* m_uscan = m_scan + kMemberChunk + 4;    // long members: unit scan    [kMemberChunk + 1]
    int32_t* m_start = m_uscan + kMemberChunk + 4;
    int32_t* m_q0 = m_start + kMemberChunk;
    int32_t* m_s0 = m_q0 + kMemberChunk;
    int32_t* m_f0 = m_s0 + kMemberChunk;             // live bound (0 when k >= W)
    int32_t* m_w = m_f0 + kMemberChunk;              // stored values of the member
    int32_t* m_min = m_w + kMemberChunk;
    int32_t* m_max = m_min + kMemberChunk;
    __shared__ int32_t sh_red[33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    if (a.n_live && *a.n_live == 0) return;      // every tuple of the sub-batch was dropped
    uint64_t t0 = 0;
    if (threadIdx.x == 0) t0 = globaltimer();
#ifdef SS_K4_PROF
    long long _pt = clock64();
#define SS_PT4(i) do { if (threadIdx.x == 0) { const long long _n = clock64(); atomicAdd(&g_k4_prof[i], (unsigned long long)(_n - _pt)); _pt = _n; } } while (0)
#else
#define SS_PT4(i) do {} while (0)
#endif
    // partition p is processed by kCtaPerPart CTAs; its members (and split
    // shares) are dealt to them round-robin
    int kCtaPerPart, p, sub;
    if (a.cta_map) {
        // work-proportional: one 16-byte load gives this CTA's slot
        if ((int)blockIdx.x >= *a.n_used) return;
        const int4 m = a.cta_map[blockIdx.x];
        p = m.x;
        sub = m.y;
        kCtaPerPart = m.z;
    } else {
        // partition-minor order: the first resident wave holds CTA 0 (and 1)
        // of every partition, later CTAs of a heavy partition start as light
        // partitions finish
        kCtaPerPart = a.cpp;
        const int P = (int)(gridDim.x / kCtaPerPart);
        p = blockIdx.x % P;
        sub = blockIdx.x / P;
    }
    const int lo = a.offsets[p], hi = a.offsets[p + 1];
    const int s_lo = a.share_off ? a.share_off[p] : 0;
    const int s_hi = a.share_off ? a.share_off[p + 1] : 0;
    const int n_mem = hi - lo;
    const int n_items = n_mem + (s_hi - s_lo);   // members, then split shares
    const int W = (int)a.W;
    const unsigned lane = lane_id();
    const int nw = kIngestThreads / 32;
    unsigned long long work_total = 0;

    // Few items (<= kMemberChunk): every CTA of the partition stages them all
    // and the CTAs interleave the warp units / short values (a hot member's
    // run spreads over all of them).  Many items: they are dealt round-robin
    // (it = sub, sub + kCtaPerPart, ...) so nothing is staged twice.
    // With many items the members are dealt round-robin but the split
    // shares (few, long: a hot group's slices) get a round of their own in
    // which every CTA of the partition stages them all and the CTAs
    // interleave their units -- dealt whole, one CTA of a partition could
    // draw twice the other's share work (C4: CTA times ~2x apart).
    const bool all_shared = n_items <= kMemberChunk;
    for (int ph = 0; ph < (all_shared ? 1 : 2); ++ph) {
    const int ibase = (all_shared || ph == 0) ? 0 : n_mem;
    const int icount = all_shared ? n_items : (ph == 0 ? n_mem : n_items - n_mem);
    const bool shared_items = all_shared || ph == 1;
    const int my_items = shared_items ? icount : (icount - sub + kCtaPerPart - 1) / kCtaPerPart;
    const int cstride = shared_items ? kCtaPerPart : 1;   // interleave factor
    const int csub = shared_items ? sub : 0;
    for (int c0 = 0; c0 < my_items; c0 += kMemberChunk) {
        SS_PT4(0);
        const int m = min(kMemberChunk, my_items - c0);
        // phase A: stage the items thread-strided (item i on thread i mod
        // 512), so a partition with few members costs one dependent load
        // chain per thread, not kMPT of them on a few threads.  Two load
        // levels for all kMPT items together: the groups, then every field
        // of each group (loaded whether or not the member stores anything --
        // the fields of a hash block's 8 ids share a sector), instead of a
        // 4-deep chain per item behind its branches.
        int q_g[kMPT], q_sh[kMPT];
#pragma unroll
        for (int q = 0; q < kMPT; ++q) {
            const int i = q * kIngestThreads + threadIdx.x;
            q_g[q] = -1;
            q_sh[q] = -1;
            if (i >= m) continue;
            const int it = ibase + (shared_items ? c0 + i : (c0 + i) * kCtaPerPart + sub);
            if (it < n_mem) {
                q_g[q] = a.order[lo + it];
            } else {
                q_sh[q] = s_lo + (it - n_mem);
                q_g[q] = a.split_g[a.share_grp[q_sh[q]]];
            }
        }
        // then per item: every field of its group at once (loaded whether or
        // not the member stores anything -- the fields of a hash block's 8
        // ids share a sector), not behind the item's branches
#pragma unroll
        for (int q = 0; q < kMPT; ++q) {
            const int i = q * kIngestThreads + threadIdx.x;
            const int g = q_g[q];
            if (g < 0) continue;
            const bool is_split = a.split_of && a.split_of[g] >= 0;
            const int kt0 = a.gcnt[g];
            const int K = a.gcount[g];                     // batch count
            const int f0 = a.fill[g];
            const int np = a.next_pos[g];
            const int gs = a.gstart[g];
            const int64_t offg = a.off[g];
            int r_lo, r_hi;               // this item's slice [r_lo, r_hi) of the sub-batch run
            int32_t tag;
            if (q_sh[q] < 0) {
                tag = g;
                r_lo = 0;
                r_hi = is_split ? 0 : kt0;
            } else {
                const int sh = q_sh[q];
                const int sg = a.share_grp[sh];
                tag = -1 - sg;
                // shares tile the stored values: the last min(K, W) of the
                // kept run (split.cuh)
                const long long kt = kt0, den = a.split_den[sg];
                const long long sto = min64(K, a.W), off0 = kt - sto;
                r_lo = (int)(off0 + sto * a.share_lo[sh] / den);
                r_hi = (int)(off0 + sto * a.share_hi[sh] / den);
            }
            int w = 0;
            if (r_hi > r_lo) {
                const int b = K - kt0;                     // batch rank of run index 0
                const int first = max(r_lo, K - W - b);    // first stored run index
                if (first < r_hi) {
                    const int jb = b + first;              // batch rank of the first stored value
                    w = r_hi - first;
                    m_start[i] = gs + first;
                    // 32-bit unsigned remainders (f0, next_pos < W <= 2^30
                    // and jb < 2^31 - 2^30 keep the sums in range; a 64-bit
                    // % is a ~70-instruction sequence)
                    const uint32_t uw = (uint32_t)W;
                    const uint32_t q0 = (uint32_t)f0 + (uint32_t)jb;
                    m_q0[i] = (int)(q0 % uw);
                    m_s0[i] = (int)(((uint32_t)np + q0) % uw);
                    m_f0[i] = (K >= W) ? 0 : f0;           // k >= W: nothing old survives
                    m_off[i] = offg;
                    m_dlo[i] = 0;
                    m_dhi[i] = 0;
                    m_min[i] = 0x7fffffff;
                    m_max[i] = (int32_t)0x80000000;
                    if (csub == 0) work_total += (unsigned long long)w;
                }
            }
            m_g[i] = w ? tag : 0x7fffffff;
            m_w[i] = w;
        }
        __syncthreads();
        SS_PT4(1);
        // phase B: thread-contiguous scans of short values and long units
        int32_t wshort[kMPT], wunits[kMPT];
        int32_t ssum = 0, usum = 0;
#pragma unroll
        for (int q = 0; q < kMPT; ++q) {
            const int i = threadIdx.x * kMPT + q;
            const int w = (i < m) ? m_w[i] : 0;
            wunits[q] = (w >= 32) ? (w + kUnit - 1) / kUnit : 0;
            wshort[q] = (w >= 32) ? 0 : w;
            ssum += wshort[q];
            usum += wunits[q];
        }
        int32_t s_total, u_total;
        int32_t sex = block_excl_scan(ssum, sh_red, &s_total);
        int32_t uex = block_excl_scan(usum, sh_red, &u_total);
#pragma unroll
        for (int q = 0; q < kMPT; ++q) {
            const int i = threadIdx.x * kMPT + q;
            if (i < m) {
                m_scan[i] = sex;
                m_uscan[i] = uex;
            }
            sex += wshort[q];
            uex += wunits[q];
        }
        if (threadIdx.x == 0) {
            m_scan[m] = s_total;
            m_uscan[m] = u_total;
        }
        __syncthreads();

        SS_PT4(2);
        // ---- long members: one warp per unit of kUnit contiguous values ----
        // The member lookup of the warp's next unit (a binary search over
        // the unit scan plus the member's fields, all shared memory) is done
        // while the current unit's global loads are in flight.
        struct UnitRef { int mi, r0; };
        auto find_unit = [&](int u) -> UnitRef {
            int mi = 0;                                 // last member with m_uscan[mi] <= u
#pragma unroll
            for (int step = kMemberChunk / 2; step >= 1; step >>= 1) {
                const int c = mi + step;
                if (c < m && m_uscan[c] <= u) mi = c;
            }
            return UnitRef{mi, (u - m_uscan[mi]) * kUnit};
        };
        // a warp's next unit is at or after its current member: gallop from
        // there (a hot member's next unit costs one shared load, a tail
        // member a few) instead of the full 11-step search
        auto next_unit = [&](int u, int mi) -> UnitRef {
            int step = 1;
            while (mi + step < m && m_uscan[mi + step] <= u) {
                mi += step;
                step <<= 1;
            }
            for (step >>= 1; step >= 1; step >>= 1)
                if (mi + step < m && m_uscan[mi + step] <= u) mi += step;
            return UnitRef{mi, (u - m_uscan[mi]) * kUnit};
        };
        const int ustride = cstride * nw;
        int u = csub * nw + warp_id();
        UnitRef cur = u < u_total ? find_unit(u) : UnitRef{0, 0};
        for (; u < u_total; u += ustride) {
            const int mi = cur.mi, r0 = cur.r0;
            const int w = m_w[mi];
            const int start = m_start[mi], q0 = m_q0[mi], s0 = m_s0[mi], f0 = m_f0[mi];
            const int64_t offg = m_off[mi];
            // ring cells are recomputed per phase instead of kept in 64-bit
            // registers: the loads of a unit stay in flight together
            // instead of being serialised by register spills
            const int32_t* vsrc = a.vals + start;
            int32_t* rg = a.ring + offg;
            int32_t v[kLILP], old[kLILP];
#pragma unroll
            for (int k = 0; k < kLILP; ++k) {
                const int r = r0 + k * 32 + (int)lane;
                v[k] = (r < w) ? vsrc[r] : 0;
            }
#pragma unroll
            for (int k = 0; k < kLILP; ++k) {
                const int r = r0 + k * 32 + (int)lane;
                int qq = q0 + r;
                if (qq >= W) qq -= W;
                int sl = s0 + r;
                if (sl >= W) sl -= W;
                old[k] = (r < w && qq < f0) ? rg[sl] : 0;
            }
            if (u + ustride < u_total) cur = next_unit(u + ustride, mi);
            long long d = 0;
            int32_t mnv = 0x7fffffff, mxv = (int32_t)0x80000000;
#pragma unroll
            for (int k = 0; k < kLILP; ++k) {
                const int r = r0 + k * 32 + (int)lane;
                if (r < w) {
                    int sl = s0 + r;
                    if (sl >= W) sl -= W;
                    rg[sl] = v[k];
                    d += (long long)v[k] - (long long)old[k];
                    mnv = min(mnv, v[k]);
                    mxv = max(mxv, v[k]);
                }
            }
            d = warp_sum(d);
            if (a.minmax) {
                mnv = warp_min(mnv);
                mxv = warp_max(mxv);
            }
            if (lane == 0) {
                add_delta(&m_dlo[mi], &m_dhi[mi], d);
                if (a.minmax) {
                    atomicMin(&m_min[mi], mnv);
                    atomicMax(&m_max[mi], mxv);
                }
            }
        }

        // ---- short members (< 32 values): kILP consecutive values per thread
        SS_PT4(3);
        // Thread-contiguous: one binary search per thread (not per value),
        // member fields re-read from shared memory only when the member
        // changes, and the delta / MIN / MAX of each member run accumulated
        // in registers -- one shared flush per (thread, member) instead of
        // a segmented warp reduction per value round.
        for (int base = csub * kIngestThreads * kILP; base < s_total; base += cstride * kIngestThreads * kILP) {
            const int t0 = base + (int)threadIdx.x * kILP;
            if (t0 >= s_total) continue;
            int l = 0;                                 // last member with m_scan[l] <= t0
#pragma unroll
            for (int step = kMemberChunk / 2; step >= 1; step >>= 1) {
                const int c = l + step;
                if (c < m && m_scan[c] <= t0) l = c;
            }
            int f_scan = m_scan[l], f_next = m_scan[l + 1];
            // the member's fields stay in registers until the member changes
            int f_start = m_start[l], f_q0 = m_q0[l], f_s0 = m_s0[l], f_f0 = m_f0[l];
            int64_t f_off = m_off[l];
            int mi[kILP], sl[kILP];
            int32_t v[kILP], old[kILP];
#pragma unroll
            for (int u = 0; u < kILP; ++u) {
                const int t = t0 + u;
                mi[u] = -1;
                sl[u] = 0;
                v[u] = 0;
                old[u] = 0;
                if (t < s_total) {
                    if (t >= f_next) {
                        while (m_scan[l + 1] <= t) ++l;
                        f_scan = m_scan[l];
                        f_next = m_scan[l + 1];
                        f_start = m_start[l];
                        f_q0 = m_q0[l];
                        f_s0 = m_s0[l];
                        f_f0 = m_f0[l];
                        f_off = m_off[l];
                    }
                    const int rr = t - f_scan;
                    mi[u] = l;
                    v[u] = a.vals[f_start + rr];
                    int q = f_q0 + rr;
                    if (q >= W) q -= W;
                    int s2 = f_s0 + rr;
                    if (s2 >= W) s2 -= W;
                    sl[u] = s2;
                    if (q < f_f0) old[u] = a.ring[f_off + s2];
                }
            }
            long long d = 0;
            int32_t mnv = 0x7fffffff, mxv = (int32_t)0x80000000;
            int cur = mi[0];
#pragma unroll
            for (int u = 0; u < kILP; ++u) {
                if (mi[u] < 0) break;
                if (mi[u] != cur) {
                    add_delta(&m_dlo[cur], &m_dhi[cur], d);
                    if (a.minmax) {
                        atomicMin(&m_min[cur], mnv);
                        atomicMax(&m_max[cur], mxv);
                    }
                    cur = mi[u];
                    d = 0;
                    mnv = 0x7fffffff;
                    mxv = (int32_t)0x80000000;
                }
                a.ring[m_off[mi[u]] + sl[u]] = v[u];
                d += (long long)v[u] - (long long)old[u];
                mnv = min(mnv, v[u]);
                mxv = max(mxv, v[u]);
            }
            add_delta(&m_dlo[cur], &m_dhi[cur], d);
            if (a.minmax) {
                atomicMin(&m_min[cur], mnv);
                atomicMax(&m_max[cur], mxv);
            }
        }
        __syncthreads();
        SS_PT4(4);

        // ---- fold into the per-group batch accumulators --------------------
        for (int i = threadIdx.x; i < m; i += kIngestThreads) {
            const int tag = m_g[i];
            if (tag == 0x7fffffff) continue;
            const unsigned long long md = ((unsigned long long)m_dhi[i] << 32) | m_dlo[i];
            // the partition's CTAs (and a split key's shares) meet here:
            // native 64-bit global atomics, integer so order-independent
            const int g = tag >= 0 ? tag : a.split_g[-1 - tag];
            if (md) atomicAdd((unsigned long long*)&a.bdelta[g], md);
            if (a.minmax && m_min[i] <= m_max[i]) {
                atomicMin(&a.bmin[g], m_min[i]);
                atomicMax(&a.bmax[g], m_max[i]);
            }
        }
        __syncthreads();
        SS_PT4(5);
    }
    }
    work_total = warp_sum(work_total);
    if (lane == 0 && a.part_work && work_total) atomicAdd(&a.part_work[p], work_total);
    if (threadIdx.x == 0 && a.part_ns) atomicAdd(&a.part_ns[p], (unsigned long long)(globaltimer() - t0));
}

// The per-batch report (tuples, tpt imbalance, max / sum of block loads,
// moves, ...) -- k_report on the side stream when a policy or split plan
// runs, else folded into k_finalize's last CTA (one launch fewer on C1's
// critical path).  Layout of the host-visible struct: engine.cu DevReport.
struct ReportArgs {
    const unsigned long long* tpt;
    const unsigned long long* loads;     // null: tpt
    int P;
    const unsigned long long* bad;
    const unsigned long long* touched;
    const int* n_moves;
    int* prev_moves;
    const long long* scanned;
    const int* n_split;
    const unsigned* n_res;
    const int* oom;
    long long tuples;
    int has_policy;
    long long* rep;                      // DevReport as 64-bit words (engine.cu)
};

// any blockDim <= 1024 (a multiple of 32); every thread of the CTA calls it
__device__ __forceinline__ void report_body(const ReportArgs& a) {
    __shared__ long long r[4][32];
    long long mx = 0, mnv = LLONG_MAX, ml = 0, ls = 0;
    for (int p = threadIdx.x; p < a.P; p += blockDim.x) {
        const long long t = (long long)a.tpt[p];
        mx = max(mx, t);
        mnv = min(mnv, t);
        const long long l = (long long)(a.loads ? a.loads[p] : a.tpt[p]);
        ml = max(ml, l);
        ls += l;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(SS_FULL, mx, o));
        mnv = min(mnv, __shfl_xor_sync(SS_FULL, mnv, o));
        ml = max(ml, __shfl_xor_sync(SS_FULL, ml, o));
        ls += __shfl_xor_sync(SS_FULL, ls, o);
    }
    if (lane_id() == 0) { r[0][warp_id()] = mx; r[1][warp_id()] = mnv; r[2][warp_id()] = ml; r[3][warp_id()] = ls; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mx = max(mx, r[0][w]); mnv = min(mnv, r[1][w]); ml = max(ml, r[2][w]); ls += r[3][w];
        }
        const unsigned long long bad = *a.bad;
        const int nm = a.has_policy ? *a.n_moves : 0;
        long long* o = a.rep;
        o[0] = (long long)bad;
        o[1] = a.tuples;
        o[2] = a.P ? mx - mnv : 0;
        o[3] = nm;
        o[4] = *a.prev_moves;
        o[5] = a.has_policy ? *a.scanned : 0;
        o[6] = ml;
        o[7] = (long long)*a.touched;
        o[8] = a.n_split ? *a.n_split : 0;
        o[9] = a.n_res ? *a.n_res : 0;
        o[10] = ls;
        reinterpret_cast<int*>(o + 11)[0] = *a.oom;
        *a.prev_moves = (bad == (unsigned long long)kNoBad) ? nm : 0;
    }
}

// K5: fold each touched group's batch delta into its window state, emit
// its result row (group, COUNT, SUM, AVG, MIN, MAX; AVG = correctly
// rounded double quotient) and reset the batch accumulators.
struct FinalizeArgs {
    ReportArgs report;          // used when ticket != null (no side-stream work)
    unsigned* ticket;           // finished CTAs; the last one writes the report
    const int32_t* gcount;
    int32_t* gcnt;              // [n_sub][G] chunk counts, cleared here
    int n_sub;
    const int32_t* lc;          // live chunks (the only rows still holding counts) or null
    const int32_t* n_lc;
    uint32_t G;
    int64_t W;
    int32_t* fill;
    int32_t* next_pos;
    long long* wsum;
    int32_t* mn;
    int32_t* mx;
    long long* bdelta;
    int32_t* bmin;
    int32_t* bmax;
    int minmax;
    int emit;
    unsigned* n_res;
    int32_t* r_g;
    int32_t* r_cnt;
    long long* r_sum;
    double* r_avg;
    int32_t* r_mn;
    int32_t* r_mx;
    int4* rescan;               // (group, result row, old next_pos | -1, batch count) whose MIN/MAX need a rescan
    unsigned* n_rescan;
    int32_t* sum_idx;           // [G] chunk-summary slot of a group (-1: none), or null (no summaries)
    uint8_t* sum_valid;         // [G] its summaries describe the current ring
    int* n_sum;                 // slots handed out
    const unsigned long long* bad;
};

__device__ __forceinline__ void finalize_body(const FinalizeArgs& a);

__global__ void __launch_bounds__(256)
k_finalize(FinalizeArgs a) { SS_PDL_ENTRY();
    if (*a.bad == (unsigned long long)kNoBad) finalize_body(a);
    if (!a.ticket) return;
    // the last CTA to finish writes the batch report
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    report_body(a.report);
    if (threadIdx.x == 0) *a.ticket = 0;
}

__device__ __forceinline__ void finalize_body(const FinalizeArgs& a) {
    const unsigned lane = lane_id(), wp = warp_id();
    const int W = (int)a.W;
    // result rows: one atomic per CTA round on the row counter (one per warp
    // serialised 31K same-address atomics at 1M groups)
    __shared__ unsigned s_wcnt[8], s_base;
    for (uint32_t g0 = blockIdx.x * blockDim.x; g0 < a.G; g0 += gridDim.x * blockDim.x) {
        const uint32_t g = g0 + threadIdx.x;
        const int K = (g < a.G) ? a.gcount[g] : 0;
        const bool t = K != 0;
        unsigned slot = 0;
        if (a.emit) {
            const unsigned bal = __ballot_sync(SS_FULL, t);
            if (lane == 0) s_wcnt[wp] = (unsigned)__popc(bal);
            __syncthreads();
            unsigned pre = 0, all = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const unsigned c = s_wcnt[q];
                pre += (q < (int)wp) ? c : 0u;
                all += c;
            }
            if (threadIdx.x == 0) s_base = all ? atomicAdd(a.n_res, all) : 0u;
            __syncthreads();
            slot = s_base + pre + __popc(bal & lanemask_lt());
        }
        if (!t) continue;
        const int f0 = a.fill[g];
        const int64_t tot = (int64_t)f0 + K;
        const int p0 = a.next_pos[g];
        const int fill = (int)min64(tot, W);
        a.fill[g] = fill;
        // 32-bit remainder: p0 < W <= 2^30 and tot - W <= K <= 2^30
        a.next_pos[g] = (int32_t)(((uint32_t)p0 + (uint32_t)max64(tot - W, 0)) % (uint32_t)W);
        const long long d = a.bdelta[g];
        const long long s = (K >= W) ? d : a.wsum[g] + d;
        a.wsum[g] = s;
        a.bdelta[g] = 0;
        bool need_rescan = false;
        int32_t lo = 0, hi = 0;
        if (a.minmax) {
            const int32_t bl = a.bmin[g], bh = a.bmax[g];
            if (tot <= W || K >= W) {
                const bool keep_old = (f0 > 0) && (K < W);
                lo = keep_old ? min(a.mn[g], bl) : bl;
                hi = keep_old ? max(a.mx[g], bh) : bh;
                a.mn[g] = lo;
                a.mx[g] = hi;
            } else {
                need_rescan = true;
            }
            a.bmin[g] = 0x7fffffff;
            a.bmax[g] = (int32_t)0x80000000;
        }
        if (need_rescan) {
            // p0 = -1: the window was not full before this batch (its chunk
            // summaries, if any, are rebuilt from the whole ring)
            if (a.sum_idx && a.sum_idx[g] < 0) a.sum_idx[g] = atomicAdd(a.n_sum, 1);
            a.rescan[atomicAdd(a.n_rescan, 1u)] = make_int4((int)g, a.emit ? (int)slot : -1, f0 == W ? p0 : -1, K);
        } else if (a.sum_valid && K >= W) {
            a.sum_valid[g] = 0;                          // the whole window was replaced
        }
        if (a.emit) {
            a.r_g[slot] = (int32_t)g;
            a.r_cnt[slot] = fill;
            a.r_sum[slot] = s;
            a.r_avg[slot] = __ll2double_rn(s) / (double)fill;
            if (a.minmax) {
                a.r_mn[slot] = lo;
                a.r_mx[slot] = hi;
            }
        }
    }
    // clear the batch's chunk histograms for the next batch: whole rows of
    // the live chunks (every other row is already zero), a row per CTA
    // (few rows of many groups: each row is cut into segments over the grid)
    const int nrows = a.lc ? *a.n_lc : a.n_sub;
    const bool v4 = (a.G & 3u) == 0;
    const uint32_t nq = v4 ? a.G / 4 : a.G;                  // stores per row
    const int segs = nrows ? max(1, min((int)gridDim.x / nrows, (int)((nq + 1023) / 1024))) : 1;
    const uint32_t per = (nq + segs - 1) / segs;
    for (int t = blockIdx.x; t < nrows * segs; t += gridDim.x) {
        const int i = t / segs, sg = t - i * segs;
        int32_t* row = a.gcnt + (int64_t)(a.lc ? a.lc[i] : i) * a.G;
        const uint32_t q1 = min(nq, (sg + 1) * per);
        for (uint32_t q = sg * per + threadIdx.x; q < q1; q += blockDim.x) {
            if (v4) reinterpret_cast<int4*>(row)[q] = make_int4(0, 0, 0, 0);
            else row[q] = 0;
        }
    }
}

// MIN/MAX of a full window after a partial eviction (hard part
// 3): every ring slot is live, so the slot order does not matter.
//  * small windows (W <= kMMSumMinW): chunk-parallel rescan of the whole
//    window -- the listed groups' windows cut into kRescanChunk-value chunks
//    over the grid, folded with atomicMin/Max after a reset;
//  * large windows: per-group chunk summaries (min, max of each kMMChunk
//    ring slots).  A batch rewrites ring slots [p0, p0 + K) mod W of a full
//    window, so only the chunks it touched are rescanned (K + 2 kMMChunk
//    values), then the W / kMMChunk summaries are folded -- instead of W
//    values per group and batch.  A group's summaries are built from the
//    whole ring the first time it needs them, and dropped (sum_valid = 0)
//    when a batch replaces its whole window or its state is imported.
constexpr int kRescanChunk = 16384;
constexpr int kMMChunk = 4096;
constexpr int64_t kMMSumMinW = 1 << 17;

__global__ void k_rescan_reset(const int4* __restrict__ rescan, const unsigned* __restrict__ n_rescan,
                               int32_t* __restrict__ mn, int32_t* __restrict__ mx) { SS_PDL_ENTRY();
    const unsigned n = *n_rescan;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        mn[rescan[i].x] = 0x7fffffff;
        mx[rescan[i].x] = (int32_t)0x80000000;
    }
}

// min / max of ring values [lo, hi) of one group, CTA-wide (256 threads)
__device__ __forceinline__ int2 cta_minmax(const int32_t* __restrict__ r, int64_t lo, int64_t hi) {
    __shared__ int32_t s_mn[8], s_mx[8];
    int32_t a = 0x7fffffff, b = (int32_t)0x80000000;
    for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
        const int32_t v = r[j];
        a = min(a, v);
        b = max(b, v);
    }
    a = warp_min(a);
    b = warp_max(b);
    if (lane_id() == 0) { s_mn[warp_id()] = a; s_mx[warp_id()] = b; }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int w = 1; w < 8; ++w) { a = min(a, s_mn[w]); b = max(b, s_mx[w]); }
    __syncthreads();
    return make_int2(a, b);         // valid in thread 0
}

__global__ void __launch_bounds__(256)
k_minmax_rescan(const int4* __restrict__ rescan, const unsigned* __restrict__ n_rescan,
                const int32_t* __restrict__ ring, const int64_t* __restrict__ off, int64_t W,
                int32_t* __restrict__ mn, int32_t* __restrict__ mx) { SS_PDL_ENTRY();
    const unsigned n = *n_rescan;
    const int64_t nch = (W + kRescanChunk - 1) / kRescanChunk;
    for (int64_t c = blockIdx.x; c < (int64_t)n * nch; c += gridDim.x) {
        const int4 e = rescan[c / nch];
        const int64_t lo = (c % nch) * kRescanChunk;
        const int2 r = cta_minmax(ring + off[e.x], lo, min64(W, lo + kRescanChunk));
        if (threadIdx.x == 0) {
            atomicMin(&mn[e.x], r.x);
            atomicMax(&mx[e.x], r.y);
        }
    }
}

__global__ void k_rescan_rows(const int4* __restrict__ rescan, const unsigned* __restrict__ n_rescan,
                              const int32_t* __restrict__ mn, const int32_t* __restrict__ mx,
                              int32_t* __restrict__ r_mn, int32_t* __restrict__ r_mx) { SS_PDL_ENTRY();
    const unsigned n = *n_rescan;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int4 e = rescan[i];
        if (e.y >= 0) {
            r_mn[e.y] = mn[e.x];
            r_mx[e.y] = mx[e.x];
        }
    }
}

// chunk summaries: rescan the chunks this batch touched (all of them when
// the group's summaries are not valid)
__global__ void __launch_bounds__(256)
k_mm_refresh(const int4* __restrict__ rescan, const unsigned* __restrict__ n_rescan,
             const int32_t* __restrict__ ring, const int64_t* __restrict__ off, int64_t W,
             const int32_t* __restrict__ sum_idx, const uint8_t* __restrict__ sum_valid, int2* __restrict__ sums) { SS_PDL_ENTRY();
    const unsigned n = *n_rescan;
    const int64_t nch = (W + kMMChunk - 1) / kMMChunk;
    for (int64_t c = blockIdx.x; c < (int64_t)n * nch; c += gridDim.x) {
        const int4 e = rescan[c / nch];
        const int64_t ci = c % nch;
        const int64_t lo = ci * kMMChunk, hi = min64(W, lo + kMMChunk);
        if (e.z >= 0 && sum_valid[e.x]) {
            // written slots: (p0 + j) mod W, 0 <= j < K
            const int64_t p0 = e.z;
            const bool touched = (p0 >= lo && p0 < hi) || ((lo - p0 + W) % W) < (int64_t)e.w;
            if (!touched) continue;
        }
        const int2 r = cta_minmax(ring + off[e.x], lo, hi);
        if (threadIdx.x == 0) sums[(int64_t)sum_idx[e.x] * nch + ci] = r;
    }
}

// fold a group's summaries -> MIN/MAX state and its result row
__global__ void __launch_bounds__(256)
k_mm_fold(const int4* __restrict__ rescan, const unsigned* __restrict__ n_rescan, int64_t W,
          const int32_t* __restrict__ sum_idx, uint8_t* __restrict__ sum_valid, const int2* __restrict__ sums,
          int32_t* __restrict__ mn, int32_t* __restrict__ mx, int32_t* __restrict__ r_mn, int32_t* __restrict__ r_mx) { SS_PDL_ENTRY();
    __shared__ int32_t s_mn[8], s_mx[8];
    const unsigned n = *n_rescan;
    const int64_t nch = (W + kMMChunk - 1) / kMMChunk;
    for (unsigned i = blockIdx.x; i < n; i += gridDim.x) {
        const int4 e = rescan[i];
        const int2* s = sums + (int64_t)sum_idx[e.x] * nch;
        int32_t a = 0x7fffffff, b = (int32_t)0x80000000;
        for (int64_t j = threadIdx.x; j < nch; j += blockDim.x) {
            const int2 v = s[j];
            a = min(a, v.x);
            b = max(b, v.y);
        }
        a = warp_min(a);
        b = warp_max(b);
        if (lane_id() == 0) { s_mn[warp_id()] = a; s_mx[warp_id()] = b; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; ++w) { a = min(a, s_mn[w]); b = max(b, s_mx[w]); }
            mn[e.x] = a;
            mx[e.x] = b;
            if (e.y >= 0) {
                r_mn[e.y] = a;
                r_mx[e.y] = b;
            }
            sum_valid[e.x] = 1;
        }
        __syncthreads();
    }
}

// Occupancy-proportional store: before a batch, grow the ring region of
// every group whose window will hold more values than its capacity
// (capacity doubles up to W; a window below W is linear, next_pos == 0,
// so growth copies `fill` values).  Phase 1 reserves (warp-aggregated
// atomics on the pool top) and lists the copies cut into kCopyChunk-value
// pieces, so a hot group's multi-million-value copy spreads over the whole
// grid; phase 2 copies one piece per CTA.
constexpr int kCopyChunk = 8192;
// growth factor of a ring region: every value is copied 1/(kGrow-1) times
// on average while its window grows (2x copied each value about once; the
// C4 growth copies were ~0.17 ms of a 1.2 ms step)
constexpr int64_t kGrow = 4;

struct RingCopy {
    int64_t src, dst;
    int32_t len, pad;
};

__global__ void __launch_bounds__(256)
k_reserve(const int32_t* __restrict__ gcount, uint32_t G, int64_t W, const int32_t* __restrict__ fill,
          int64_t* __restrict__ off, int32_t* __restrict__ cap, unsigned long long* __restrict__ pool_top,
          unsigned long long pool_cap, int* __restrict__ oom, RingCopy* __restrict__ copies,
          unsigned* __restrict__ n_copies, const unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    __shared__ long long sh_red[33];
    __shared__ unsigned long long sh_base;
    __shared__ unsigned sh_cbase;
    __shared__ unsigned sh_cred[33];
    if (*bad != (unsigned long long)kNoBad) return;
    // one pool reservation and one copy-list reservation per CTA and round
    // (a reservation per warp serialises ~G/32 atomics on one address)
    for (uint32_t g0 = blockIdx.x * blockDim.x; g0 < G; g0 += gridDim.x * blockDim.x) {
        const uint32_t g = g0 + threadIdx.x;
        int64_t ncap = 0, oldoff = 0;
        int f = 0;
        if (g < G) {
            const int k = gcount[g];
            if (k) {
                f = fill[g];
                const int c = cap[g];
                const int64_t need = min64((int64_t)f + k, W);
                if (need > c) {
                    ncap = min64(W, max64(max64(need, kGrow * (int64_t)c), 16));
                    oldoff = off[g];
                }
            }
        }
        const unsigned nch = (ncap && f) ? (unsigned)((f + kCopyChunk - 1) / kCopyChunk) : 0u;
        long long tot;
        const long long ex = block_excl_scan((long long)ncap, sh_red, &tot);
        unsigned ctot;
        const unsigned cex = block_excl_scan(nch, sh_cred, &ctot);
        if (threadIdx.x == 0) {
            sh_base = tot ? atomicAdd(pool_top, (unsigned long long)tot) : 0ull;
            sh_cbase = ctot ? atomicAdd(n_copies, ctot) : 0u;
        }
        __syncthreads();
        if (ncap) {
            const int64_t noff = (int64_t)sh_base + ex;
            if ((unsigned long long)(noff + ncap) > pool_cap) {
                *oom = 1;
            } else {
                const unsigned c0 = sh_cbase + cex;
                for (unsigned c = 0; c < nch; ++c) {
                    RingCopy rc;
                    rc.src = oldoff + (int64_t)c * kCopyChunk;
                    rc.dst = noff + (int64_t)c * kCopyChunk;
                    rc.len = min(kCopyChunk, f - (int)c * kCopyChunk);
                    rc.pad = 0;
                    copies[c0 + c] = rc;
                }
                off[g] = noff;
                cap[g] = (int32_t)ncap;
            }
        }
        __syncthreads();
    }
}

// Most copies are short (tail groups growing 16 -> 32 -> 64 ...): a warp
// takes 32 consecutive copy records, each lane copies a short one (<= 64
// values) on its own.  Long records (a growing hot group, cut into
// kCopyChunk pieces) are copied by whole CTAs afterwards, 8 values in
// flight per thread -- one warp per long record left a serial chain of
// 64 load -> store round trips per 8192-value piece (C4: 42 us per batch
// at 4 % of DRAM bandwidth).
constexpr int kShortCopy = 64;

__global__ void __launch_bounds__(256)
k_ring_copy(const RingCopy* __restrict__ copies, const unsigned* __restrict__ n_copies, int32_t* __restrict__ ring) { SS_PDL_ENTRY();
    const unsigned n = *n_copies;
    const unsigned lane = lane_id();
    const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
    for (unsigned base = (blockIdx.x * (blockDim.x >> 5) + warp_id()) * 32u; base < n; base += nwarps * 32u) {
        const unsigned i = base + lane;
        RingCopy c{};
        if (i < n) c = copies[i];
        if (c.len > 0 && c.len <= kShortCopy) {
            const int32_t* src = ring + c.src;
            int32_t* dst = ring + c.dst;
            for (int j = 0; j < c.len; j += 8) {
                int32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = (j + u < c.len) ? src[j + u] : 0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (j + u < c.len) dst[j + u] = v[u];
            }
        }
    }
    // long records: one CTA each (grid-stride)
    for (unsigned r = blockIdx.x; r < n; r += gridDim.x) {
        const RingCopy c = copies[r];
        if (c.len <= kShortCopy) continue;
        constexpr int U = 8;
        for (int j0 = 0; j0 < c.len; j0 += U * (int)blockDim.x) {
            int32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * (int)blockDim.x + (int)threadIdx.x;
                v[u] = j < c.len ? ring[c.src + j] : 0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * (int)blockDim.x + (int)threadIdx.x;
                if (j < c.len) ring[c.dst + j] = v[u];
            }
        }
    }
}

}  // namespace ss
