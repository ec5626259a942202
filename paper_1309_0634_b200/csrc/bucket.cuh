// bucket.cuh -- K3c: stable placement for large group domains (G > 2^14)
// as two local passes over group BUCKETS instead of a global radix sort.
//
// Reference behaviour: reorder_batch (partition.py:161-178) / the stable
// regroup of ingest_sequence (engine.py:274-280): every group's tuples end
// up contiguous, in arrival order.  What the window update needs is the
// kept suffix of each group's batch run at gstart[g] (exclusive prefix of
// the kept counts), in arrival order.
//
// The batch's group counts are known before placement (K2), so the group
// id space is cut into BINS, in group order:
//   * a hot group (batch count K >= kBkTau) is a bin of its own; its final
//     run is known, so pass 1 writes its kept tuples straight there (a
//     tuple of batch rank r < K - kept is never stored and is dropped);
//   * the other (cold) groups form buckets: maximal runs of consecutive
//     cold groups whose run starts gstart[g] fall in the same kBkC-window
//     and whose ids share the same 2^kBkSpanBits block.  A bucket holds
//     < kBkC + kBkTau tuples and spans <= 2^kBkSpanBits groups.
// Because bins follow group order, a bin's tuples occupy one contiguous
// range of the final layout: [gstart[first group], gstart[next bin's]).
//
//   k_bk_flags_*  per group: bin starts -> bin_of[g] (u16), bin_first[b],
//                 hot flag of b; the bin count (3-kernel scan over G)
//   k_bk_hist     one CTA per super-tile (1/148 of the batch): per-bin
//                 tuple counts in shared memory; the tuples' bin ids are
//                 written out (2 B/tuple) so pass 1 needs no gather
//   k_bk_colscan  per bin: exclusive prefix over the super-tiles + total
//   k_bk_binscan  staging base of every cold bucket (scan over bins)
//   k_bk_scatter  pass 1, one CTA per super-tile walking it in 4096-tuple
//                 sub-tiles (double-buffered cp.async.bulk loads onto an
//                 mbarrier): a stable LSD sort of the sub-tile by bin in
//                 shared memory (2 x 7-bit digits, warp ranks by MATCH),
//                 then each run of equal bins is written contiguously from
//                 the bin's cursor (shared memory, carried across
//                 sub-tiles): hot bins to the final layout, cold buckets to
//                 a staging area in arrival order
//   k_bk_local    pass 2, a CTA per cold bucket: a stable LSD sort by the
//                 group's offset inside the bucket (<= 2 x 6-bit digits) in
//                 shared memory; sorted order IS the final order, so the
//                 values are written to gstart[first group] + position
// Traffic: keys 4 B (hist) + keys/values/bins 10 B (pass 1) + hot values
// 4 B or cold staging 8 B + 8 B (pass 2) + values 4 B out, against 16 B per
// radix pass x 2 plus the chunk histograms of the previous placement.
// Requires every cold group to keep all its tuples (W >= kBkTau) and a
// batch <= 2^24; otherwise the engine uses the radix passes.
#pragma once

#include "common.cuh"

namespace ss {

constexpr int kBkTau = 8192;          // hot: batch count >= kBkTau
constexpr int kBkC = 4096;            // cold bucket window in the kept prefix
constexpr int kBkSpanBits = 12;       // a bucket spans <= 4096 group ids
constexpr int kBkNBMax = 16384;       // bins (a 2^24 batch needs <= ~8.5K)
constexpr int kBkCap = kBkC + kBkTau; // tuples of one cold bucket (exclusive bound)
constexpr int kBkSub = 4096;          // pass-1 sub-tile
constexpr int kBkSupers = kNumSM;     // pass-1 / hist super-tiles (one CTA per SM)
constexpr int kBkBlk = 4096;          // groups per block in the flag scans
constexpr int64_t kBkMaxBatch = 1 << 24;

// ---- cp.async.bulk + mbarrier (Blackwell bulk copies, one thread issues) --
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" :: "r"(a), "r"(parity) : "memory");
}
// streamed input: evict_first in L2, so the scattered staging writes keep
// their partially written sectors resident
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"(d), "l"(src), "r"(bytes), "r"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct BucketArgs {
    const uint32_t* keys;       // [n] group ids (slots)
    const int32_t* vals;        // [n]
    int64_t n;
    uint32_t G;
    const int32_t* gcount;      // [G] batch count K
    const int32_t* gkept;       // [G] kept count (suffix of the batch run)
    const int32_t* gstart;      // [G] exclusive prefix of gkept
    uint16_t* bin_of;           // [G]
    int32_t* bin_first;         // [kBkNBMax + 1] first group of each bin (G after the last)
    uint8_t* bin_hot;           // [kBkNBMax]
    int32_t* n_bins;            // [1]
    int32_t* fsum;              // [G / kBkBlk + 1] flag block sums
    uint16_t* tbin;             // [n] bin of each tuple
    uint32_t* hist;             // [kBkSupers][kBkNBMax] counts -> exclusive prefixes
    uint32_t* btot;             // [kBkNBMax] bin totals
    uint32_t* sbase;            // [kBkNBMax] staging base of each cold bucket
    uint32_t* skey;             // [n] staging
    int32_t* sval;              // [n]
    int32_t* vout;              // [kept total] final layout
    const unsigned long long* bad;
};

__device__ __forceinline__ bool bk_hot(const BucketArgs& a, uint32_t g) { return a.gcount[g] >= kBkTau; }

// bin-start flag of group g (reads g-1's state)
__device__ __forceinline__ int bk_flag(const BucketArgs& a, uint32_t g) {
    if (bk_hot(a, g)) return 1;
    if (g == 0) return 1;
    if (bk_hot(a, g - 1)) return 1;
    const uint32_t w0 = (uint32_t)a.gstart[g - 1] / kBkC, w1 = (uint32_t)a.gstart[g] / kBkC;
    return (w0 != w1 || ((g - 1) >> kBkSpanBits) != (g >> kBkSpanBits)) ? 1 : 0;
}

__global__ void __launch_bounds__(1024)
k_bk_flags_reduce(BucketArgs a) { SS_PDL_ENTRY();
    __shared__ int32_t red[33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const uint32_t g0 = blockIdx.x * kBkBlk;
    int c = 0;
    for (uint32_t g = g0 + threadIdx.x; g < min(a.G, g0 + kBkBlk); g += blockDim.x) c += bk_flag(a, g);
    int32_t tot;
    block_excl_scan(c, red, &tot);
    if (threadIdx.x == 0) a.fsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024)
k_bk_flags_top(BucketArgs a, int nblk) { SS_PDL_ENTRY();
    __shared__ int32_t red[33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    int32_t carry = 0;
    for (int b0 = 0; b0 < nblk; b0 += 1024) {
        const int b = b0 + threadIdx.x;
        const int32_t v = b < nblk ? a.fsum[b] : 0;
        int32_t tot;
        const int32_t ex = block_excl_scan(v, red, &tot);
        if (b < nblk) a.fsum[b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) {
        // unreachable for batches <= kBkMaxBatch (<= ~8.5K bins)
        if (carry > kBkNBMax) __trap();
        *a.n_bins = carry;
        a.bin_first[carry] = (int32_t)a.G;
    }
}

// bin ids: groups in block order, 4 consecutive groups per thread
__global__ void __launch_bounds__(1024)
k_bk_flags_down(BucketArgs a) { SS_PDL_ENTRY();
    __shared__ int32_t red[33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const uint32_t g0 = blockIdx.x * kBkBlk + threadIdx.x * 4;
    int f[4];
    int c = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        f[q] = (g0 + q < a.G) ? bk_flag(a, g0 + q) : 0;
        c += f[q];
    }
    int32_t tot;
    int32_t ex = block_excl_scan(c, red, &tot) + a.fsum[blockIdx.x];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t g = g0 + q;
        if (g >= a.G) break;
        ex += f[q];
        const int32_t b = ex - 1;
        if (b < kBkNBMax) {
            a.bin_of[g] = (uint16_t)b;
            if (f[q]) {
                a.bin_first[b] = (int32_t)g;
                a.bin_hot[b] = bk_hot(a, g) ? 1 : 0;
            }
        }
    }
}

__device__ __forceinline__ int bk_range(int64_t n, int c, int64_t* t0) {
    // super-tile c: whole sub-tiles, the last one possibly short
    const int64_t per = ((n + kBkSupers - 1) / kBkSupers + kBkSub - 1) / kBkSub * kBkSub;
    const int64_t s = min64(n, (int64_t)c * per), e = min64(n, s + per);
    *t0 = s;
    return (int)(e - s);
}

// per-bin counts of one super-tile; the tuples' bin ids are written out
__global__ void __launch_bounds__(1024)
k_bk_hist(BucketArgs a) { SS_PDL_ENTRY();
    extern __shared__ uint32_t bk_sm[];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int nb = *a.n_bins;
    if (nb > kBkNBMax) return;
    int64_t t0;
    const int len = bk_range(a.n, blockIdx.x, &t0);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) bk_sm[i] = 0;
    __syncthreads();
    const unsigned lane = lane_id();
    const bool vec = ((uintptr_t)(a.keys + t0) % 16) == 0;
    for (int base = 0; base < len; base += 4 * blockDim.x) {
        const int i = base + 4 * threadIdx.x;
        uint32_t k[4] = {0, 0, 0, 0};
        const bool full = vec && i + 4 <= len;
        if (full) {
            const uint4 v = ld_stream_v4(a.keys + t0 + i);
            k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) if (i + q < len) k[q] = a.keys[t0 + i + q];
        }
        uint32_t b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) b[q] = (i + q < len) ? (uint32_t)a.bin_of[k[q]] : 0xffffffffu;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // hot bins carry many tuples of a warp: one shared atomic per distinct bin
            const unsigned peers = __match_any_sync(SS_FULL, b[q]);
            if (b[q] != 0xffffffffu && lane == 31u - __clz(peers)) atomicAdd(&bk_sm[b[q]], (uint32_t)__popc(peers));
        }
        if (full) {
            uint2 o;
            o.x = (b[0] & 0xffffu) | (b[1] << 16);
            o.y = (b[2] & 0xffffu) | (b[3] << 16);
            *(uint2*)(a.tbin + t0 + i) = o;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) if (i + q < len) a.tbin[t0 + i + q] = (uint16_t)b[q];
        }
    }
    __syncthreads();
    uint32_t* row = a.hist + (int64_t)blockIdx.x * kBkNBMax;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) row[i] = bk_sm[i];
}

// per bin (lane), the super-tiles split over the warps: exclusive prefix
// over the super-tiles in place, the bin total
__global__ void __launch_bounds__(1024)
k_bk_colscan(BucketArgs a) { SS_PDL_ENTRY();
    __shared__ uint32_t part[32][33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int nb = *a.n_bins;
    if (nb > kBkNBMax) return;
    const int b = blockIdx.x * 32 + (int)lane_id();
    if (blockIdx.x * 32 >= nb) return;
    const int w = warp_id();
    constexpr int per = (kBkSupers + 31) / 32;
    const int r0 = w * per, r1 = min(kBkSupers, r0 + per);
    uint32_t s = 0;
    for (int r = r0; r < r1; ++r) s += (b < nb) ? a.hist[(int64_t)r * kBkNBMax + b] : 0u;
    part[w][lane_id()] = s;
    __syncthreads();
    uint32_t base = 0;
    for (int ww = 0; ww < w; ++ww) base += part[ww][lane_id()];
    if (w == 31 && b < nb) a.btot[b] = base + s;
    for (int r = r0; r < r1; ++r) {
        if (b < nb) {
            uint32_t* p = a.hist + (int64_t)r * kBkNBMax + b;
            const uint32_t c = *p;
            *p = base;
            base += c;
        }
    }
}

// staging base of each cold bucket (hot bins take no staging space)
__global__ void __launch_bounds__(1024)
k_bk_binscan(BucketArgs a) { SS_PDL_ENTRY();
    __shared__ uint32_t red[33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int nb = *a.n_bins;
    if (nb > kBkNBMax) return;
    uint32_t carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 1024) {
        const int b = b0 + threadIdx.x;
        const uint32_t v = (b < nb && !a.bin_hot[b]) ? a.btot[b] : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan(v, red, &tot);
        if (b < nb) a.sbase[b] = carry + ex;
        carry += tot;
    }
}

// ---- block-local stable LSD pass over 7-bit digits ------------------------
// NT threads, items in warp-blocked order (warp w owns [w*IPW, (w+1)*IPW),
// round r holds w*IPW + 32r + lane).  `wh` = NW x 128 u16 counters.
template <int NT, int IPW, typename KeyF>
__device__ __forceinline__ void bk_lsd_pass(const uint32_t* src, uint32_t* dst, int shift, uint16_t* wh, KeyF getk) {
    constexpr int NW = NT / 32;
    constexpr int R = IPW / 32;
    constexpr int D = 128;
    // few rounds: keys and ranks stay in registers between the count and the
    // scatter; many rounds: the scatter re-ranks from the scanned offsets
    constexpr bool REG = R <= 8;
    constexpr int RR = REG ? R : 1;
    const unsigned w = warp_id(), lane = lane_id();
    uint16_t* my = wh + w * D;
    for (int i = lane; i < D; i += 32) my[i] = 0;
    __syncwarp();
    uint32_t key[RR];
    uint16_t rk[RR];
    const unsigned lt = lanemask_lt();
#pragma unroll(REG ? R : 1)
    for (int r = 0; r < R; ++r) {
        const int it = (int)w * IPW + r * 32 + (int)lane;
        const uint32_t k = src ? src[it] : getk(it);
        const uint32_t d = (k >> shift) & (D - 1);
        const unsigned peers = __match_any_sync(SS_FULL, d);
        const uint16_t before = my[d];
        __syncwarp();
        if (REG) {
            key[REG ? r : 0] = k;
            rk[REG ? r : 0] = (uint16_t)(before + __popc(peers & lt));
        }
        if (lane == 31u - __clz(peers)) my[d] = (uint16_t)(before + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    // exclusive scan over (digit, warp), digit-major: NT threads, each
    // (D * NW) / NT consecutive entries
    constexpr int E = D * NW / NT;
    __shared__ uint32_t red[33];
    const int e0 = threadIdx.x * E;
    uint32_t v[E], s = 0;
#pragma unroll
    for (int q = 0; q < E; ++q) {
        const int e = e0 + q, d = e / NW, ww = e % NW;
        v[q] = wh[ww * D + d];
        s += v[q];
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan_nt(s, red, &tot);
    __syncthreads();                  // every counter read before any is overwritten
#pragma unroll
    for (int q = 0; q < E; ++q) {
        const int e = e0 + q, d = e / NW, ww = e % NW;
        wh[ww * D + d] = (uint16_t)ex;
        ex += v[q];
    }
    __syncthreads();
    if (REG) {
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            const uint32_t d = (key[r] >> shift) & (D - 1);
            dst[my[d] + rk[r]] = key[r];
        }
    } else {
        for (int r = 0; r < R; ++r) {
            const int it = (int)w * IPW + r * 32 + (int)lane;
            const uint32_t k = src ? src[it] : getk(it);
            const uint32_t d = (k >> shift) & (D - 1);
            const unsigned peers = __match_any_sync(SS_FULL, d);
            const uint16_t before = my[d];
            __syncwarp();
            dst[before + __popc(peers & lt)] = k;
            if (lane == 31u - __clz(peers)) my[d] = (uint16_t)(before + __popc(peers));
            __syncwarp();
        }
    }
    __syncthreads();
}

constexpr int kBkThreads = 1024;
constexpr int kBkIPW = kBkSub / (kBkThreads / 32);     // 128 items per warp
struct BkSmem {
    static constexpr size_t cursor = 0;                                   // u32[kBkNBMax]
    static constexpr size_t runst = cursor + (size_t)kBkNBMax * 4;        // u16[kBkNBMax]
    static constexpr size_t ka = runst + (size_t)kBkNBMax * 2;            // u32[kBkSub]
    static constexpr size_t kb = ka + (size_t)kBkSub * 4;                 // u32[kBkSub]
    static constexpr size_t sl = kb + (size_t)kBkSub * 4;                 // u32[2][kBkSub]
    static constexpr size_t va = sl + (size_t)2 * kBkSub * 4;             // i32[2][kBkSub]
    static constexpr size_t bn = va + (size_t)2 * kBkSub * 4;             // u16[2][kBkSub]
    static constexpr size_t wh = bn + (size_t)2 * kBkSub * 2;             // u16[32][128]
    static constexpr size_t bar = wh + (size_t)32 * 128 * 2;              // u64[2]
    static constexpr size_t bytes = bar + 16;
};

// pass 1
__global__ void __launch_bounds__(kBkThreads, 1)
k_bk_scatter(BucketArgs a) { SS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char bsm[];
    uint32_t* cursor = (uint32_t*)(bsm + BkSmem::cursor);
    uint16_t* runst = (uint16_t*)(bsm + BkSmem::runst);
    uint32_t* ka = (uint32_t*)(bsm + BkSmem::ka);
    uint32_t* kb = (uint32_t*)(bsm + BkSmem::kb);
    uint32_t* sl = (uint32_t*)(bsm + BkSmem::sl);
    int32_t* va = (int32_t*)(bsm + BkSmem::va);
    uint16_t* bn = (uint16_t*)(bsm + BkSmem::bn);
    uint16_t* wh = (uint16_t*)(bsm + BkSmem::wh);
    uint64_t* bar = (uint64_t*)(bsm + BkSmem::bar);
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int nb = *a.n_bins;
    if (nb > kBkNBMax) return;
    int64_t t0;
    const int len = bk_range(a.n, blockIdx.x, &t0);
    if (len <= 0) return;
    // cursors: cold buckets from their staging base, hot bins from their
    // batch rank base
    const uint32_t* row = a.hist + (int64_t)blockIdx.x * kBkNBMax;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) cursor[b] = row[b] + (a.bin_hot[b] ? 0u : a.sbase[b]);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nsub = (len + kBkSub - 1) / kBkSub;
    // a sub-tile: full ones by bulk copies (thread 0), the short last one by
    // plain loads
    auto issue = [&](int k) {
        const int buf = k & 1;
        const int64_t s0 = t0 + (int64_t)k * kBkSub;
        const int m = min(kBkSub, len - k * kBkSub);
        if (m == kBkSub && threadIdx.x == 0) {
            fence_proxy_async();
            mbar_expect_tx(&bar[buf], kBkSub * 10);
            bulk_g2s(sl + buf * kBkSub, a.keys + s0, kBkSub * 4, &bar[buf]);
            bulk_g2s(va + buf * kBkSub, a.vals + s0, kBkSub * 4, &bar[buf]);
            bulk_g2s(bn + buf * kBkSub, a.tbin + s0, kBkSub * 2, &bar[buf]);
        }
    };
    const bool bulk_ok = ((uintptr_t)(a.keys + t0) % 16) == 0 && ((uintptr_t)(a.vals + t0) % 16) == 0 &&
                         ((uintptr_t)(a.tbin + t0) % 16) == 0;
    unsigned phase[2] = {0u, 0u};
    if (bulk_ok) issue(0);
    for (int k = 0; k < nsub; ++k) {
        const int buf = k & 1;
        const int m = min(kBkSub, len - k * kBkSub);
        uint32_t* csl = sl + buf * kBkSub;
        int32_t* cva = va + buf * kBkSub;
        uint16_t* cbn = bn + buf * kBkSub;
        if (bulk_ok && m == kBkSub) {
            mbar_wait(&bar[buf], phase[buf]);
            phase[buf] ^= 1u;
        } else {
            const int64_t s0 = t0 + (int64_t)k * kBkSub;
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                csl[i] = a.keys[s0 + i];
                cva[i] = a.vals[s0 + i];
                cbn[i] = a.tbin[s0 + i];
            }
            __syncthreads();
        }
        // the next sub-tile's copies overlap this one (its buffer was last
        // read by sub-tile k-1, which ended with a barrier)
        if (bulk_ok && k + 1 < nsub) issue(k + 1);
        // stable sort of (bin << 12 | index) by bin: 2 x 7-bit digits
        auto k0 = [&](int it) -> uint32_t {
            return it < m ? (((uint32_t)cbn[it] << 12) | (uint32_t)it) : 0xffffffffu;
        };
        bk_lsd_pass<kBkThreads, kBkIPW>(nullptr, kb, 12, wh, k0);
        bk_lsd_pass<kBkThreads, kBkIPW>(kb, ka, 19, wh, k0);
        // runs of equal bins -> contiguous writes from the bin's cursor
        constexpr int Q = kBkSub / kBkThreads;
        uint32_t key[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int s = q * kBkThreads + threadIdx.x;
            key[q] = ka[s];
            if (s < m && (s == 0 || (ka[s - 1] >> 12) != (key[q] >> 12))) runst[key[q] >> 12] = (uint16_t)s;
        }
        __syncthreads();
        uint32_t newc[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int s = q * kBkThreads + threadIdx.x;
            newc[q] = 0xffffffffu;
            if (s >= m) continue;
            const uint32_t b = key[q] >> 12, it = key[q] & 4095u;
            const uint32_t rank = (uint32_t)s - runst[b];
            const uint32_t pos = cursor[b] + rank;
            const uint32_t g = csl[it];
            if (a.bin_hot[b]) {
                // batch rank `pos` of hot group g: stored iff among its kept suffix
                const int32_t drop = a.gcount[g] - a.gkept[g];
                if ((int32_t)pos >= drop) a.vout[a.gstart[g] + (int32_t)pos - drop] = cva[it];
            } else {
                a.skey[pos] = g;
                a.sval[pos] = cva[it];
            }
            if (s == m - 1 || (ka[s + 1] >> 12) != b) newc[q] = pos + 1;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if (newc[q] != 0xffffffffu) cursor[key[q] >> 12] = newc[q];
        __syncthreads();
    }
}

// pass 2: a cold bucket at a time (persistent CTAs, bins dealt by stride)
constexpr int kBkLocThreads = 512;
constexpr int kBkLocIPW = ((kBkCap + kBkLocThreads - 1) / kBkLocThreads) * 32;    // 768
struct BkLocSmem {
    static constexpr size_t ka = 0;                                          // u32[IPW * 16]
    static constexpr size_t kb = ka + (size_t)kBkLocIPW * 16 * 4;
    static constexpr size_t wh = kb + (size_t)kBkLocIPW * 16 * 4;            // u16[16][128]
    static constexpr size_t bytes = wh + (size_t)16 * 128 * 2;
};

__global__ void __launch_bounds__(kBkLocThreads, 2)
k_bk_local(BucketArgs a) { SS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char lsm[];
    uint32_t* ka = (uint32_t*)(lsm + BkLocSmem::ka);
    uint32_t* kb = (uint32_t*)(lsm + BkLocSmem::kb);
    uint16_t* wh = (uint16_t*)(lsm + BkLocSmem::wh);
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int nb = *a.n_bins;
    if (nb > kBkNBMax) return;
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
        if (a.bin_hot[b]) continue;
        const int m = (int)a.btot[b];
        if (m == 0) continue;
        const uint32_t g0 = (uint32_t)a.bin_first[b];
        const uint32_t span = (uint32_t)a.bin_first[b + 1] - g0;
        const uint32_t sb = a.sbase[b];
        const int32_t out0 = a.gstart[g0];
        if (span == 1) {
            // one group: staging order is the final order
            for (int i = threadIdx.x; i < m; i += blockDim.x) a.vout[out0 + i] = a.sval[sb + i];
            continue;
        }
        // key = (offset in bucket << 14) | staging index, padded to the
        // CTA's item count with keys that sort last
        for (int it = threadIdx.x; it < kBkLocIPW * (kBkLocThreads / 32); it += blockDim.x)
            ka[it] = it < m ? (((a.skey[sb + it] - g0) << 14) | (uint32_t)it) : 0xffffffffu;
        __syncthreads();
        auto none = [](int) -> uint32_t { return 0u; };
        const uint32_t* res;
        bk_lsd_pass<kBkLocThreads, kBkLocIPW>(ka, kb, 14, wh, none);
        res = kb;
        if (span > 128) {
            bk_lsd_pass<kBkLocThreads, kBkLocIPW>(kb, ka, 21, wh, none);
            res = ka;
        }
        for (int s = threadIdx.x; s < m; s += blockDim.x) a.vout[out0 + s] = a.sval[sb + (res[s] & 16383u)];
        __syncthreads();
    }
}

}  // namespace ss
