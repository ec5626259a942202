// partition.cuh -- K2 (count / partition histogram) and K3 (stable rank +
// placement) of the skewstream B200 pipeline.
//
// Reference behaviour (read-only, /root/reference/pkg/src/skewstream):
//   count_batch    partition.py:117-130  group_counts = bincount(groups),
//                                       tpt = bincount(g2t[groups]);
//                                       DataError names the first bad tuple
//   reorder_batch  partition.py:161-178  stable, thread-major, group-
//                                       contiguous placement
//   ingest_sequence engine.py:274-280   stable regroup preserving arrival order
//
// B200 design: a batch is counted once into per-chunk group histograms
// (shared memory per chunk for G <= 16K, else warp-aggregated atomics).
// The kept tuples are then placed stably by group: for G <= 2^14 in ONE
// pass (k_rank_place: a CTA per live chunk, group cursors in shared
// memory advanced in arrival order), otherwise by an LSD multisplit whose
// passes use decoupled look-back (one pass when G <= 2^11, two up to
// 2^22).  The stable placement gives every tuple its exact arrival rank
// inside its group as (position - group start), which is all the window
// update needs.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace ss {

constexpr int kScanBlk = 4096;   // groups per block in the G-sized scans
constexpr int kMaxBins = 2048;   // radix digit <= 11 bits
constexpr int kSortThreads = 512;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;   // 4096 tuples

// --------------------------------------------------------------------------
// K2: per-sub-batch group histogram.  `chunk` divides the sub-batch size S,
// so a CTA never straddles two sub-batches.
//   SMEM (G <= 16K): the whole histogram lives in shared memory.
//   else: groups that were hot in the previous batch (hot_of[g] >= 0, at
//   most kHotCache of them) are counted in shared memory, the cold tail
//   with warp-aggregated global atomics -- under Zipf skew the hottest
//   keys would otherwise serialise on one L2 slice.
// --------------------------------------------------------------------------
constexpr int kHotCache = 2048;

template <bool SMEM>
__global__ void __launch_bounds__(512)
k_count(const uint32_t* __restrict__ groups, int64_t n, uint32_t G, int64_t S, int64_t chunk,
        int32_t* __restrict__ gcnt, unsigned long long* __restrict__ bad, int vec_ok,
        const int32_t* __restrict__ hot_of, const int32_t* __restrict__ hot_g, int n_hot) { SS_PDL_ENTRY();
    extern __shared__ int32_t sh_hist[];
    const int64_t c0 = (int64_t)blockIdx.x * chunk;
    if (c0 >= n) return;
    const int64_t c1 = min(n, c0 + chunk);
    int32_t* dst = gcnt + (c0 / S) * (int64_t)G;
    const int nbins = SMEM ? (int)G : n_hot;
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
    const unsigned lane = lane_id();
    for (int64_t base = c0; base < c1; base += 4 * (int64_t)blockDim.x) {
        const int64_t i = base + 4 * (int64_t)threadIdx.x;
        uint32_t k[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
        if (i + 3 < c1 && vec_ok) {
            uint4 v = ld_stream_v4(groups + i);
            k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (i + q < c1) k[q] = groups[i + q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t g = k[q];
            const bool in = (i + q < c1);
            if (in && g >= G) {
                atomicMin(bad, (unsigned long long)(i + q));
                g = 0xffffffffu;
            }
            if (!in) g = 0xffffffffu;
            if (SMEM) {
                if (g != 0xffffffffu) atomicAdd(&sh_hist[g], 1);
            } else {
                const int h = (g != 0xffffffffu && n_hot) ? hot_of[g] : -1;
                if (h >= 0) {
                    atomicAdd(&sh_hist[h], 1);
                    g = 0xffffffffu;
                }
                // keys outside the hot cache: warp-aggregated (a hot key the
                // cache missed, e.g. after the skew drifts, still costs one
                // atomic per warp instead of one per lane)
                const unsigned peers = __match_any_sync(SS_FULL, g);
                if (g != 0xffffffffu && lane == 31u - __clz(peers)) atomicAdd(&dst[g], __popc(peers));
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) {
        const int32_t c = sh_hist[i];
        if (c) atomicAdd(&dst[SMEM ? i : hot_g[i]], c);
    }
}

// K2 for the fused step with G <= 16K: one CTA per count chunk of the batch
// (S = 2^k tuples) builds the chunk's whole histogram in shared memory and
// writes its row of gcnt with plain stores (no zeroing, no global atomics).
// Each thread keeps four 128-bit loads in flight; a warp's load instruction
// covers 512 contiguous bytes.
// histogram of groups[c0, c1) into shared memory (zeroed by the caller)
__device__ __forceinline__ void count_range(const uint32_t* __restrict__ groups, int64_t c0, int64_t c1, uint32_t G,
                                            int32_t* sh_hist, unsigned long long* __restrict__ bad, int vec_ok) {
    constexpr int U = 4;                         // 128-bit loads in flight per thread
    const int64_t step = (int64_t)U * 4 * blockDim.x;
    int64_t base = c0;
    if (vec_ok) {
        for (; base + step <= c1; base += step) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ld_stream_v4(groups + base + ((int64_t)u * blockDim.x + threadIdx.x) * 4);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t k[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (k[q] < G) atomicAdd(&sh_hist[k[q]], 1);
                    else atomicMin(bad, (unsigned long long)(base + ((int64_t)u * blockDim.x + threadIdx.x) * 4 + q));
                }
            }
        }
    }
    for (int64_t i = base + threadIdx.x; i < c1; i += blockDim.x) {
        const uint32_t g = groups[i];
        if (g < G) atomicAdd(&sh_hist[g], 1);
        else atomicMin(bad, (unsigned long long)i);
    }
}

__global__ void __launch_bounds__(512)
k_count_rows(const uint32_t* __restrict__ groups, int64_t n, uint32_t G, int64_t S, int32_t* __restrict__ gcnt,
             unsigned long long* __restrict__ bad, int vec_ok) { SS_PDL_ENTRY();
    extern __shared__ int32_t sh_hist[];
    const int64_t c0 = (int64_t)blockIdx.x * S;
    const int64_t c1 = min(n, c0 + S);
    for (int i = threadIdx.x; i < (int)G; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
    count_range(groups, c0, c1, G, sh_hist, bad, vec_ok);
    __syncthreads();
    int32_t* dst = gcnt + (int64_t)blockIdx.x * G;
    for (int i = threadIdx.x; i < (int)G; i += blockDim.x) dst[i] = sh_hist[i];
}

// The hot-group cache of the next batch's count: groups above `thr` in
// this batch (first kHotCache found).  hot_of is reset for the old list.
__global__ void __launch_bounds__(256)
k_hot_select(const int32_t* __restrict__ gcount, uint32_t G, long long thr, int32_t* __restrict__ hot_of,
             int32_t* __restrict__ hot_g, int* __restrict__ n_hot_dev, const unsigned long long* __restrict__ bad,
             int32_t* __restrict__ ent_words = nullptr, const int32_t* __restrict__ slot_ent = nullptr) { SS_PDL_ENTRY();
    if (*bad != (unsigned long long)kNoBad) return;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
        int h = -1;
        if (gcount[g] > thr) {
            const int slot = atomicAdd(n_hot_dev, 1);
            if (slot < kHotCache) {
                hot_g[slot] = (int32_t)g;
                h = slot;
            }
        }
        // int64 keys: the hot index also lives in the key's table entry
        // (word 3 of the 16-byte entry), read by the fused probe + count
        if (ent_words && hot_of[g] != h) ent_words[4 * (int64_t)slot_ent[g] + 3] = h;
        hot_of[g] = h;
    }
}

// --------------------------------------------------------------------------
// Batch statistics: gcount[g] = sum over chunks, tpt[pmap[g]] (the
// reference's count_batch outputs), the touched-group count and, for the
// fused step, the kept tuples of every group.
//
// A group's tuples in chunk c can never be stored when all of them precede
// the last W of the batch (pre_c + cnt_c <= K - W): their count is zeroed
// (the placement drops them without reading their attrs).  The kept tuples
// of a group are therefore a suffix of its batch tuples: gkept[g] of them,
// the first at batch rank K - gkept.  chunk_live[c] marks chunks with any
// kept tuple; the others are never read again.
// --------------------------------------------------------------------------
__device__ __forceinline__ void stats_account(uint32_t g, int32_t c, const int32_t* __restrict__ pmap,
                                              uint32_t* sh_tpt, const int32_t* __restrict__ fill, int64_t W,
                                              uint32_t& my_touched, unsigned long long& my_bytes,
                                              int P) {
    const int p = pmap[g];
    atomicAdd(&sh_tpt[p], (uint32_t)c);
    ++my_touched;
    // algorithmic bytes: stored values, retracted old values
    // that must be read, state + result row
    const int64_t f0 = fill[g];
    const int64_t stored = min64(c, W), retracted = c < W ? max64(0, f0 + c - W) : 0;
    my_bytes += 4ull * (unsigned long long)(stored + retracted) + 76ull;
    // window-update work of the partition (values moved + a per-group
    // overhead), for the work-proportional K4 grid
    atomicAdd(&sh_tpt[P + p], (uint32_t)min64(stored + retracted + 16, 0x3fffffff));
}

// Few chunks (<= 32): one thread per group, coalesced over consecutive
// groups; chunk_live is a bitmap (bit c of word c / 32).
constexpr int kMaxChunkWords = 4096 / 32;

// the CTA's touched-group and byte totals: one global atomic each per CTA
// (per warp, 2368 CTAs x 8 warps queued ~19K atomics on each of the two
// words at 1M groups); every thread of the CTA calls it
__device__ __forceinline__ void stats_flush(uint32_t my_touched, unsigned long long my_bytes,
                                            unsigned long long* touched, unsigned long long* alg_bytes) {
    __shared__ unsigned long long sh_t[32], sh_b[32];
    my_touched = warp_sum(my_touched);
    my_bytes = warp_sum(my_bytes);
    if (lane_id() == 0) {
        sh_t[warp_id()] = my_touched;
        sh_b[warp_id()] = my_bytes;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0, b = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
            t += sh_t[q];
            b += sh_b[q];
        }
        if (t) {
            atomicAdd(touched, t);
            atomicAdd(alg_bytes, b);
        }
    }
}

__global__ void __launch_bounds__(1024)
k_batch_stats(int32_t* __restrict__ gcnt, int n_chunk, uint32_t G, const int32_t* __restrict__ pmap,
              int P, int32_t* __restrict__ gcount, int32_t* __restrict__ gkept, uint32_t* __restrict__ chunk_live,
              unsigned long long* __restrict__ tpt, unsigned long long* __restrict__ touched,
              const unsigned long long* __restrict__ bad, const int32_t* __restrict__ fill, int64_t W,
              unsigned long long* __restrict__ alg_bytes, int nodrop, int32_t* __restrict__ gpre = nullptr,
              uint32_t* __restrict__ pwork = nullptr, int* __restrict__ any_dead = nullptr) { SS_PDL_ENTRY();
    extern __shared__ uint32_t sh_tpt[];     // per-CTA partial loads (< 2^31)
    __shared__ uint32_t sh_live[kMaxChunkWords];
    if (*bad != (unsigned long long)kNoBad) return;
    const int nwords = (n_chunk + 31) >> 5;
    for (int p = threadIdx.x; p < 2 * P; p += blockDim.x) sh_tpt[p] = 0;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) sh_live[i] = 0;
    __syncthreads();
    uint32_t my_touched = 0;
    unsigned long long my_bytes = 0;
    const unsigned lane = lane_id();
    uint32_t lbits = 0;                      // n_chunk <= 32 here
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
        int32_t c = 0;
        for (int s = 0; s < n_chunk; ++s) c += gcnt[(int64_t)s * G + g];
        gcount[g] = c;
        int32_t kept = c;
        if (c > W && gkept && !nodrop) {
            int32_t pre = 0;
            kept = 0;
            for (int s = 0; s < n_chunk; ++s) {
                const int64_t idx = (int64_t)s * G + g;
                const int32_t k = gcnt[idx];
                if (k) {
                    if ((int64_t)pre + k <= (int64_t)c - W) {
                        gcnt[idx] = 0;
                        if (any_dead) *any_dead = 1;
                    } else {
                        kept += k;
                        lbits |= 1u << s;
                    }
                }
                pre += k;
            }
        } else if (c) {
            for (int s = 0; s < n_chunk; ++s)
                if (gcnt[(int64_t)s * G + g]) lbits |= 1u << s;
        }
        if (gkept) gkept[g] = kept;
        if (gpre) {
            int32_t pre = 0;
            for (int s = 0; s < n_chunk; ++s) {
                const int64_t idx = (int64_t)s * G + g;
                const int32_t k = gcnt[idx];
                gpre[idx] = k ? pre : -1;
                pre += k;
            }
        }
        if (c) stats_account(g, c, pmap, sh_tpt, fill, W, my_touched, my_bytes, P);
    }
    lbits = __reduce_or_sync(SS_FULL, lbits);
    if (chunk_live && lane == 0 && lbits) atomicOr(&sh_live[0], lbits);
    stats_flush(my_touched, my_bytes, touched, alg_bytes);   // (ends with a CTA barrier)
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        if (sh_tpt[p]) atomicAdd(&tpt[p], (unsigned long long)sh_tpt[p]);
        if (pwork && sh_tpt[P + p]) atomicAdd(&pwork[p], sh_tpt[P + p]);
    }
    if (chunk_live)
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) {
            const uint32_t v = sh_live[i];
            if (v && (chunk_live[i] & v) != v) atomicOr(&chunk_live[i], v);
        }
}

// Many chunks (> 32): one CTA per 32 consecutive groups (lane = group), its
// warps over contiguous chunk ranges, so every gcnt access is a coalesced
// 128-byte row segment (a warp per group reading down a column touched 32
// sectors per request).  Per group: the chunk total and each warp's base
// (shared memory), the never-stored runs -- a prefix of the group's chunks,
// ending at the largest inclusive prefix <= K - W -- zeroed, then the kept
// prefix of every live chunk (gpre, -1 elsewhere) and the live-chunk bits.
// warps per CTA: 32 for small G (few CTAs, so more warps in flight each),
// 16 otherwise (measured: C1 G=1K 12 -> 9.8 us with 32; C2 G=10K 15 us
// with 16, slower with 32)
template <int kStatsWarps>
__global__ void __launch_bounds__(kStatsWarps * 32)
k_batch_stats_cols(int32_t* __restrict__ gcnt, int n_chunk, uint32_t G, const int32_t* __restrict__ pmap,
                   int P, int32_t* __restrict__ gcount, int32_t* __restrict__ gkept,
                   uint32_t* __restrict__ chunk_live, unsigned long long* __restrict__ tpt,
                   unsigned long long* __restrict__ touched, const unsigned long long* __restrict__ bad,
                   const int32_t* __restrict__ fill, int64_t W, unsigned long long* __restrict__ alg_bytes,
                   int nodrop, int32_t* __restrict__ gpre, uint32_t* __restrict__ pwork, int* __restrict__ any_dead) { SS_PDL_ENTRY();
    extern __shared__ uint32_t sh_tpt[];     // per-CTA partial loads (< 2^31), then partition work
    __shared__ uint32_t sh_live[kMaxChunkWords];
    __shared__ int32_t sh_part[kStatsWarps][32];
    __shared__ int32_t sh_dead[kStatsWarps][32];
    if (*bad != (unsigned long long)kNoBad) return;
    const int nwords = (n_chunk + 31) >> 5;
    for (int p = threadIdx.x; p < 2 * P; p += blockDim.x) sh_tpt[p] = 0;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) sh_live[i] = 0;
    const unsigned lane = lane_id(), w = warp_id();
    const int R = (n_chunk + kStatsWarps - 1) / kStatsWarps;
    const int c_lo = min(n_chunk, (int)w * R), c_hi = min(n_chunk, c_lo + R);
    uint32_t my_touched = 0;
    unsigned long long my_bytes = 0;
    for (uint32_t g0 = blockIdx.x * 32; g0 < G; g0 += gridDim.x * 32) {
        const uint32_t g = g0 + lane;
        const bool gv = g < G;
        const int32_t* col = gcnt + g;
        int32_t part = 0;
        if (gv) {
            int c = c_lo;
            for (; c + 8 <= c_hi; c += 8) {
                int32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = col[(int64_t)(c + u) * G];
#pragma unroll
                for (int u = 0; u < 8; ++u) part += v[u];
            }
            for (; c < c_hi; ++c) part += col[(int64_t)c * G];
        }
        sh_part[w][lane] = part;
        __syncthreads();
        int32_t C = 0, base = 0;
#pragma unroll
        for (int i = 0; i < kStatsWarps; ++i) {
            const int32_t v = sh_part[i][lane];
            base += (i < (int)w) ? v : 0;
            C += v;
        }
        const bool drop = gv && C > W && gkept && !nodrop;
        int32_t dmax = 0;
        if (drop) {
            int32_t pre = base;
            for (int c = c_lo; c < c_hi; ++c) {
                const int64_t idx = (int64_t)c * G + g;
                const int32_t k = gcnt[idx];
                if (k && (int64_t)pre + k <= (int64_t)C - W) {
                    gcnt[idx] = 0;
                    dmax = pre + k;
                    if (any_dead) *any_dead = 1;
                }
                pre += k;
            }
        }
        sh_dead[w][lane] = dmax;
        __syncthreads();
        int32_t D = 0;
#pragma unroll
        for (int i = 0; i < kStatsWarps; ++i) D = max(D, sh_dead[i][lane]);
        // kept prefix: the never-stored runs all precede every live one
        int32_t pre = base - min(D, base);
        for (int c = c_lo; c < c_hi; ++c) {
            const int64_t idx = (int64_t)c * G + g;
            const int32_t k = gv ? gcnt[idx] : 0;
            const bool live = k != 0;
            if (gpre && gv) gpre[idx] = live ? pre : -1;
            pre += k;
            const uint32_t bits = __ballot_sync(SS_FULL, live);
            if (chunk_live && bits && lane == 0) atomicOr(&sh_live[c >> 5], 1u << (c & 31));
        }
        if (w == 0 && gv) {
            gcount[g] = C;
            if (gkept) gkept[g] = C - D;
            if (C) stats_account(g, C, pmap, sh_tpt, fill, W, my_touched, my_bytes, P);
        }
        __syncthreads();                         // sh_part / sh_dead reused
    }
    stats_flush(my_touched, my_bytes, touched, alg_bytes);   // (ends with a CTA barrier)
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        if (sh_tpt[p]) atomicAdd(&tpt[p], (unsigned long long)sh_tpt[p]);
        if (pwork && sh_tpt[P + p]) atomicAdd(&pwork[p], sh_tpt[P + p]);
    }
    if (chunk_live)
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) {
            const uint32_t v = sh_live[i];
            if (v && (chunk_live[i] & v) != v) atomicOr(&chunk_live[i], v);
        }
}

// --------------------------------------------------------------------------
// G-sized exclusive scan of the per-sub-batch group histograms -> run
// starts gstart[s][g], plus the radix digit histograms of every pass.
// grid = (ceil(G / kScanBlk), n_sub), block = 1024 (4 groups per thread).
// --------------------------------------------------------------------------
struct DigitPlan {
    int npass;
    int shift[2];
    int bits[2];   // digit width actually ranked (instantiated width may be larger)
};

__global__ void __launch_bounds__(1024)
k_scan_reduce(const int32_t* __restrict__ gcnt, uint32_t G, int32_t* __restrict__ bsum, int nblk,
              DigitPlan plan, uint32_t* __restrict__ dhist, const unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    __shared__ uint32_t sh_dh[2][kMaxBins];
    __shared__ int32_t sh_red[33];
    if (*bad != (unsigned long long)kNoBad) return;
    const int s = blockIdx.y;
    const int32_t* row = gcnt + (int64_t)s * G;
    for (int i = threadIdx.x; i < 2 * kMaxBins; i += blockDim.x) (&sh_dh[0][0])[i] = 0;
    __syncthreads();
    const uint32_t g0 = blockIdx.x * kScanBlk + 4 * threadIdx.x;
    int32_t c[4];
    int32_t tsum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        c[q] = (g0 + q < G) ? row[g0 + q] : 0;
        tsum += c[q];
    }
    for (int d = 0; d < plan.npass; ++d) {
        const uint32_t mask = (1u << plan.bits[d]) - 1u;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (c[q]) atomicAdd(&sh_dh[d][((g0 + q) >> plan.shift[d]) & mask], (uint32_t)c[q]);
    }
    int32_t total;
    block_excl_scan(tsum, sh_red, &total);
    if (threadIdx.x == 0) bsum[(int64_t)s * nblk + blockIdx.x] = total;
    __syncthreads();
    for (int d = 0; d < plan.npass; ++d) {
        const int bins = 1 << plan.bits[d];
        uint32_t* out = dhist + ((int64_t)s * 2 + d) * kMaxBins;
        for (int b = threadIdx.x; b < bins; b += blockDim.x)
            if (sh_dh[d][b]) atomicAdd(&out[b], sh_dh[d][b]);
    }
}

// exclusive scan of the block sums (<= 1024 blocks) and of each pass's
// digit histogram -> digit bases.  grid = n_sub, block = 1024.  Block 0 also
// compacts the live-chunk flags into the ordered live-chunk list the first
// placement pass walks (and clears the flags for the next batch).
__global__ void __launch_bounds__(1024)
k_scan_top(int32_t* __restrict__ bsum, int nblk, DigitPlan plan, uint32_t* __restrict__ dhist,
           const unsigned long long* __restrict__ bad, int32_t* __restrict__ n_live,
           uint32_t* __restrict__ chunk_live = nullptr, int n_chunk = 0, int32_t* __restrict__ lc = nullptr,
           int32_t* __restrict__ n_lc = nullptr, int32_t* __restrict__ btile = nullptr,
           uint32_t* __restrict__ ep_dev = nullptr) { SS_PDL_ENTRY();
    __shared__ int32_t sh_red[33];
    __shared__ uint32_t sh_ured[33];
    if (ep_dev && blockIdx.x == 0 && threadIdx.x == 0) *ep_dev = epoch_next(*ep_dev);
    if (*bad != (unsigned long long)kNoBad) return;
    const int s = blockIdx.x;
    {
        int32_t v = (threadIdx.x < (unsigned)nblk) ? bsum[(int64_t)s * nblk + threadIdx.x] : 0;
        int32_t tot;
        int32_t ex = block_excl_scan(v, sh_red, &tot);
        if (threadIdx.x < (unsigned)nblk) bsum[(int64_t)s * nblk + threadIdx.x] = ex;
        if (threadIdx.x == 0 && n_live) n_live[s] = tot;
    }
    for (int d = 0; d < plan.npass; ++d) {
        uint32_t* h = dhist + ((int64_t)s * 2 + d) * kMaxBins;
        // 2048 bins, 2 per thread
        uint32_t a = h[2 * threadIdx.x], b = h[2 * threadIdx.x + 1];
        uint32_t tot;
        uint32_t ex = block_excl_scan(a + b, sh_ured, &tot);
        h[2 * threadIdx.x] = ex;
        h[2 * threadIdx.x + 1] = ex + a;
        if (d == 0 && btile && plan.npass == 2) {
            // tiles of the second pass: each first-pass digit bucket is cut
            // into 4096-tuple tiles of its own (SortSeg mode 2)
            const int32_t ta = (int32_t)((a + kSortTile - 1) / kSortTile);
            const int32_t tb = (int32_t)((b + kSortTile - 1) / kSortTile);
            int32_t ttot;
            const int32_t tex = block_excl_scan(ta + tb, sh_red, &ttot);
            btile[2 * threadIdx.x] = tex;
            btile[2 * threadIdx.x + 1] = tex + ta;
            if (threadIdx.x == 0) btile[kMaxBins] = ttot;
        }
    }
    if (chunk_live && s == 0) {
        // n_chunk <= 4 * 1024, 4 consecutive chunks per thread
        int32_t f[4], mine = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = 4 * threadIdx.x + q;
            f[q] = (c < n_chunk) ? (int32_t)((chunk_live[c >> 5] >> (c & 31)) & 1u) : 0;
            mine += f[q] ? 1 : 0;
        }
        int32_t tot;
        int32_t ex = block_excl_scan(mine, sh_red, &tot);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = 4 * threadIdx.x + q;
            if (f[q]) lc[ex++] = c;

        }
        if (threadIdx.x == 0) *n_lc = tot;
        __syncthreads();                         // every bit read before the words are cleared
        for (int i = threadIdx.x; i < (n_chunk + 31) / 32; i += blockDim.x) chunk_live[i] = 0;
    }
}

// k_scan_reduce + k_scan_top + k_scan_down in one CTA for G <= 16384 (16
// groups per thread): run starts, digit bases of every pass, the kept total,
// second-pass bucket tiles and the live-chunk list.
constexpr int kScanSmallG = 16384;

__global__ void __launch_bounds__(1024)
k_scan_small(const int32_t* __restrict__ row, uint32_t G, DigitPlan plan, uint32_t* __restrict__ dhist,
             int32_t* __restrict__ gstart, const unsigned long long* __restrict__ bad, int32_t* __restrict__ n_live,
             uint32_t* __restrict__ chunk_live, int n_chunk, int32_t* __restrict__ lc, int32_t* __restrict__ n_lc,
             int32_t* __restrict__ btile, uint32_t* __restrict__ ep_dev, int* __restrict__ sub_shift_dev = nullptr) { SS_PDL_ENTRY();
    __shared__ uint32_t sh_dh[2][kMaxBins];
    __shared__ int32_t sh_red[33];
    __shared__ uint32_t sh_ured[33];
    if (ep_dev && threadIdx.x == 0) *ep_dev = epoch_next(*ep_dev);
    if (*bad != (unsigned long long)kNoBad) return;
    for (int i = threadIdx.x; i < 2 * kMaxBins; i += blockDim.x) (&sh_dh[0][0])[i] = 0;
    __syncthreads();
    constexpr int GPT = kScanSmallG / 1024;
    const uint32_t g0 = threadIdx.x * GPT;
    int32_t c[GPT];
    int32_t tsum = 0;
    // each thread owns GPT consecutive groups: 128-bit loads and stores
    // when the whole run is in range (row and gstart are 16-byte aligned)
    const bool vec = g0 + GPT <= G;
    if (vec) {
#pragma unroll
        for (int q = 0; q < GPT; q += 4) {
            const int4 v = *reinterpret_cast<const int4*>(row + g0 + q);
            c[q] = v.x; c[q + 1] = v.y; c[q + 2] = v.z; c[q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < GPT; ++q) c[q] = (g0 + q < G) ? row[g0 + q] : 0;
    }
#pragma unroll
    for (int q = 0; q < GPT; ++q) tsum += c[q];
    for (int d = 0; d < plan.npass; ++d) {
        const uint32_t mask = (1u << plan.bits[d]) - 1u;
#pragma unroll
        for (int q = 0; q < GPT; ++q)
            if (c[q]) atomicAdd(&sh_dh[d][((g0 + q) >> plan.shift[d]) & mask], (uint32_t)c[q]);
    }
    int32_t total;
    int32_t ex = block_excl_scan(tsum, sh_red, &total);
    if (vec) {
#pragma unroll
        for (int q = 0; q < GPT; q += 4) {
            int4 v;
            v.x = ex; ex += c[q];
            v.y = ex; ex += c[q + 1];
            v.z = ex; ex += c[q + 2];
            v.w = ex; ex += c[q + 3];
            *reinterpret_cast<int4*>(gstart + g0 + q) = v;
        }
    } else {
#pragma unroll
        for (int q = 0; q < GPT; ++q) {
            if (g0 + q < G) gstart[g0 + q] = ex;
            ex += c[q];
        }
    }
    if (threadIdx.x == 0) *n_live = total;
    __syncthreads();
    for (int d = 0; d < plan.npass; ++d) {
        uint32_t* h = dhist + (int64_t)d * kMaxBins;
        const uint32_t a = sh_dh[d][2 * threadIdx.x], b = sh_dh[d][2 * threadIdx.x + 1];
        uint32_t tot;
        const uint32_t e2 = block_excl_scan(a + b, sh_ured, &tot);
        h[2 * threadIdx.x] = e2;
        h[2 * threadIdx.x + 1] = e2 + a;
        if (d == 0 && btile && plan.npass == 2) {
            const int32_t ta = (int32_t)((a + kSortTile - 1) / kSortTile);
            const int32_t tb = (int32_t)((b + kSortTile - 1) / kSortTile);
            int32_t ttot;
            const int32_t tex = block_excl_scan(ta + tb, sh_red, &ttot);
            btile[2 * threadIdx.x] = tex;
            btile[2 * threadIdx.x + 1] = tex + ta;
            if (threadIdx.x == 0) btile[kMaxBins] = ttot;
        }
    }
    if (chunk_live) {
        int32_t f[4], mine = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int ch = 4 * threadIdx.x + q;
            f[q] = (ch < n_chunk) ? (int32_t)((chunk_live[ch >> 5] >> (ch & 31)) & 1u) : 0;
            mine += f[q] ? 1 : 0;
        }
        int32_t tot;
        int32_t e3 = block_excl_scan(mine, sh_red, &tot);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int ch = 4 * threadIdx.x + q;
            if (f[q]) lc[e3++] = ch;

        }
        if (threadIdx.x == 0) {
            *n_lc = tot;
            if (sub_shift_dev) {
                // sub-chunks until the live units fill two CTAs per SM
                // (only with fewer live chunks than half the SMs: at C2 all
                // 256 chunks are live, and 2 sub-chunks each cost more in
                // the extra count and cursor set-up than the finer grid won)
                int ssh = 0;
                while (tot > 0 && tot < kNumSM / 2 && (tot << ssh) < 2 * kNumSM && ssh < 4) ++ssh;
                *sub_shift_dev = ssh;
            }
        }
        __syncthreads();                         // every bit read before the words are cleared
        for (int i = threadIdx.x; i < (n_chunk + 31) / 32; i += blockDim.x) chunk_live[i] = 0;
    }
}

// block-local exclusive scan + block base -> gstart[s][g]
__global__ void __launch_bounds__(1024)
k_scan_down(const int32_t* __restrict__ gcnt, uint32_t G, const int32_t* __restrict__ bsum, int nblk,
            int32_t* __restrict__ gstart, const unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    __shared__ int32_t sh_red[33];
    if (*bad != (unsigned long long)kNoBad) return;
    const int s = blockIdx.y;
    const int32_t* row = gcnt + (int64_t)s * G;
    int32_t* out = gstart + (int64_t)s * G;
    const uint32_t g0 = blockIdx.x * kScanBlk + 4 * threadIdx.x;
    int32_t c[4], tsum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        c[q] = (g0 + q < G) ? row[g0 + q] : 0;
        tsum += c[q];
    }
    int32_t total;
    int32_t ex = block_excl_scan(tsum, sh_red, &total) + bsum[(int64_t)s * nblk + blockIdx.x];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (g0 + q < G) out[g0 + q] = ex;
        ex += c[q];
    }
}

// --------------------------------------------------------------------------
// K3: one stable LSD multisplit pass with decoupled look-back.
//
// A tile of 4096 tuples is ranked warp by warp: each of the 16 warps owns
// 256 consecutive tuples held warp-striped (item j of lane l = tuple
// j*32+l) and ranks them in arrival order with __match_any_sync against a
// per-warp digit histogram.  Per-bin prefixes across warps, across bins
// of the tile, across earlier tiles (look-back on [epoch|flag|count] words)
// and across lower digits (bin base) give the output position.  The tile
// is first sorted in shared memory, so the global writes are contiguous
// runs per digit.  Tile ids come from an atomic ticket so a tile only ever
// waits on tiles that are already resident.
// --------------------------------------------------------------------------
// Where a placement tile's bin bases come from.  Long look-back chains
// (every in-flight tile walking back to the last finished one) are avoided
// by cutting the tile sequence into segments whose bin bases are known in
// advance: the first tile of a segment publishes its inclusive prefix at
// once, later tiles look back only inside their segment.
//   mode 0: one segment (bin_base), tiles = the input in 4096-tuple steps
//   mode 1: first pass of the fused step -- segments = live count chunks,
//           bases from the per-chunk digit histograms (k_chunk_hist/scan)
//   mode 2: second pass -- segments = the first pass's digit buckets; the
//           base of bin d in bucket b is the run start of group (d<<b0)|b
struct SortSeg {
    int mode;
    const int32_t* live;        // mode 1: kept counts [n_chunk][G]
    const int32_t* lc;          // mode 1: ordered live chunks
    const int32_t* n_lc;
    int chunk_shift;
    uint32_t G;
    const uint32_t* cbase;      // mode 1: [n_lc][BINS]
    const int32_t* btile;       // mode 2: tile prefix over buckets [nb + 1]
    const uint32_t* bpos;       // mode 2: bucket starts (previous pass's exclusive bases)
    int nb;
    int b0;
    const int32_t* gstart;      // mode 2: run start of every group
    const int* any_dead;        // mode 1: 0 = no tuple of the batch is dropped (skip the kept lookups)
};

// per-live-chunk histogram of the first digit over the kept counts.
// grid = (n_chunk, slices): each CTA bins a slice of the chunk's groups in
// shared memory and adds it to H0 (zeroed before the launch)
__global__ void __launch_bounds__(1024)
k_chunk_hist(const int32_t* __restrict__ gcnt, uint32_t G, const int32_t* __restrict__ lc,
             const int32_t* __restrict__ n_lc, uint32_t m0, int nb, uint32_t* __restrict__ H0,
             const unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    extern __shared__ uint32_t sh_h[];
    if (*bad != (unsigned long long)kNoBad) return;
    const int i = blockIdx.x;
    if (i >= *n_lc) return;
    const int64_t c = lc[i];
    for (int d = threadIdx.x; d < nb; d += blockDim.x) sh_h[d] = 0;
    __syncthreads();
    const int32_t* row = gcnt + c * (int64_t)G;
    const uint32_t per = (G + gridDim.y - 1) / gridDim.y;
    const uint32_t g0 = blockIdx.y * per, g1 = min(G, g0 + per);
    for (uint32_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) {
        const int32_t v = row[g];
        if (v) atomicAdd(&sh_h[g & m0], (uint32_t)v);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nb; d += blockDim.x)
        if (sh_h[d]) atomicAdd(&H0[(int64_t)i * nb + d], sh_h[d]);
}

// per digit: exclusive scan of the live chunks' histograms + the bin base
// -> cbase[i][d].  A warp per digit, lanes over chunks.
__global__ void __launch_bounds__(1024)
k_chunk_scan(const uint32_t* __restrict__ H0, const int32_t* __restrict__ n_lc, int nb,
             const uint32_t* __restrict__ bin_base, uint32_t* __restrict__ cbase,
             const unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    if (*bad != (unsigned long long)kNoBad) return;
    const int d = blockIdx.x * (blockDim.x >> 5) + warp_id();
    if (d >= nb) return;
    const int nl = *n_lc;
    const unsigned lane = lane_id();
    uint32_t carry = bin_base[d];
    for (int i0 = 0; i0 < nl; i0 += 32) {
        const int i = i0 + (int)lane;
        const uint32_t v = (i < nl) ? H0[(int64_t)i * nb + d] : 0u;
        const uint32_t incl = warp_incl_scan(v);
        if (i < nl) cbase[(int64_t)i * nb + d] = carry + incl - v;
        carry += __shfl_sync(SS_FULL, incl, 31);
    }
}

#ifdef SS_SORT_PROF
__device__ unsigned long long g_sort_prof[8];
#endif

template <int RB>
struct SortSmem {
    static constexpr int BINS = 1 << RB;
    static constexpr int NW = kSortThreads / 32;
    // two input stages of keys + values (the current one doubles as the
    // tile-local sort buffer), per-warp digit histograms, bin starts/bases
    static constexpr size_t bytes = (size_t)2 * kSortTile * 8 + (size_t)NW * BINS * 2 + (size_t)BINS * 8 + 16;
};

template <int RB, bool MAPPED = false>
__global__ void __launch_bounds__(kSortThreads, 2)
k_sort_pass(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
            uint32_t* __restrict__ kout, int32_t* __restrict__ vout, int n, int shift, uint32_t mask,
            const uint32_t* __restrict__ bin_base, unsigned long long* __restrict__ status,
            const uint32_t* __restrict__ ep_dev, uint32_t ep_off, uint32_t* __restrict__ ticket,
            const unsigned long long* __restrict__ bad,
            int stream_in, const int32_t* __restrict__ dmap = nullptr,
            const int32_t* __restrict__ n_dev = nullptr, SortSeg seg = SortSeg{}) { SS_PDL_ENTRY();
    constexpr int BINS = 1 << RB;
    constexpr int NW = kSortThreads / 32;
    constexpr int BPT = (BINS + kSortThreads - 1) / kSortThreads;   // bins owned per thread
    extern __shared__ __align__(16) unsigned char sort_sm[];
    uint32_t* in_k = (uint32_t*)sort_sm;                     // [2][TILE] staged keys
    int32_t* in_v = (int32_t*)(in_k + 2 * kSortTile);        // [2][TILE] staged values
    uint32_t* tbin = (uint32_t*)(in_v + 2 * kSortTile);      // [BINS] tile-local bin start
    uint32_t* gbase = tbin + BINS;                           // [BINS] global pos of local pos 0
    uint16_t* whist = (uint16_t*)(gbase + BINS);             // [NW][BINS]
    __shared__ uint32_t sh_red[33];
    __shared__ int64_t sh_t0[2];
    __shared__ int sh_tn[2], sh_k[2], sh_seg[2];
    __shared__ uint32_t sh_tile[2];
    if (*bad != (unsigned long long)kNoBad) return;
    if (n_dev && *n_dev == 0) return;            // nothing kept in this batch
    // look-back words are tagged with a device-side epoch (bumped once per
    // placement by the scan kernel), so status memory is never cleared and
    // a captured CUDA graph can be replayed unchanged
    const uint32_t epoch = *ep_dev + ep_off;
    if (n_dev && seg.mode != 1) n = *n_dev;      // consumes a compacted (kept-only) input
    const unsigned w = warp_id(), lane = lane_id();
    const int wbase = (int)w * 32 * kSortItems;
    // nothing dropped in this batch (no group above W): every staged tuple is kept
    const bool no_dead = seg.mode == 1 && seg.any_dead && *seg.any_dead == 0;
    // second-pass bucket tile prefix, searched by every claim: staged in
    // shared memory once per CTA
    __shared__ int32_t sh_btile[kMaxBins + 1];
    if (seg.mode == 2)
        for (int i = threadIdx.x; i <= seg.nb; i += kSortThreads) sh_btile[i] = seg.btile[i];
    // claim a tile (thread 0): ticket -> input range and segment.  The
    // ticket's atomic is issued one phase before its result is needed.
    auto claim = [&](int slot, uint32_t t) {
        int64_t t0 = -1;
        int tn = 0, k = 0, sg = 0;
        if (seg.mode == 1) {
            // ticket t is tile (t mod tpc) of the (t / tpc)-th live chunk
            const int tpc_shift = seg.chunk_shift - 12;          // kSortTile = 2^12
            const int ci = (int)(t >> tpc_shift);
            if (ci < *seg.n_lc) {
                k = (int)(t & ((1u << tpc_shift) - 1u));
                t0 = ((int64_t)seg.lc[ci] << seg.chunk_shift) + ((int64_t)k << 12);
                sg = ci;
                if (t0 >= n) t0 = -1;                             // past a short last chunk
            }
        } else if (seg.mode == 2) {
            if ((int)t < sh_btile[seg.nb]) {
                int lo2 = 0, hi2 = seg.nb - 1;                     // last bucket with btile <= t
                while (lo2 < hi2) {
                    const int mid = (lo2 + hi2 + 1) >> 1;
                    if (sh_btile[mid] <= (int)t) lo2 = mid; else hi2 = mid - 1;
                }
                sg = lo2;
                k = (int)t - sh_btile[lo2];
                const int64_t bend = (lo2 + 1 < seg.nb) ? (int64_t)seg.bpos[lo2 + 1] : (int64_t)n;
                t0 = (int64_t)seg.bpos[lo2] + ((int64_t)k << 12);
                tn = (int)min64(kSortTile, bend - t0);
            }
        } else {
            k = (int)t;
            t0 = (int64_t)t * kSortTile;
            if (t0 >= n) t0 = -1;
        }
        if (seg.mode != 2 && t0 >= 0) tn = (int)min64(kSortTile, (int64_t)n - t0);
        sh_tile[slot] = t;
        sh_t0[slot] = t0;
        sh_tn[slot] = tn;
        sh_k[slot] = k;
        sh_seg[slot] = sg;
    };
    // stage a tile's keys and values into shared memory with cp.async: the
    // next tile's loads are in flight while the current tile is ranked
    auto stage = [&](int slot) {
        const int64_t t0 = sh_t0[slot];
        const int tn = sh_tn[slot];
        if (t0 >= 0) {
            uint32_t* dk = in_k + slot * kSortTile;
            int32_t* dv = in_v + slot * kSortTile;
#pragma unroll
            for (int j = 0; j < kSortItems; ++j) {
                const int li = wbase + j * 32 + (int)lane;
                if (li < tn) {
                    cp_async4(dk + li, kin + t0 + li);
                    cp_async4(dv + li, vin + t0 + li);
                }
            }
        }
        cp_async_commit();
    };
    const int32_t* live = nullptr;
    // persistent CTAs: tiles are taken by atomic ticket in arrival order, so
    // a tile only ever looks back at tiles that are already being processed
    // (the prefetched ticket is always newer than the one being processed)
    for (int i = threadIdx.x; i < NW * BINS / 2; i += kSortThreads) ((uint32_t*)whist)[i] = 0;
    __syncthreads();                             // sh_btile, zeroed histograms
    if (threadIdx.x == 0) claim(0, atomicAdd(ticket, 1u));
    __syncthreads();
    stage(0);
    int cur = 0;
    while (true) {
#ifdef SS_SORT_PROF
    long long _pt = clock64();
#define SS_PT(i) do { if (threadIdx.x == 0) { const long long _n = clock64(); atomicAdd(&g_sort_prof[i], (unsigned long long)(_n - _pt)); _pt = _n; } } while (0)
#else
#define SS_PT(i) do {} while (0)
#endif
    const uint32_t tile = sh_tile[cur];
    const int64_t tile0 = sh_t0[cur];            // input offset of this tile
    if (tile0 < 0) break;                        // beyond the tiles: nobody looks back at it
    const int tile_n = sh_tn[cur];
    const int seg_k = sh_k[cur];                 // index of the tile inside its segment
    const int seg_id = sh_seg[cur];
    uint32_t t_next = 0;
    if (threadIdx.x == 0) t_next = atomicAdd(ticket, 1u);   // consumed after the ranking
    // (the warp histograms were zeroed at the end of the previous tile)
    SS_PT(0);
    cp_async_wait_0();                           // this thread's copies of the current tile have landed
    uint32_t* skey = in_k + cur * kSortTile;     // staged input, then the tile-local sort buffer
    int32_t* sval = in_v + cur * kSortTile;
    if (seg.mode == 1 && !no_dead) live = seg.live + (int64_t)seg.lc[seg_id] * seg.G;   // the chunk's kept counts
    uint16_t* myh = whist + w * BINS;

    uint32_t key[kSortItems];
    int32_t val[kSortItems];
    uint32_t rank[kSortItems];
    uint32_t ok = 0;                             // bit j: item j is valid (and live)
    // keys and values come from the staged tile; the kept-count lookups are
    // all in flight together
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int li = wbase + j * 32 + (int)lane;
        key[j] = (li < tile_n) ? skey[li] : 0xffffffffu;
    }
    int32_t lv[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int li = wbase + j * 32 + (int)lane;
        lv[j] = (li < tile_n) ? 1 : 0;
        if (live && li < tile_n) lv[j] = __ldg(live + key[j]);
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int li = wbase + j * 32 + (int)lane;
        val[j] = 0;
        if (lv[j] > 0) {
            val[j] = sval[li];
            ok |= 1u << j;
        }
    }
    const unsigned lt = lanemask_lt();
    SS_PT(1);
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const bool valid = (ok >> j) & 1u;
        const uint32_t d = valid ? (MAPPED ? (uint32_t)dmap[key[j]] : ((key[j] >> shift) & mask)) : 0xffffffffu;
        const unsigned peers = __match_any_sync(SS_FULL, d);
        uint32_t r = 0;
        if (valid) r = myh[d];
        __syncwarp();
        if (valid) {
            rank[j] = r + __popc(peers & lt);
            if (lane == 31u - __clz(peers)) myh[d] = (uint16_t)(r + __popc(peers));
        }
        __syncwarp();
    }
    if (threadIdx.x == 0) claim(cur ^ 1, t_next);
    __syncthreads();
    stage(cur ^ 1);                              // next tile's loads overlap the rest of this one
    SS_PT(2);
    // per owned bin: exclusive prefix across warps and the tile total
    uint32_t tot[BPT];
    uint32_t tsum = 0;
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int b = threadIdx.x * BPT + q;
        tot[q] = 0;
        if (b < BINS) {
            uint32_t run = 0;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww) {
                const uint32_t c = whist[ww * BINS + b];
                whist[ww * BINS + b] = (uint16_t)run;
                run += c;
            }
            tot[q] = run;
            st_relaxed_u64(&status[(int64_t)tile * BINS + b],
                           lb_pack(epoch, seg_k == 0 ? kFlagInc : kFlagAgg, run));
        }
        tsum += tot[q];
    }
    // tile-local bin starts (bins are owned contiguously, so one block scan)
    uint32_t ttot;
    uint32_t lex = block_excl_scan_nt(tsum, sh_red, &ttot);   // sh_red is next used after the look-back barrier
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int b = threadIdx.x * BPT + q;
        if (b < BINS) tbin[b] = lex;
        lex += tot[q];
    }
    // look-back across tiles
    SS_PT(3);
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int b = threadIdx.x * BPT + q;
        if (b < BINS) {
            uint32_t excl = 0;
            if (seg_k > 0) {
                // windowed look-back: the status words of up to kLB
                // predecessors are loaded together, summed from the nearest
                // back to the first inclusive prefix; an unpublished word
                // restarts the window at that tile
                constexpr int kLB = 4;
                int64_t t = (int64_t)tile - 1;
                while (true) {
                    unsigned long long v[kLB];
#pragma unroll
                    for (int k = 0; k < kLB; ++k)
                        v[k] = (t - k >= 0) ? ld_relaxed_u64(&status[(t - k) * BINS + b]) : 0ull;
                    bool done = false;
                    int used = 0;
#pragma unroll
                    for (int k = 0; k < kLB; ++k) {
                        if (done || used < k) continue;             // stopped earlier in the window
                        const uint32_t ep = (uint32_t)(v[k] >> 34);
                        const unsigned long long fl = (v[k] >> 32) & 3ull;
                        if (t - k < 0 || ep != epoch || fl == 0) continue;   // not published yet
                        excl += (uint32_t)v[k];
                        used = k + 1;
                        if (fl == kFlagInc) done = true;
                    }
                    if (done) break;
                    t -= used;
                }
                st_relaxed_u64(&status[(int64_t)tile * BINS + b], lb_pack(epoch, kFlagInc, excl + tot[q]));
            }
            uint32_t base;
            if (seg.mode == 1) base = seg.cbase[(int64_t)seg_id * BINS + b];
            else if (seg.mode == 2) {
                const uint32_t g = ((uint32_t)b << seg.b0) | (uint32_t)seg_id;
                base = (g < seg.G) ? (uint32_t)seg.gstart[g] : 0u;
            } else base = bin_base[b];
            gbase[b] = base + excl - tbin[b];
        }
    }
    __syncthreads();
    SS_PT(4);
    // tile-local sort into shared memory
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        if ((ok >> j) & 1u) {
            const uint32_t d = MAPPED ? (uint32_t)dmap[key[j]] : ((key[j] >> shift) & mask);
            const uint32_t lp = tbin[d] + myh[d] + rank[j];
            skey[lp] = key[j];
            sval[lp] = val[j];
        }
    }
    __syncthreads();
    // contiguous runs per digit to global memory
    const uint32_t tlive = ttot;                 // live items of the tile
    // the warp histograms are not read again in this tile: each warp zeroes
    // its own for the next one (no barrier needed before its next ranking)
    for (int i = lane; i < BINS / 2; i += 32) ((uint32_t*)myh)[i] = 0;
    __syncwarp();
    for (int i = threadIdx.x; i < (int)tlive; i += kSortThreads) {
        const uint32_t k = skey[i];
        const uint32_t pos = gbase[MAPPED ? (uint32_t)dmap[k] : ((k >> shift) & mask)] + (uint32_t)i;
        if (MAPPED && !vout) {
            // multi-GPU route: one 8-byte (group, attr) record per tuple, the
            // message the all-to-all ships
            reinterpret_cast<uint2*>(kout)[pos] = make_uint2(k, (uint32_t)sval[i]);
        } else {
            vout[pos] = sval[i];
            if (kout) kout[pos] = k;
        }
    }
    // no closing barrier: everything this tile reads (staging buffer, gbase,
    // tile slots) is rewritten only after the next tile's post-ranking
    // barrier, which every thread reaches after finishing this tile
    SS_PT(5);
    cur ^= 1;
    }
    cp_async_wait_0();
}

// --------------------------------------------------------------------------
// Single-pass placement for small group domains (G <= kRankMaxG): the
// per-group output cursors of one count chunk fit in shared memory, so a
// chunk's kept tuples are placed by ONE CTA walking the chunk in order --
// no radix passes, no cross-tile look-back.
//
// Cursor of group g in live chunk c: gstart[g] + gpre[c][g], where gpre is
// the exclusive prefix of g's kept counts over the chunks before c (written
// by k_batch_stats; -1 marks a never-stored (c, g) run, whose tuples are
// dropped).  The chunk is cut into sub-tiles of kRankSub tuples dealt
// round-robin to the warps; each warp ranks its sub-tile with
// __match_any_sync and advances the shared cursors by one leader atomic per
// distinct group and round.  The cursor updates are passed from warp to
// warp in sub-tile order through named barriers (warp w waits on barrier
// 1 + w, arrived at by the warp holding the previous sub-tile), so every
// group's tuples get consecutive positions in arrival order; loads (a
// 3-deep cp.async ring per warp), matching and the scattered stores of the
// other warps run outside that chain.
// --------------------------------------------------------------------------
constexpr int kRankWarps = 16;                     // one named barrier per warp (ids 0..15)
constexpr int kRankItems = 8;
constexpr int kRankSub = 32 * kRankItems;          // tuples per sub-tile
constexpr int kRankStages = 2;
constexpr int kRankMaxG = 16384;
#ifndef SS_RANK_BALLOT
#define SS_RANK_BALLOT 2
#endif
// of every 4 rounds, how many match keys by ballots (ALU) -- the rest use
// MATCH (MIO pipe), so both pipes share the ranking (measured at C2: 142 us
// with 2 of 4, against 162 all-ballot and 168 all-MATCH)
constexpr int kRankBallot = SS_RANK_BALLOT;

// Sub-chunk prefixes for the single-pass placement when few chunks are
// live: k_scan_small picks ss (live chunks x 2^ss >= 2 x 148, ss <= 4);
// k_sub_hist counts every live sub-chunk's keys, k_sub_scan turns them into
// gsub[u][g] = gpre[c][g] + g's count in the chunk's earlier sub-chunks
// (-1 for a never-stored run).  Unit u = live chunk index << ss | sub-chunk.
constexpr int kSubUnitsMax = 2 * 2 * kNumSM;        // (n_lc << ss) < 2 x 296

__global__ void __launch_bounds__(512)
k_sub_hist(const uint32_t* __restrict__ keys, int64_t n, int chunk_shift, const int32_t* __restrict__ lc,
           const int32_t* __restrict__ n_lc, const int* __restrict__ sub_shift_dev, uint32_t G,
           int32_t* __restrict__ subh, const unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    extern __shared__ int32_t sh_hist[];
    if (*bad != (unsigned long long)kNoBad) return;
    const int ss = *sub_shift_dev;
    if (ss == 0 || (int)blockIdx.x >= (*n_lc << ss)) return;
    const int64_t c = lc[blockIdx.x >> ss];
    const int sb = (int)blockIdx.x & ((1 << ss) - 1);
    const int64_t c0 = (c << chunk_shift) + ((int64_t)sb << (chunk_shift - ss));
    const int64_t c1 = min64(n, c0 + ((int64_t)1 << (chunk_shift - ss)));
    for (int i = threadIdx.x; i < (int)G; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
    for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
        const uint32_t g = keys[i];
        if (g < G) atomicAdd(&sh_hist[g], 1);
    }
    __syncthreads();
    int32_t* dst = subh + (int64_t)blockIdx.x * G;
    for (int i = threadIdx.x; i < (int)G; i += blockDim.x) dst[i] = sh_hist[i];
}

__global__ void __launch_bounds__(256)
k_sub_scan(const int32_t* __restrict__ gpre, const int32_t* __restrict__ lc, const int32_t* __restrict__ n_lc,
           const int* __restrict__ sub_shift_dev, uint32_t G, const int32_t* __restrict__ subh,
           int32_t* __restrict__ gsub, const unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    if (*bad != (unsigned long long)kNoBad) return;
    const int ss = *sub_shift_dev;
    if (ss == 0) return;
    const int64_t total = (int64_t)*n_lc * G;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int li = (int)(i / G);
        const uint32_t g = (uint32_t)(i - (int64_t)li * G);
        int32_t run = gpre[(int64_t)lc[li] * G + g];
        const int64_t u0 = (int64_t)li << ss;
        int32_t h[16];
#pragma unroll
        for (int sb = 0; sb < 16; ++sb) h[sb] = sb < (1 << ss) ? subh[(u0 + sb) * G + g] : 0;   // all in flight
#pragma unroll
        for (int sb = 0; sb < 16; ++sb) {
            if (sb < (1 << ss)) gsub[(u0 + sb) * G + g] = run;
            if (run >= 0) run += h[sb];
        }
    }
}

__host__ __device__ constexpr size_t rank_smem_bytes(uint32_t G) {
    return (size_t)kRankWarps * kRankStages * kRankSub * 8 + (size_t)((G + 31) & ~31u) * 4 + 128;
}


// BITS > 0: group matching from BITS ballots (keys < 2^BITS); 0: MATCH
template <int BITS>
__global__ void __launch_bounds__(kRankWarps * 32)
k_rank_place(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin, uint32_t* __restrict__ kout,
             int32_t* __restrict__ vout, int64_t n, int chunk_shift, const int32_t* __restrict__ lc,
             const int32_t* __restrict__ n_lc, const int32_t* __restrict__ gpre, const int32_t* __restrict__ gstart,
             uint32_t G, const int32_t* __restrict__ n_live, const unsigned long long* __restrict__ bad,
             const int* __restrict__ sub_shift_dev = nullptr, const int32_t* __restrict__ gsub = nullptr) { SS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char rank_sm[];
    uint32_t* stage_k = (uint32_t*)rank_sm;                            // [warp][stage][kRankSub]
    int32_t* stage_v = (int32_t*)(stage_k + kRankWarps * kRankStages * kRankSub);
    uint32_t* cur = (uint32_t*)(stage_v + kRankWarps * kRankStages * kRankSub);   // [G]
    if (*bad != (unsigned long long)kNoBad) return;
    if (*n_live == 0) return;
    // few live chunks (a small kept set, e.g. C1): each is cut into 2^ss
    // sub-chunks placed by CTAs of their own, from sub-chunk prefixes (gsub)
    const int ss = sub_shift_dev ? *sub_shift_dev : 0;
    if ((int)blockIdx.x >= (*n_lc << ss)) return;
    const int64_t c = lc[blockIdx.x >> ss];
    const int sb = (int)blockIdx.x & ((1 << ss) - 1);
    const int32_t* pre = ss ? gsub + (int64_t)blockIdx.x * G : gpre + c * (int64_t)G;
    const int64_t c0 = (c << chunk_shift) + ((int64_t)sb << (chunk_shift - ss));
    if (c0 >= n) return;
    for (uint32_t g0 = threadIdx.x; g0 < G; g0 += 4 * blockDim.x) {
        int32_t p[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t g = g0 + u * blockDim.x;
            p[u] = g < G ? pre[g] : -1;
            b[u] = g < G ? gstart[g] : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t g = g0 + u * blockDim.x;
            if (g < G) cur[g] = p[u] < 0 ? 0x80000000u : (uint32_t)(b[u] + p[u]);
        }
    }
    const int cn = (int)min64((int64_t)1 << (chunk_shift - ss), n - c0);
    const int nsub = (cn + kRankSub - 1) / kRankSub;
    const int w = (int)warp_id();
    const unsigned lane = lane_id();
    uint32_t* my_k = stage_k + w * kRankStages * kRankSub;
    int32_t* my_v = stage_v + w * kRankStages * kRankSub;
    // full, aligned sub-tiles arrive by two bulk copies (1 KB each) on the
    // warp's mbarrier of the slot; the rest by per-lane cp.async
    __shared__ uint64_t rbar[kRankWarps][kRankStages];
    unsigned bulk_slots = 0, bulk_phase = 0;       // warp-uniform bit per slot
    if (lane == 0)
        for (int q = 0; q < kRankStages; ++q) mbar_init1(&rbar[w][q]);
    __syncwarp();
    // stage sub-tile s of this warp into ring slot q (always commits a group)
    auto stage = [&](int s, int q) {
        if (s < nsub) {
            const int64_t t0 = c0 + (int64_t)s * kRankSub;
            const int tn = min(kRankSub, cn - s * kRankSub);
            uint32_t* dk = my_k + q * kRankSub;
            int32_t* dv = my_v + q * kRankSub;
            if (tn == kRankSub && (((uintptr_t)(kin + t0) | (uintptr_t)(vin + t0)) & 15) == 0) {
                if (lane == 0) bulk_load2(dk, kin + t0, dv, vin + t0, kRankSub * 4, &rbar[w][q]);
                bulk_slots |= 1u << q;
            } else {
                bulk_slots &= ~(1u << q);
                for (int li = (int)lane; li < tn; li += 32) {
                    cp_async4(dk + li, kin + t0 + li);
                    cp_async4(dv + li, vin + t0 + li);
                }
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int q = 0; q < kRankStages; ++q) stage(w + q * kRankWarps, q);
    __syncthreads();                             // cursors initialised
    const unsigned lt = lanemask_lt();
    const uint32_t cur_sa = (uint32_t)__cvta_generic_to_shared(cur);
    const uint32_t dummy_sa = cur_sa + ((G + 31u) & ~31u) * 4u;     // [32], 128-B aligned
    // one sub-tile; FULL: all kRankSub tuples present (every sub-tile but
    // the batch's last), so no validity tests
    auto sub_tile = [&](auto full_c, int s, int q, int tn) {
        constexpr bool FULL = decltype(full_c)::value;
        uint32_t key[kRankItems];
        int32_t val[kRankItems];
#pragma unroll
        for (int j = 0; j < kRankItems; ++j) {
            const int li = j * 32 + (int)lane;
            key[j] = (FULL || li < tn) ? my_k[q * kRankSub + li] : 0xffffffffu;
            val[j] = (FULL || li < tn) ? my_v[q * kRankSub + li] : 0;
        }
        __syncwarp();                            // slot q is read: refill it
        stage(s + kRankStages * kRankWarps, q);
        unsigned peers[kRankItems];
#pragma unroll
        for (int j = 0; j < kRankItems; ++j) {
            if (BITS && (j & 3) < kRankBallot)
                peers[j] = FULL ? match_bits_all<BITS>(key[j]) : match_bits<BITS>(key[j], key[j] != 0xffffffffu);
            else
                peers[j] = __match_any_sync(SS_FULL, key[j]);
        }
        // leader (highest peer) of each item's group in its round, the
        // round's count for the leader (0 elsewhere) and the cursor address,
        // all ready before the ordered section
        uint32_t lead[kRankItems], cnt[kRankItems], addr[kRankItems], old[kRankItems];
#pragma unroll
        for (int j = 0; j < kRankItems; ++j) {
            const bool valid = FULL || key[j] != 0xffffffffu;
            lead[j] = 31u - (uint32_t)__clz(peers[j]);
            cnt[j] = (valid && lane == lead[j]) ? (uint32_t)__popc(peers[j]) : 0u;
            addr[j] = cnt[j] ? cur_sa + key[j] * 4u : dummy_sa + lane * 4u;
            old[j] = 0;
            asm volatile("" :: "r"(cnt[j]), "r"(addr[j]));
        }
        // ---- in sub-tile order across the warps: advance the cursors
        // one asm block of unpredicated atomics in round order: non-leaders
        // add 0 to a private dummy word (bank = lane), so the warp issues 8
        // ATOMS back to back with no branches (a per-round predicated asm +
        // __syncwarp compiled to a divergent branch per round, ~9 dependent
        // instructions each on this serial chain)
        if (s > 0) named_bar_sync(w, 64);
        static_assert(kRankItems == 8, "the ordered section below is written for 8 rounds");
        asm volatile("{\n\t"
                     "atom.shared.add.u32 %0, [%8], %16;\n\t"
                     "atom.shared.add.u32 %1, [%9], %17;\n\t"
                     "atom.shared.add.u32 %2, [%10], %18;\n\t"
                     "atom.shared.add.u32 %3, [%11], %19;\n\t"
                     "atom.shared.add.u32 %4, [%12], %20;\n\t"
                     "atom.shared.add.u32 %5, [%13], %21;\n\t"
                     "atom.shared.add.u32 %6, [%14], %22;\n\t"
                     "atom.shared.add.u32 %7, [%15], %23;\n\t}"
                     : "+r"(old[0]), "+r"(old[1]), "+r"(old[2]), "+r"(old[3]),
                       "+r"(old[4]), "+r"(old[5]), "+r"(old[6]), "+r"(old[7])
                     : "r"(addr[0]), "r"(addr[1]), "r"(addr[2]), "r"(addr[3]),
                       "r"(addr[4]), "r"(addr[5]), "r"(addr[6]), "r"(addr[7]),
                       "r"(cnt[0]), "r"(cnt[1]), "r"(cnt[2]), "r"(cnt[3]),
                       "r"(cnt[4]), "r"(cnt[5]), "r"(cnt[6]), "r"(cnt[7])
                     : "memory");
        if (s + 1 < nsub) named_bar_arrive((w + 1) % kRankWarps, 64);
        // ---- scatter (never-stored runs have bit 31 set in their cursor)
#pragma unroll
        for (int j = 0; j < kRankItems; ++j) {
            const uint32_t base = __shfl_sync(SS_FULL, old[j], lead[j]);
            const uint32_t pos = base + (uint32_t)__popc(peers[j] & lt);
            if ((FULL || key[j] != 0xffffffffu) && !(pos & 0x80000000u)) {
                vout[pos] = val[j];
                if (kout) kout[pos] = key[j];
            }
        }
    };
    int q = 0;
    for (int s = w; s < nsub; s += kRankWarps) {
        cp_async_wait_n<kRankStages - 1>();
        if ((bulk_slots >> q) & 1u) {
            mbar_wait_parity(&rbar[w][q], (bulk_phase >> q) & 1u);
            bulk_phase ^= 1u << q;
        }
        __syncwarp();
        const int tn = min(kRankSub, cn - s * kRankSub);
        if (tn == kRankSub) sub_tile(std::integral_constant<bool, true>{}, s, q, tn);
        else sub_tile(std::integral_constant<bool, false>{}, s, q, tn);
        q = (q + 1 == kRankStages) ? 0 : q + 1;
    }
    cp_async_wait_0();
}

// histogram of destination owners for the multi-GPU route (<= 16 owners)
__global__ void __launch_bounds__(256)
k_owner_hist(const uint32_t* __restrict__ keys, int64_t n, uint32_t G, const int32_t* __restrict__ owner,
             unsigned long long* __restrict__ counts, unsigned long long* __restrict__ bad) { SS_PDL_ENTRY();
    __shared__ uint32_t h[16];
    if (threadIdx.x < 16) h[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        if (k >= G) { atomicMin(bad, (unsigned long long)i); continue; }
        atomicAdd(&h[owner[k]], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 16 && h[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

}  // namespace ss
