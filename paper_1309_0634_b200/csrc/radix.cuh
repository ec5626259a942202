// radix.cuh -- K3d: stable placement for large group domains (G > 2^14) as
// LSD passes over 7-bit digits of the group id, with NO cross-tile
// look-back: every pass first histograms its tiles, scans the histograms,
// then places each tile independently.
//
// Reference behaviour: reorder_batch (partition.py:161-178) / the stable
// regroup of ingest_sequence (engine.py:274-280) -- each group's kept
// tuples contiguous, in arrival order, the run of group g at gstart[g].
//
// Why this shape on B200 (measured): the decoupled look-back of
// a one-sweep pass stalls every tile on its predecessors' status words, and
// wide digits (10 bits, 1024 bins) cost more per-bin work per 4096-tuple
// tile than the tuples themselves.  Here a pass is
//   k_os_up    a CTA per 8192-tuple tile: per-warp shared histograms of the
//              digit -> hist[tile][128] (pass 0 also drops the tuples that
//              are never stored, from the kept-count rows of k_batch_stats)
//   k_os_red / k_os_top / k_os_down
//              column scan of hist over the tiles (blocks of 16 tiles),
//              digit bases from the digit totals -> the global output base
//              of every (tile, digit)
//   k_os_pass  persistent, one CTA per SM walking tiles c, c + 148, ...:
//              a tile's keys and values arrive by two cp.async.bulk copies
//              on an mbarrier, the next tile's copies in flight while the
//              current one is ranked (double-buffered); warps rank
//              their 256 tuples in arrival order against per-warp digit
//              histograms (MATCH and ballot-built matches alternating, so the
//              MIO and ALU pipes share the work); the tile is sorted by digit
//              in shared memory, then written as contiguous runs per digit
// 128 bins and 8192-tuple tiles give ~64-tuple runs per (tile, digit), so
// the scattered writes are whole sectors.  Traffic per pass: keys 4 B (up)
// + keys and values 8 B read + 8 B written (4 B in the last pass).
#pragma once

#include "common.cuh"

namespace ss {

constexpr int kOsBits = 7;                              // default digit width
constexpr int kOsBitsWide = 10;                         // wide variant (2 passes up to 2^20 groups)
constexpr int kOsTile = 8192;
constexpr int kOsThreads = 1024;
constexpr int kOsItems = kOsTile / kOsThreads;          // 8 per thread
constexpr int kOsWarps = kOsThreads / 32;
constexpr int kOsBlkTiles = 8;                          // tiles per block of the column scan (C4: 256 blocks: 16-tile blocks left k_os_red / k_os_down on 128 CTAs, under one wave)
constexpr int kOsMaxPass = 4;

template <int BITS>
struct OsSmem {
    static constexpr int BINS = 1 << BITS;
    static constexpr size_t keys = 0;                                   // u32[2][kOsTile]
    static constexpr size_t vals = keys + (size_t)2 * kOsTile * 4;      // i32[2][kOsTile]
    static constexpr size_t wh = vals + (size_t)2 * kOsTile * 4;        // u16[kOsWarps][BINS]
    static constexpr size_t base = wh + (size_t)kOsWarps * BINS * 2;    // u32[BINS] global base - local start
    static constexpr size_t lst = base + (size_t)BINS * 4;              // u32[BINS] local start
    static constexpr size_t bar = lst + (size_t)BINS * 4;               // u64[2]
    static constexpr size_t bytes = bar + 16;
};

struct OsArgs {
    const uint32_t* kin;
    const int32_t* vin;
    uint32_t* kout;             // null: values only (last pass, no trace)
    int32_t* vout;
    int64_t n;                  // tuples (pass 0), else read from n_dev
    const int32_t* n_dev;       // kept total (passes >= 1)
    int shift;
    uint32_t mask;
    uint32_t* hist;             // [tiles][BINS] counts -> output bases
    uint32_t* bsum;             // [blocks][BINS]
    uint32_t* dtot;             // [BINS] digit totals
    // pass 0: drop never-stored tuples (live = kept counts per count chunk)
    const int32_t* live;
    int chunk_shift;
    uint32_t G;
    const int* any_dead;
    int match;                  // 0: ballot-built matches, 1: alternate with MATCH, 2: MATCH only
    const unsigned long long* bad;
};

__device__ __forceinline__ int64_t os_count(const OsArgs& a) { return a.n_dev ? (int64_t)*a.n_dev : a.n; }

__device__ __forceinline__ bool os_live(const OsArgs& a, bool drop, int64_t i, uint32_t g) {
    return !drop || a.live[(i >> a.chunk_shift) * (int64_t)a.G + g] > 0;
}

// kOsUpTiles tiles per CTA: every load of the CTA's tiles is issued before
// the histograms are zeroed, so their latency overlaps the zeroing barrier
// (one tile per CTA left the load pipe idle through zero / barrier / flush)
constexpr int kOsUpTiles = 2;

template <int BITS>
__global__ void __launch_bounds__(kOsThreads)
k_os_up(OsArgs a) { SS_PDL_ENTRY();
    constexpr int BINS = 1 << BITS;
    constexpr int NH = BINS <= 128 ? kOsWarps : 4;      // sub-histograms (one per warp for narrow digits)
    constexpr int TPC = kOsUpTiles;
    __shared__ uint32_t wh[TPC][NH][BINS];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int64_t n = os_count(a);
    const int64_t tile0 = (int64_t)blockIdx.x * TPC;
    if (tile0 * kOsTile >= n) return;
    const bool drop = a.live && *a.any_dead;
    const unsigned h = warp_id() % NH;
    // 8 consecutive tuples per thread and tile: two 128-bit loads each
    const int i0 = threadIdx.x * kOsItems;
    uint32_t k[TPC][kOsItems];
    int tn[TPC];
#pragma unroll
    for (int t = 0; t < TPC; ++t) {
        const int64_t t0 = (tile0 + t) * kOsTile;
        tn[t] = t0 < n ? (int)min64(kOsTile, n - t0) : 0;
        if (i0 + kOsItems <= tn[t] && ((uintptr_t)(a.kin + t0) % 16) == 0) {
            const uint4 x = ld_stream_v4(a.kin + t0 + i0), y = ld_stream_v4(a.kin + t0 + i0 + 4);
            k[t][0] = x.x; k[t][1] = x.y; k[t][2] = x.z; k[t][3] = x.w;
            k[t][4] = y.x; k[t][5] = y.y; k[t][6] = y.z; k[t][7] = y.w;
        } else {
#pragma unroll
            for (int q = 0; q < kOsItems; ++q) k[t][q] = (i0 + q < tn[t]) ? a.kin[t0 + i0 + q] : 0u;
        }
    }
    for (int i = threadIdx.x; i < TPC * NH * BINS; i += blockDim.x) (&wh[0][0][0])[i] = 0;
    __syncthreads();
#pragma unroll
    for (int t = 0; t < TPC; ++t) {
        const int64_t t0 = (tile0 + t) * kOsTile;
#pragma unroll
        for (int q = 0; q < kOsItems; ++q)
            if (i0 + q < tn[t] && os_live(a, drop, t0 + i0 + q, k[t][q])) atomicAdd(&wh[t][h][(k[t][q] >> a.shift) & a.mask], 1u);
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < TPC; ++t) {
        if (tn[t] == 0) continue;
        for (int d = threadIdx.x; d < BINS; d += blockDim.x) {
            uint32_t s = 0;
#pragma unroll 4
            for (int q = 0; q < NH; ++q) s += wh[t][q][d];
            a.hist[(tile0 + t) * BINS + d] = s;
        }
    }
}

// block b of kOsBlkTiles tiles: per digit (t mod BINS) and tile slice
// (t / BINS) -- 1024 / BINS slices of the block's tiles
template <int BITS>
__global__ void __launch_bounds__(1024)
k_os_red(OsArgs a) { SS_PDL_ENTRY();
    constexpr int BINS = 1 << BITS, J = 1024 / BINS, per = kOsBlkTiles / J;
    __shared__ uint32_t part[J][BINS];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int64_t ntile = (os_count(a) + kOsTile - 1) / kOsTile;
    const int64_t tb = (int64_t)blockIdx.x * kOsBlkTiles;
    if (tb >= ntile) return;
    const int d = threadIdx.x & (BINS - 1), j = threadIdx.x / BINS;
    uint32_t s = 0;
    for (int q = 0; q < per; ++q) {
        const int64_t t = tb + j * per + q;
        if (t < ntile) s += a.hist[t * BINS + d];
    }
    part[j][d] = s;
    __syncthreads();
    if (j == 0) {
        uint32_t tot = 0;
#pragma unroll
        for (int q = 0; q < J; ++q) tot += part[q][d];
        a.bsum[(int64_t)blockIdx.x * BINS + d] = tot;
    }
}

// per digit: exclusive scan of the block sums (in place) and the digit's
// total (dtot).  CTA x owns 32 digits (lane = digit); its 32 warps own
// contiguous block ranges, so every load is a coalesced 128-byte row
// segment and the scan over the blocks is one pass plus a cross-warp
// prefix (a thread per digit walking all blocks serially cost ~29 us per
// pass at C4).  The digit bases (scan over the totals) are formed by every
// k_os_down CTA from dtot.
template <int BITS>
__global__ void __launch_bounds__(1024)
k_os_top(OsArgs a) { SS_PDL_ENTRY();
    __shared__ uint32_t part[32][33];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int64_t ntile = (os_count(a) + kOsTile - 1) / kOsTile;
    const int nblk = (int)((ntile + kOsBlkTiles - 1) / kOsBlkTiles);
    const unsigned lane = lane_id(), w = warp_id();
    const int d = (int)blockIdx.x * 32 + (int)lane;
    constexpr int BINS = 1 << BITS;
    const int per = (nblk + 31) / 32;
    const int b0 = min(nblk, (int)w * per), b1 = min(nblk, b0 + per);
    uint32_t s = 0;
    for (int b = b0; b < b1; ++b) s += a.bsum[(int64_t)b * BINS + d];
    part[w][lane] = s;
    __syncthreads();
    uint32_t run = 0, tot = 0;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
        const uint32_t v = part[q][lane];
        run += (q < (int)w) ? v : 0u;
        tot += v;
    }
    for (int b = b0; b < b1; ++b) {
        uint32_t* p = a.bsum + (int64_t)b * BINS + d;
        const uint32_t c = *p;
        *p = run;
        run += c;
    }
    if (w == 0) a.dtot[d] = tot;
}

// per tile and digit: global output base (in place over hist)
template <int BITS>
__global__ void __launch_bounds__(1024)
k_os_down(OsArgs a) { SS_PDL_ENTRY();
    constexpr int BINS = 1 << BITS, J = 1024 / BINS, per = kOsBlkTiles / J;
    __shared__ uint32_t part[J][BINS];
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int64_t ntile = (os_count(a) + kOsTile - 1) / kOsTile;
    const int64_t tb = (int64_t)blockIdx.x * kOsBlkTiles;
    if (tb >= ntile) return;
    const int d = threadIdx.x & (BINS - 1), j = threadIdx.x / BINS;
    uint32_t s = 0;
    for (int q = 0; q < per; ++q) {
        const int64_t t = tb + j * per + q;
        if (t < ntile) s += a.hist[t * BINS + d];
    }
    part[j][d] = s;
    // digit bases: exclusive scan of the digit totals
    __shared__ uint32_t sdb[BINS];
    __shared__ uint32_t red[33];
    {
        const uint32_t t = threadIdx.x < BINS ? a.dtot[threadIdx.x] : 0u;
        uint32_t all;
        const uint32_t ex = block_excl_scan(t, red, &all);
        if (threadIdx.x < BINS) sdb[threadIdx.x] = ex;
    }
    __syncthreads();
    uint32_t run = a.bsum[(int64_t)blockIdx.x * BINS + d] + sdb[d];
    for (int q = 0; q < j; ++q) run += part[q][d];
    for (int q = 0; q < per; ++q) {
        const int64_t t = tb + j * per + q;
        if (t < ntile) {
            uint32_t* p = a.hist + t * BINS + d;
            const uint32_t c = *p;
            *p = run;
            run += c;
        }
    }
}

// ---- mbarrier + bulk copies ------------------------------------------------
__device__ __forceinline__ void os_mbar_init(uint64_t* bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void os_load_tile(void* dk, const void* sk, void* dv, const void* sv, unsigned bytes,
                                             uint64_t* bar) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(2 * bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"((unsigned)__cvta_generic_to_shared(dk)), "l"(sk), "r"(bytes), "r"(b), "l"(pol) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"((unsigned)__cvta_generic_to_shared(dv)), "l"(sv), "r"(bytes), "r"(b), "l"(pol) : "memory");
}
// one more bulk copy on the same mbarrier transaction (caller adds its
// bytes to the expected count first)
__device__ __forceinline__ void os_load_extra(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                    "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void os_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;"
                 :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void os_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "OSW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra OSW_%=;\n}" :: "r"(a), "r"(parity) : "memory");
}

// persistent: CTA c places tiles c, c + gridDim.x, ...; the next tile's
// bulk copies are in flight while the current one is ranked and written
template <int BITS>
__global__ void __launch_bounds__(kOsThreads, 1)
k_os_pass(OsArgs a) { SS_PDL_ENTRY();
    constexpr int BINS = 1 << BITS;
    using OsSmem = ss::OsSmem<BITS>;
    extern __shared__ __align__(16) unsigned char osm[];
    uint16_t* wh = (uint16_t*)(osm + OsSmem::wh);
    uint32_t* gb = (uint32_t*)(osm + OsSmem::base);
    uint32_t* lst = (uint32_t*)(osm + OsSmem::lst);
    uint64_t* bar = (uint64_t*)(osm + OsSmem::bar);
    __shared__ uint32_t red[33];
    __shared__ uint32_t s_total;
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int64_t n = os_count(a);
    const bool drop = a.live && *a.any_dead;
    const unsigned w = warp_id(), lane = lane_id();
    const bool aligned = ((uintptr_t)a.kin % 16) == 0 && ((uintptr_t)a.vin % 16) == 0;
    auto full = [&](int64_t t) { return aligned && (t + 1) * kOsTile <= n; };
    auto issue = [&](int64_t t, int st) {
        if (t * kOsTile < n && full(t)) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            os_load_tile(osm + OsSmem::keys + (size_t)st * kOsTile * 4, a.kin + t * kOsTile,
                         osm + OsSmem::vals + (size_t)st * kOsTile * 4, a.vin + t * kOsTile, kOsTile * 4, &bar[st]);
        }
    };
    if (threadIdx.x == 0) {
        os_mbar_init(&bar[0]);
        os_mbar_init(&bar[1]);
        issue(blockIdx.x, 0);
    }
    __syncthreads();
    unsigned phase[2] = {0u, 0u};
    int k = 0;
    for (int64_t tile = blockIdx.x; tile * kOsTile < n; tile += gridDim.x, ++k) {
#ifdef SS_SORT_PROF
    long long _pt = clock64();
#endif
    const int st = k & 1;
    uint32_t* sk = (uint32_t*)(osm + OsSmem::keys + (size_t)st * kOsTile * 4);
    int32_t* sv = (int32_t*)(osm + OsSmem::vals + (size_t)st * kOsTile * 4);
    const int64_t t0 = tile * kOsTile;
    const int tn = (int)min64(kOsTile, n - t0);
    const bool bulk = full(tile);
    if (bulk) {
        os_wait(&bar[st], phase[st]);
        phase[st] ^= 1u;
    } else {
        for (int i = threadIdx.x; i < tn; i += blockDim.x) {
            sk[i] = a.kin[t0 + i];
            sv[i] = a.vin[t0 + i];
        }
    }
    SS_PT(0);
    // the other stage was last read by the previous tile (closing barrier)
    if (threadIdx.x == 0) issue(tile + gridDim.x, st ^ 1);
    uint16_t* my = wh + w * BINS;
    // 16-byte stores (a 10-bit digit's per-warp histogram is 2 KB)
    for (int i = lane; i < BINS / 8; i += 32) reinterpret_cast<uint4*>(my)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();                     // plain loads and zeroed histograms visible
    // rank: warp w owns tuples [w*256, (w+1)*256), round r = w*256 + 32r + lane
    uint32_t key[kOsItems];
    int32_t val[kOsItems];
    uint16_t rk[kOsItems];
    uint32_t ok = 0;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const int it = (int)w * (kOsItems * 32) + r * 32 + (int)lane;
        bool valid = it < tn;
        key[r] = valid ? sk[it] : 0u;
        val[r] = valid ? sv[it] : 0;
        valid = valid && os_live(a, drop, t0 + it, key[r]);
        const uint32_t d = (key[r] >> a.shift) & a.mask;
        // even rounds: MATCH (MIO pipe); odd rounds: matches built from
        // ballots (ALU pipe)
        const bool use_match = a.match == 2 || (a.match == 1 && !(r & 1));
        const unsigned peers = use_match ? __match_any_sync(SS_FULL, valid ? d : 0xffffffffu) : match_bits<BITS>(d, valid);
        uint16_t before = 0;
        if (valid) before = my[d];
        __syncwarp();
        if (valid) {
            ok |= 1u << r;
            rk[r] = (uint16_t)(before + __popc(peers & lt));
            if (lane == 31u - __clz(peers)) my[d] = (uint16_t)(before + __popc(peers));
        }
        __syncwarp();
    }
    __syncthreads();
    SS_PT(1);
    // per (digit, warp) exclusive offsets: thread (d = t >> 3, j = t & 7)
    // owns warps [4j, 4j+4) of digit d; the 8 threads of a digit are
    // consecutive lanes, so one shuffle scan gives their prefix
    {
        // J consecutive threads per digit, each owning WPT warps
        constexpr int J = kOsThreads / BINS, WPT = kOsWarps / J;
        const int d = threadIdx.x / J, j = threadIdx.x % J;
        uint32_t c[WPT], s = 0;
#pragma unroll
        for (int q = 0; q < WPT; ++q) {
            c[q] = wh[(WPT * j + q) * BINS + d];
            s += c[q];
        }
        uint32_t inc = s;
#pragma unroll
        for (int o = 1; o < J; o <<= 1) {
            const uint32_t x = __shfl_up_sync(SS_FULL, inc, o, J);
            if (j >= o) inc += x;
        }
        uint32_t ex = inc - s;
#pragma unroll
        for (int q = 0; q < WPT; ++q) {
            wh[(WPT * j + q) * BINS + d] = (uint16_t)ex;
            ex += c[q];
        }
        if (j == J - 1) lst[d] = inc;    // the digit's tile count (scanned below)
    }
    __syncthreads();
    SS_PT(2);
    if (threadIdx.x < BINS) {
        // exclusive scan of the digit counts (BINS threads, named barrier)
        const uint32_t cnt = lst[threadIdx.x];
        const uint32_t inc = warp_incl_scan(cnt);
        if (lane == 31) red[w] = inc;
        if (BINS == kOsThreads) __syncthreads(); else named_bar_sync(1, BINS);
        uint32_t add = 0;
        for (unsigned q = 0; q < w; ++q) add += red[q];
        const uint32_t ls = add + inc - cnt;
        lst[threadIdx.x] = ls;
        gb[threadIdx.x] = a.hist[tile * BINS + threadIdx.x] - ls;
        if (threadIdx.x == BINS - 1) s_total = ls + cnt;
    }
    __syncthreads();
    SS_PT(3);
    // local sort by digit into shared memory (every item is in registers)
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        if ((ok >> r) & 1u) {
            const uint32_t d = (key[r] >> a.shift) & a.mask;
            const uint32_t p = lst[d] + my[d] + rk[r];
            sk[p] = key[r];
            sv[p] = val[r];
        }
    }
    __syncthreads();
    SS_PT(4);
    // contiguous runs per digit to global memory (the tile's kept tuples)
    const int total = (int)s_total;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        const uint32_t k = sk[i];
        const uint32_t pos = gb[(k >> a.shift) & a.mask] + (uint32_t)i;
        a.vout[pos] = sv[i];
        if (a.kout) a.kout[pos] = k;
    }
    __syncthreads();                     // this stage and the histograms are free again
    SS_PT(5);
    }
}

// Variant for wide digits: 512 threads x 16 items per 8192-tuple tile, a
// single staged tile and 16 per-warp histograms (104 KB of shared memory,
// 64 registers), so TWO CTAs share an SM and one's ranking overlaps the
// other's copies and write-out (the 1024-thread kernel above holds a whole
// SM and double-buffers instead).  Same ranking / scan / local sort.
constexpr int kOs2Threads = 512;
constexpr int kOs2Warps = kOs2Threads / 32;
constexpr int kOs2Items = kOsTile / kOs2Threads;     // 16

template <int BITS>
struct Os2Smem {
    static constexpr int BINS = 1 << BITS;
    static constexpr size_t keys = 0;                                   // u32[kOsTile]
    static constexpr size_t vals = keys + (size_t)kOsTile * 4;          // i32[kOsTile]
    static constexpr size_t wh = vals + (size_t)kOsTile * 4;            // u16[kOs2Warps][BINS]
    static constexpr size_t base = wh + (size_t)kOs2Warps * BINS * 2;   // u32[BINS]
    static constexpr size_t lst = base + (size_t)BINS * 4;              // u32[BINS]
    static constexpr size_t bar = lst + (size_t)BINS * 4;               // u64
    static constexpr size_t bytes = bar + 16;
};

template <int BITS>
__global__ void __launch_bounds__(kOs2Threads, 2)
k_os_pass2(OsArgs a) { SS_PDL_ENTRY();
    constexpr int BINS = 1 << BITS;
    constexpr int DPT = (BINS + kOs2Threads - 1) / kOs2Threads;        // digits per thread (scans)
    using SM = ss::Os2Smem<BITS>;
    extern __shared__ __align__(16) unsigned char osm[];
    uint32_t* sk = (uint32_t*)(osm + SM::keys);
    int32_t* sv = (int32_t*)(osm + SM::vals);
    uint16_t* wh = (uint16_t*)(osm + SM::wh);
    uint32_t* gb = (uint32_t*)(osm + SM::base);
    uint32_t* lst = (uint32_t*)(osm + SM::lst);
    uint64_t* bar = (uint64_t*)(osm + SM::bar);
    __shared__ uint32_t red[33];
    __shared__ uint32_t s_total;
    if (*a.bad != (unsigned long long)kNoBad) return;
    const int64_t n = os_count(a);
    const bool drop = a.live && *a.any_dead;
    const unsigned w = warp_id(), lane = lane_id();
    const bool aligned = ((uintptr_t)a.kin % 16) == 0 && ((uintptr_t)a.vin % 16) == 0;
    if (threadIdx.x == 0) os_mbar_init(&bar[0]);
    __syncthreads();
    unsigned phase = 0u;
    for (int64_t tile = blockIdx.x; tile * kOsTile < n; tile += gridDim.x) {
        const int64_t t0 = tile * kOsTile;
        const int tn = (int)min64(kOsTile, n - t0);
        const bool bulk = aligned && tn == kOsTile;
        if (bulk) {
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                // the tile's digit bases (hist row, 4 B x BINS) ride on the
                // same transaction into gb; the expect_tx precedes the
                // arrive in os_load_tile so the phase cannot complete early
                os_expect(&bar[0], BINS * 4);
                os_load_extra(gb, a.hist + tile * BINS, BINS * 4, &bar[0]);
                os_load_tile(sk, a.kin + t0, sv, a.vin + t0, kOsTile * 4, &bar[0]);
                // the CTA's next tile into L2 while this one is ranked
                const int64_t t1 = t0 + (int64_t)gridDim.x * kOsTile;
                if (t1 + kOsTile <= n) {
                    l2_prefetch(a.kin + t1, kOsTile * 4);
                    l2_prefetch(a.vin + t1, kOsTile * 4);
                }
            }
            uint16_t* my = wh + w * BINS;
            for (int i = lane; i < BINS / 8; i += 32) reinterpret_cast<uint4*>(my)[i] = make_uint4(0u, 0u, 0u, 0u);
            os_wait(&bar[0], phase);
            phase ^= 1u;
        } else {
            for (int i = threadIdx.x; i < tn; i += blockDim.x) {
                sk[i] = a.kin[t0 + i];
                sv[i] = a.vin[t0 + i];
            }
            for (int i = threadIdx.x; i < BINS; i += blockDim.x) gb[i] = a.hist[tile * BINS + i];
            uint16_t* my = wh + w * BINS;
            for (int i = lane; i < BINS / 8; i += 32) reinterpret_cast<uint4*>(my)[i] = make_uint4(0u, 0u, 0u, 0u);
        }
        __syncthreads();                     // tile, digit bases and zeroed histograms visible
        uint16_t* my = wh + w * BINS;
        uint32_t key[kOs2Items];
        int32_t val[kOs2Items];
        // ranks packed two per register (16 separate u16 ranks spilled)
        uint32_t rkp[kOs2Items / 2];
#pragma unroll
        for (int r = 0; r < kOs2Items / 2; ++r) rkp[r] = 0u;
        uint32_t ok = 0;
        const unsigned lt = lanemask_lt();
#pragma unroll
        for (int r = 0; r < kOs2Items; ++r) {
            const int it = (int)w * (kOs2Items * 32) + r * 32 + (int)lane;
            bool valid = it < tn;
            key[r] = valid ? sk[it] : 0u;
            val[r] = valid ? sv[it] : 0;
            valid = valid && os_live(a, drop, t0 + it, key[r]);
            const uint32_t d = (key[r] >> a.shift) & a.mask;
            const bool use_match = a.match == 2 || (a.match == 1 && !(r & 1));
            const unsigned peers = use_match ? __match_any_sync(SS_FULL, valid ? d : 0xffffffffu) : match_bits<BITS>(d, valid);
            uint16_t before = 0;
            if (valid) before = my[d];
            __syncwarp();
            if (valid) {
                ok |= 1u << r;
                const uint32_t rank = (uint32_t)(uint16_t)(before + __popc(peers & lt));
                rkp[r >> 1] |= (r & 1) ? (rank << 16) : rank;
                if (lane == 31u - __clz(peers)) my[d] = (uint16_t)(before + __popc(peers));
            }
            __syncwarp();
        }
        __syncthreads();
        // per digit: exclusive offsets over the 16 warps, the digit's count
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            const int d = (int)threadIdx.x + q * kOs2Threads;
            if (d < BINS) {
                uint32_t run = 0;
#pragma unroll
                for (int v = 0; v < kOs2Warps; ++v) {
                    const uint32_t c = wh[v * BINS + d];
                    wh[v * BINS + d] = (uint16_t)run;
                    run += c;
                }
                lst[d] = run;
            }
        }
        __syncthreads();
        // exclusive scan of the digit counts: DPT consecutive digits per thread
        {
            uint32_t c[DPT], s = 0;
#pragma unroll
            for (int q = 0; q < DPT; ++q) {
                const int d = (int)threadIdx.x * DPT + q;
                c[q] = d < BINS ? lst[d] : 0u;
                s += c[q];
            }
            uint32_t tot;
            uint32_t ex = block_excl_scan(s, red, &tot);
#pragma unroll
            for (int q = 0; q < DPT; ++q) {
                const int d = (int)threadIdx.x * DPT + q;
                if (d < BINS) {
                    lst[d] = ex;
                    gb[d] -= ex;             // gb holds the tile's hist row
                }
                ex += c[q];
            }
            if (threadIdx.x == 0) s_total = tot;
        }
        __syncthreads();
        // local sort by digit into shared memory (every item is in registers)
#pragma unroll
        for (int r = 0; r < kOs2Items; ++r) {
            if ((ok >> r) & 1u) {
                const uint32_t d = (key[r] >> a.shift) & a.mask;
                const uint32_t p = lst[d] + my[d] + ((r & 1) ? (rkp[r >> 1] >> 16) : (rkp[r >> 1] & 0xffffu));
                sk[p] = key[r];
                sv[p] = val[r];
            }
        }
        __syncthreads();
        const int total = (int)s_total;
        // 4 independent LDS -> LDS -> STG chains per thread in flight
#pragma unroll 4
        for (int i = threadIdx.x; i < total; i += blockDim.x) {
            const uint32_t k = sk[i];
            const uint32_t pos = gb[(k >> a.shift) & a.mask] + (uint32_t)i;
            a.vout[pos] = sv[i];
            if (a.kout) a.kout[pos] = k;
        }
        __syncthreads();                     // the tile buffer and histograms are free again
    }
}

}  // namespace ss
