// common.cuh -- shared device helpers for the skewstream B200 engine.
//
// Everything here is integer / byte work: scans, histograms and the
// decoupled look-back status words of the stable multisplit.  Nothing on
// this path is GEMM-shaped, so there are no tensor-core paths; the
// kernels are tuned for coalescing, L2 residency and SM-count-sized grids.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define SS_WARP 32
#define SS_FULL 0xffffffffu

// Programmatic dependent launch: every kernel of the library is launched
// with programmatic stream serialisation (engine.cu ss_launch), so its CTAs
// may be scheduled while the previous kernel of the stream drains; the
// first thing each kernel does is wait for that predecessor to complete
// (griddepcontrol.wait -- a no-op without a programmatic predecessor) and
// let its own successor be scheduled (launch_dependents).  The successor
// still waits for this grid's completion and memory flush before it runs.
#define SS_PDL_ENTRY() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

namespace ss {

constexpr int kNumSM = 148;                 // B200: 2 dies x 74 SMs
constexpr int64_t kNoBad = 0x7fffffffffffffffLL;

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// relaxed gpu-scope 64-bit load/store for the look-back status words: the
// payload (a count) lives in the same word as its flag, so no fence is
// needed between payload and flag.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// streaming loads of the input batch: read once, do not keep in L1, first
// to leave L2 (the sort ping-pong buffers are what must stay resident).
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const void* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// Ampere-style asynchronous global -> shared copies (4 bytes, any alignment)
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(sa), "l"(gmem) : "memory");
}
// 16-byte copy, L1 bypassed (both addresses 16-byte aligned)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_n() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

// named CTA barriers (id 0 is __syncthreads): a producer warp arrives, a
// consumer warp waits; prior shared-memory writes of the producer are
// visible to the consumer after the wait
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}

// match_bits for a full warp of valid values
template <int BITS>
__device__ __forceinline__ unsigned match_bits_all(uint32_t v) {
    unsigned m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        const unsigned bb = __ballot_sync(SS_FULL, v & (1u << b));
        m &= (v & (1u << b)) ? bb : ~bb;
    }
    return m;
}

// __match_any_sync for a BITS-bit value built from BITS ballots (plus one
// for the valid flag): fixed cost, where the MATCH instruction's cost grows
// with the number of distinct values in the warp
template <int BITS>
__device__ __forceinline__ unsigned match_bits(uint32_t v, bool valid) {
    unsigned m = __ballot_sync(SS_FULL, valid);
    m = valid ? m : ~m;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        const bool bit = (v >> b) & 1u;
        const unsigned bb = __ballot_sync(SS_FULL, bit);
        m &= bit ? bb : ~bb;
    }
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(SS_FULL, v, o);
    return v;
}
__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(SS_FULL, v, o));
    return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(SS_FULL, v, o));
    return v;
}

// inclusive warp scan
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(SS_FULL, v, o);
        if ((int)lane_id() >= o) v += n;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread (blockDim.x <= 1024).
// `smem` needs 33 slots.  Returns the exclusive prefix; *total gets the sum.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* smem, T* total) {
    const unsigned w = warp_id(), l = lane_id(), nw = (blockDim.x + 31) >> 5;
    T inc = warp_incl_scan(v);
    if (l == 31) smem[w] = inc;
    __syncthreads();
    if (w == 0) {
        T s = (l < nw) ? smem[l] : T(0);
        T si = warp_incl_scan(s);
        if (l < nw) smem[l] = si - s;
        if (l == nw - 1) smem[32] = si;
    }
    __syncthreads();
    T res = smem[w] + inc - v;
    *total = smem[32];
    __syncthreads();
    return res;
}

// block_excl_scan without the trailing barrier: only for a caller whose
// next use of `smem` is behind another __syncthreads
template <typename T>
__device__ __forceinline__ T block_excl_scan_nt(T v, T* smem, T* total) {
    const unsigned w = warp_id(), l = lane_id(), nw = (blockDim.x + 31) >> 5;
    T inc = warp_incl_scan(v);
    if (l == 31) smem[w] = inc;
    __syncthreads();
    if (w == 0) {
        T s = (l < nw) ? smem[l] : T(0);
        T si = warp_incl_scan(s);
        if (l < nw) smem[l] = si - s;
        if (l == nw - 1) smem[32] = si;
    }
    __syncthreads();
    *total = smem[32];
    return smem[w] + inc - v;
}

// look-back status word: [epoch:30 | flag:2 | count:32].  Epochs advance by
// 2 per placement (one per pass) and stay in [1, 2^30); a wrap takes 2^29
// placements.
__host__ __device__ __forceinline__ uint32_t epoch_next(uint32_t e) {
    return (e + 2u >= (1u << 30) - 2u) ? 1u : e + 2u;
}
constexpr unsigned long long kFlagAgg = 1ull, kFlagInc = 2ull;
__device__ __forceinline__ unsigned long long lb_pack(uint32_t epoch, unsigned long long flag, uint32_t cnt) {
    return ((unsigned long long)epoch << 34) | (flag << 32) | (unsigned long long)cnt;
}

// ---- bulk asynchronous copies (TMA engine, no tensor map) on an mbarrier --
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// two equal-size global -> shared copies completing on `bar` (16-byte
// aligned, size a multiple of 16); the streamed input leaves L2 first
__device__ __forceinline__ void bulk_load2(void* d0, const void* s0, void* d1, const void* s1, unsigned bytes,
                                           uint64_t* bar) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(2 * bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"((unsigned)__cvta_generic_to_shared(d0)), "l"(s0), "r"(bytes), "r"(b), "l"(pol) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"((unsigned)__cvta_generic_to_shared(d1)), "l"(s1), "r"(bytes), "r"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MBW_%=;\n}" :: "r"(a), "r"(parity) : "memory");
}

}  // namespace ss
