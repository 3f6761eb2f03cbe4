// Device-wide exclusive prefix sums (reduce-then-scan, recursive over the
// per-block totals).  Used for tile-overlap offsets, survivor compaction and
// varint byte offsets.
#include "ss_internal.cuh"

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// exclusive block scan of one value per thread; returns the block total in *total
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t* total) {
    __shared__ uint64_t warp_tot[SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t incl = warp_incl_scan(v);
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < SCAN_THREADS / 32 ? warp_tot[lane] : 0;
        uint64_t wi = warp_incl_scan(w);
        if (lane < SCAN_THREADS / 32) warp_tot[lane] = wi - w;
        if (lane == SCAN_THREADS / 32 - 1) *total = wi;
    }
    __syncthreads();
    uint64_t out = warp_tot[warp] + incl - v;
    __syncthreads();
    return out;
}

template <typename Tin>
__global__ void k_block_sums(const Tin* __restrict__ in, int64_t n, uint64_t* __restrict__ sums) {
    SS_PDL_WAIT();
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i)
        if (base + i < n) s += (uint64_t)in[base + i];
    __shared__ uint64_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <typename Tin>
__global__ void k_block_scan(const Tin* __restrict__ in, int64_t n, const uint64_t* __restrict__ offsets,
                             uint64_t* __restrict__ out, uint64_t* __restrict__ total) {
    SS_PDL_WAIT();
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint64_t v[SCAN_ITEMS];
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = base + i < n ? (uint64_t)in[base + i] : 0;
        s += v[i];
    }
    __shared__ uint64_t tot;
    uint64_t run = block_excl_scan(s, &tot) + (offsets ? offsets[blockIdx.x] : 0);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_THREADS - 1) *total = run;
}

__global__ void k_zero_u64(uint64_t* p) {
    SS_PDL_WAIT(); *p = 0; }

template <typename Tin>
int scan_impl(ss_ctx* ctx, const Tin* in, uint64_t* out, int64_t n, uint64_t* total) {
    if (n <= 0) {
        if (total) {
            SS_CUDA(ctx, ss_launch((k_zero_u64), dim3(1), dim3(1), 0, ctx->stream, total));
            SS_CHECK_LAUNCH(ctx);
        }
        return SS_OK;
    }
    int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    uint64_t* offs = nullptr;
    if (nb > 1) {
        uint64_t* sums = SS_SCRATCH(ctx, uint64_t, nb);
        offs = SS_SCRATCH(ctx, uint64_t, nb);
        if (!sums || !offs) return SS_ERR_CUDA;
        SS_CUDA(ctx, ss_launch((k_block_sums<Tin>), dim3((unsigned)nb), dim3(SCAN_THREADS), 0, ctx->stream, in, n, sums));
        SS_CHECK_LAUNCH(ctx);
        SS_TRY(scan_impl<uint64_t>(ctx, sums, offs, nb, nullptr));
    }
    SS_CUDA(ctx, ss_launch((k_block_scan<Tin>), dim3((unsigned)nb), dim3(SCAN_THREADS), 0, ctx->stream, in, n, offs, out, total));
    SS_CHECK_LAUNCH(ctx);
    return SS_OK;
}

}  // namespace

int ss_scan_u32_to_u64(ss_ctx* ctx, const uint32_t* in, uint64_t* out, int64_t n, uint64_t* total) {
    return scan_impl<uint32_t>(ctx, in, out, n, total);
}

int ss_scan_u8_to_u64(ss_ctx* ctx, const uint8_t* in, uint64_t* out, int64_t n, uint64_t* total) {
    return scan_impl<uint8_t>(ctx, in, out, n, total);
}
